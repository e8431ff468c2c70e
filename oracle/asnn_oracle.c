/*
 * oracle/asnn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot path (arxiv/paper_2005_04347,
 * /root/reference/proj): compute_required -> segment -> flatten ->
 * eval_sequential, plus the sigmoid32 epilogue.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg load this file's
 * shared object, and only as the checker.  It is never linked into the product
 * library (paper_2005_04347_b200/libasnn_b200.so), which fails loudly when its
 * CUDA code is unavailable.
 *
 * Parity of this restatement is pinned two ways:
 *   1. the reference's own known-answer values (proj/tests/test_network.cpp,
 *      test_segmentation.cpp, test_layout.cpp, test_eval.cpp), restated in
 *      tests/test_oracle_golden.py;
 *   2. the reference itself, compiled from /root/reference by oracle/Makefile
 *      into oracle/_ref/libasnn_ref.so, whose outputs on seeded corpora are
 *      committed as tests/golden/*.npz by tests/golden/make_golden.py.
 *
 * Arithmetic contract: fp32 multiply then fp32 add in
 * the stored predecessor order, no FMA contraction (built with
 * -ffp-contract=off and no -march, i.e. SSE2 mulss/addss exactly like the
 * reference's x86-64 build), sigmoid in double through libm exp.
 *
 * All arrays are caller-allocated; sizes are upper bounds documented per
 * function so ctypes callers never need to free oracle memory.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_UNASSIGNED 0xFFFFFFFFu

enum {
    ORC_OK = 0,
    ORC_E_ARITY = 2,             /* InputArityMismatch        (eval.cpp:26-28)   */
    ORC_E_UNASSIGNED_OUTPUT = 3, /* UnassignedOutput          (layout.cpp:13-17) */
    ORC_E_INVALID = 5,
    ORC_E_OOM = 7,
};

/* ---- activation math: network.hpp:44-59 ------------------------------- */

double orc_sigmoid(double x) {
    /* network.hpp:45 -- 1/(1+exp(-4.97x)) in double, glibc exp. */
    const double v = 1.0 / (1.0 + exp(-4.97 * x));
    /* network.hpp:46-47 -- keep strictly inside (0,1). */
    if (v <= 0.0) return DBL_TRUE_MIN;
    if (v >= 1.0) return 1.0 - DBL_EPSILON / 2;
    return v;
}

float orc_sigmoid32(float x) {
    /* network.hpp:54-59 -- evaluated in double, rounded to float, clamped. */
    const float v = (float)orc_sigmoid((double)x);
    if (v <= 0.0f) return FLT_TRUE_MIN;
    if (v >= 1.0f) return 1.0f - FLT_EPSILON / 2;
    return v;
}

/* Vectorised helper for tests: out[i] = sigmoid32(in[i]). */
void orc_sigmoid32_many(const float* in, float* out, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_sigmoid32(in[i]);
}

/* ---- node_index: network.cpp:57-61 (binary search in sorted nodes) ------ */

static int64_t node_index(const uint32_t* nodes, uint32_t n, uint32_t id) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (nodes[mid] < id) lo = mid + 1;
        else hi = mid;
    }
    if (lo == n || nodes[lo] != id) return -1;
    return (int64_t)lo;
}

/* Adjacency in node-index space for edges with both endpoints known and
 * source != target -- the filter at network.cpp:226-228 and
 * segmentation.cpp:26-31.  Multiplicity is kept, as in the reference's
 * vector-of-vectors. */
typedef struct {
    uint64_t* off; /* [n+1] */
    uint32_t* adj; /* [m]   */
} csr_t;

static int build_csr(uint32_t n, const uint32_t* nodes, uint64_t n_edges, const uint32_t* src,
                     const uint32_t* dst, int by_target, csr_t* out) {
    out->off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    int64_t* si = (int64_t*)malloc((n_edges ? n_edges : 1) * sizeof(int64_t));
    int64_t* ti = (int64_t*)malloc((n_edges ? n_edges : 1) * sizeof(int64_t));
    if (!out->off || !si || !ti) {
        free(out->off); free(si); free(ti);
        return ORC_E_OOM;
    }
    uint64_t m = 0;
    for (uint64_t e = 0; e < n_edges; ++e) {
        si[e] = node_index(nodes, n, src[e]);
        ti[e] = node_index(nodes, n, dst[e]);
        if (si[e] >= 0 && ti[e] >= 0 && src[e] != dst[e]) {
            out->off[(by_target ? ti[e] : si[e]) + 1]++;
            ++m;
        }
    }
    for (uint32_t i = 0; i < n; ++i) out->off[i + 1] += out->off[i];
    out->adj = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
    uint64_t* cur = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
    if (!out->adj || !cur) {
        free(out->off); free(out->adj); free(cur); free(si); free(ti);
        return ORC_E_OOM;
    }
    memcpy(cur, out->off, ((size_t)n + 1) * sizeof(uint64_t));
    /* Edge order is preserved inside each list (push_back order). */
    for (uint64_t e = 0; e < n_edges; ++e) {
        if (si[e] >= 0 && ti[e] >= 0 && src[e] != dst[e]) {
            if (by_target) out->adj[cur[ti[e]]++] = (uint32_t)si[e];
            else out->adj[cur[si[e]]++] = (uint32_t)ti[e];
        }
    }
    free(cur); free(si); free(ti);
    return ORC_OK;
}

static void free_csr(csr_t* c) {
    free(c->off);
    free(c->adj);
}

/* ---- compute_required: network.cpp:222-255 -------------------------------
 * Backward reachability from the outputs over predecessor lists.
 * required[n_nodes] receives 1 for members (node-index space). */
int orc_compute_required(uint32_t n_nodes, const uint32_t* nodes, uint32_t n_out,
                         const uint32_t* outputs, uint64_t n_edges, const uint32_t* src,
                         const uint32_t* dst, uint8_t* required) {
    csr_t pred;
    int rc = build_csr(n_nodes, nodes, n_edges, src, dst, /*by_target=*/1, &pred);
    if (rc) return rc;
    memset(required, 0, n_nodes);
    uint32_t* stack = (uint32_t*)malloc(((size_t)n_nodes + 1) * sizeof(uint32_t));
    if (!stack) { free_csr(&pred); return ORC_E_OOM; }
    uint64_t sp = 0;
    /* network.cpp:234-239 -- seed with the declared outputs. */
    for (uint32_t k = 0; k < n_out; ++k) {
        const int64_t i = node_index(nodes, n_nodes, outputs[k]);
        if (i >= 0 && !required[i]) {
            required[i] = 1;
            stack[sp++] = (uint32_t)i;
        }
    }
    /* network.cpp:240-249 -- LIFO worklist over predecessors. */
    while (sp) {
        const uint32_t node = stack[--sp];
        for (uint64_t k = pred.off[node]; k < pred.off[node + 1]; ++k) {
            const uint32_t p = pred.adj[k];
            if (!required[p]) {
                required[p] = 1;
                stack[sp++] = p;
            }
        }
    }
    free(stack);
    free_csr(&pred);
    return ORC_OK;
}

/* ---- segment: segmentation.cpp:20-101 ------------------------------------
 * Round-based layering, restated round for round (NOT as Kahn, so it is an
 * independent check of the device's Kahn pass).  level[n_nodes] receives the
 * layer of every node index, ORC_UNASSIGNED for the rest.  Returns the number
 * of layers including layer 0 (>= 1), or a negative error code.
 * Layer 0 is the set of declared inputs that are known nodes (ids missing
 * from `nodes` are rejected by validate(), network.cpp:166-168). */
int64_t orc_segment(uint32_t n_nodes, const uint32_t* nodes, uint32_t n_in, const uint32_t* inputs,
                    uint64_t n_edges, const uint32_t* src, const uint32_t* dst,
                    const uint8_t* required, uint32_t* level) {
    csr_t pred, succ;
    if (build_csr(n_nodes, nodes, n_edges, src, dst, 1, &pred)) return -ORC_E_OOM;
    if (build_csr(n_nodes, nodes, n_edges, src, dst, 0, &succ)) {
        free_csr(&pred);
        return -ORC_E_OOM;
    }
    uint8_t* in_s = (uint8_t*)calloc((size_t)n_nodes + 1, 1);
    uint8_t* is_candidate = (uint8_t*)calloc((size_t)n_nodes + 1, 1);
    uint32_t* frontier = (uint32_t*)malloc(((size_t)n_nodes + 1) * sizeof(uint32_t));
    uint32_t* promoted = (uint32_t*)malloc(((size_t)n_nodes + 1) * sizeof(uint32_t));
    if (!in_s || !is_candidate || !frontier || !promoted) {
        free(in_s); free(is_candidate); free(frontier); free(promoted);
        free_csr(&pred); free_csr(&succ);
        return -ORC_E_OOM;
    }
    for (uint32_t i = 0; i < n_nodes; ++i) level[i] = ORC_UNASSIGNED;

    /* segmentation.cpp:41-47 -- layer 0 = sorted unique inputs. */
    for (uint32_t k = 0; k < n_in; ++k) {
        const int64_t i = node_index(nodes, n_nodes, inputs[k]);
        if (i >= 0) { in_s[i] = 1; level[i] = 0; }
    }
    /* segmentation.cpp:50-52 -- first frontier in index order. */
    uint64_t nf = 0;
    for (uint32_t i = 0; i < n_nodes; ++i)
        if (in_s[i]) frontier[nf++] = i;

    uint32_t layer = 0;
    for (;;) {
        /* segmentation.cpp:60-62 -- successors of the last frontier. */
        for (uint64_t f = 0; f < nf; ++f) {
            const uint32_t a = frontier[f];
            for (uint64_t k = succ.off[a]; k < succ.off[a + 1]; ++k)
                if (!in_s[succ.adj[k]]) is_candidate[succ.adj[k]] = 1;
        }
        /* segmentation.cpp:65-76 -- required candidates whose predecessors
         * are all in s (full O(N) scan, as in the reference). */
        uint64_t np = 0;
        for (uint32_t b = 0; b < n_nodes; ++b) {
            if (!is_candidate[b] || !required[b]) continue;
            int all_in = 1;
            for (uint64_t k = pred.off[b]; k < pred.off[b + 1]; ++k)
                if (!in_s[pred.adj[k]]) { all_in = 0; break; }
            if (all_in) promoted[np++] = b;
        }
        if (np == 0) break; /* segmentation.cpp:78 */
        ++layer;
        /* segmentation.cpp:80-90 -- commit the round. */
        for (uint64_t k = 0; k < np; ++k) {
            in_s[promoted[k]] = 1;
            is_candidate[promoted[k]] = 0;
            level[promoted[k]] = layer;
        }
        memcpy(frontier, promoted, np * sizeof(uint32_t));
        nf = np;
    }
    free(in_s); free(is_candidate); free(frontier); free(promoted);
    free_csr(&pred); free_csr(&succ);
    return (int64_t)layer + 1;
}

/* ---- flatten: layout.cpp:12-83 -------------------------------------------
 * Caller-allocated outputs (upper bounds in brackets):
 *   layer_offsets [n_layers+1], node_ids [n_nodes] in (layer, id) order,
 *   row_ptr [n_nodes+1], in_nodes [n_edges] (predecessor ids),
 *   in_weights [n_edges].
 * Scalars: *n_assigned, *dropped (edges into unassigned targets),
 * *id_bound (max id + 1).  Returns ORC_E_UNASSIGNED_OUTPUT when an output has
 * no layer (layout.cpp:13-17). */
int orc_flatten(uint32_t n_nodes, const uint32_t* nodes, uint32_t n_out, const uint32_t* outputs,
                uint64_t n_edges, const uint32_t* src, const uint32_t* dst, const float* w,
                const uint32_t* level, uint32_t n_layers, uint32_t* layer_offsets,
                uint32_t* node_ids, uint64_t* row_ptr, uint32_t* in_nodes, float* in_weights,
                uint32_t* n_assigned, uint64_t* dropped, uint32_t* id_bound) {
    /* layout.cpp:13-17 -- every output must have a layer. */
    for (uint32_t k = 0; k < n_out; ++k) {
        const int64_t i = node_index(nodes, n_nodes, outputs[k]);
        if (i < 0 || level[i] == ORC_UNASSIGNED) return ORC_E_UNASSIGNED_OUTPUT;
    }
    /* layout.cpp:24-26 -- value arrays span max id + 1. */
    *id_bound = n_nodes ? nodes[n_nodes - 1] + 1 : 0;

    /* layout.cpp:28-50 -- positions in (layer, id) order: a stable counting
     * sort by layer over the id-sorted node array. */
    memset(layer_offsets, 0, ((size_t)n_layers + 1) * sizeof(uint32_t));
    for (uint32_t i = 0; i < n_nodes; ++i)
        if (level[i] != ORC_UNASSIGNED) layer_offsets[level[i] + 1]++;
    for (uint32_t l = 0; l < n_layers; ++l) layer_offsets[l + 1] += layer_offsets[l];
    *n_assigned = layer_offsets[n_layers];
    uint32_t* cursor = (uint32_t*)malloc(((size_t)n_layers + 1) * sizeof(uint32_t));
    uint32_t* position = (uint32_t*)malloc(((size_t)n_nodes + 1) * sizeof(uint32_t));
    if (!cursor || !position) { free(cursor); free(position); return ORC_E_OOM; }
    memcpy(cursor, layer_offsets, ((size_t)n_layers + 1) * sizeof(uint32_t));
    for (uint32_t i = 0; i < n_nodes; ++i) {
        position[i] = ORC_UNASSIGNED;
        if (level[i] != ORC_UNASSIGNED) {
            position[i] = cursor[level[i]]++;
            node_ids[position[i]] = nodes[i];
        }
    }
    free(cursor);

    /* layout.cpp:52-62 -- scatter connections into their target's row in
     * connection order; edges into unassigned targets are dropped. */
    const uint32_t na = *n_assigned;
    memset(row_ptr, 0, ((size_t)na + 1) * sizeof(uint64_t));
    int64_t* tpos = (int64_t*)malloc((n_edges ? n_edges : 1) * sizeof(int64_t));
    if (!tpos) { free(position); return ORC_E_OOM; }
    uint64_t drop = 0;
    for (uint64_t e = 0; e < n_edges; ++e) {
        const int64_t t = node_index(nodes, n_nodes, dst[e]);
        tpos[e] = (t >= 0 && level[t] != ORC_UNASSIGNED) ? (int64_t)position[t] : -1;
        if (tpos[e] < 0) ++drop;
        else row_ptr[tpos[e] + 1]++;
    }
    *dropped = drop;
    for (uint32_t p = 0; p < na; ++p) row_ptr[p + 1] += row_ptr[p];
    uint64_t* fill = (uint64_t*)malloc(((size_t)na + 1) * sizeof(uint64_t));
    if (!fill) { free(tpos); free(position); return ORC_E_OOM; }
    memcpy(fill, row_ptr, ((size_t)na + 1) * sizeof(uint64_t));
    for (uint64_t e = 0; e < n_edges; ++e) {
        if (tpos[e] < 0) continue;
        const uint64_t k = fill[tpos[e]]++;
        in_nodes[k] = src[e];
        in_weights[k] = w[e];
    }
    free(fill); free(tpos); free(position);

    /* layout.cpp:64-80 -- predecessors sorted ascending by source id.  The
     * reference uses std::sort on an index permutation; ids within a row are
     * distinct for validated networks (no duplicate connections,
     * network.cpp:200-205), so the order is unique.  Insertion sort keeps
     * equal ids in connection order for unvalidated input. */
    for (uint32_t p = 0; p < na; ++p) {
        const uint64_t b = row_ptr[p], e = row_ptr[p + 1];
        for (uint64_t i = b + 1; i < e; ++i) {
            const uint32_t id = in_nodes[i];
            const float wt = in_weights[i];
            uint64_t j = i;
            while (j > b && in_nodes[j - 1] > id) {
                in_nodes[j] = in_nodes[j - 1];
                in_weights[j] = in_weights[j - 1];
                --j;
            }
            in_nodes[j] = id;
            in_weights[j] = wt;
        }
    }
    return ORC_OK;
}

/* ---- eval_sequential: eval.cpp:16-47 ---------------------------------------
 * One input vector x[n_x].  state_inputs / state_outputs are id-indexed arrays
 * of id_bound floats (ActivationState, eval.hpp:14-17); unassigned ids stay
 * 0.0f (eval.cpp:30-31).  Node p is a sensor iff p < layer_offsets[1]. */
int orc_eval_sequential(uint32_t node_count, const uint32_t* node_ids, uint32_t n_sensors,
                        const uint64_t* row_ptr, const uint32_t* in_nodes,
                        const float* in_weights, uint32_t n_in, const uint32_t* input_order,
                        uint32_t id_bound, const float* x, uint32_t n_x, float* state_inputs,
                        float* state_outputs) {
    /* eval.cpp:26-28 -- arity check. */
    if (n_x != n_in) return ORC_E_ARITY;
    /* eval.cpp:29-33 -- zeroed id-indexed state, inputs scattered by the
     * declared input order (later duplicates win, as with the reference's
     * sequential assignment). */
    memset(state_inputs, 0, (size_t)id_bound * sizeof(float));
    memset(state_outputs, 0, (size_t)id_bound * sizeof(float));
    for (uint32_t i = 0; i < n_x; ++i) state_inputs[input_order[i]] = x[i];
    /* eval.cpp:43-45 -- every node in (layer, id) order. */
    for (uint32_t p = 0; p < node_count; ++p) {
        const uint32_t id = node_ids[p];
        if (p < n_sensors) {
            /* eval.cpp:17 -- sensors are sigmoided, not passed through. */
            state_outputs[id] = orc_sigmoid32(state_inputs[id]);
            continue;
        }
        /* eval.cpp:18-22 -- fp32 multiply, fp32 add, stored order. */
        float sum = 0.0f;
        for (uint64_t k = row_ptr[p]; k < row_ptr[p + 1]; ++k)
            sum += in_weights[k] * state_outputs[in_nodes[k]];
        state_outputs[id] = orc_sigmoid32(sum);
    }
    return ORC_OK;
}

/* Self-consistency check at any size (test_eval.cpp:109-134): recompute the
 * nodes at the given flat positions from a finished id-indexed op array of
 * one vector and return the values (sensors from `x`).  The caller compares
 * them bitwise with op[node_ids[pos]]. */
void orc_recompute(uint32_t n_sensors, const uint32_t* node_ids, const uint64_t* row_ptr,
                   const uint32_t* in_nodes, const float* in_weights, const uint32_t* input_order,
                   uint32_t n_in, const float* x, const float* op, const uint32_t* positions,
                   uint64_t n_pos, float* out) {
    for (uint64_t i = 0; i < n_pos; ++i) {
        const uint32_t p = positions[i];
        if (p < n_sensors) {
            float xv = 0.0f;
            for (uint32_t k = 0; k < n_in; ++k)
                if (input_order[k] == node_ids[p]) xv = x[k];
            out[i] = orc_sigmoid32(xv);
            continue;
        }
        float sum = 0.0f;
        for (uint64_t k = row_ptr[p]; k < row_ptr[p + 1]; ++k)
            sum += in_weights[k] * op[in_nodes[k]];
        out[i] = orc_sigmoid32(sum);
    }
}

/* Batch convenience for tests: X is [n_vec][n_in] row-major, OP is
 * [n_vec][id_bound]. */
int orc_eval_sequential_batch(uint32_t node_count, const uint32_t* node_ids, uint32_t n_sensors,
                              const uint64_t* row_ptr, const uint32_t* in_nodes,
                              const float* in_weights, uint32_t n_in, const uint32_t* input_order,
                              uint32_t id_bound, const float* X, uint32_t n_x, uint32_t n_vec,
                              float* OP) {
    float* scratch = (float*)malloc(((size_t)id_bound + 1) * sizeof(float));
    if (!scratch) return ORC_E_OOM;
    for (uint32_t v = 0; v < n_vec; ++v) {
        const int rc = orc_eval_sequential(node_count, node_ids, n_sensors, row_ptr, in_nodes,
                                           in_weights, n_in, input_order, id_bound,
                                           X + (size_t)v * n_x, n_x, scratch,
                                           OP + (size_t)v * id_bound);
        if (rc) { free(scratch); return rc; }
    }
    free(scratch);
    return ORC_OK;
}
