// preprocess.cu -- the reference's dependency-group preprocessing on the GPU.
//
//   compute_required (network.cpp:222-255)  -> k_bfs_required: reverse-frontier
//        BFS over the incoming-edge CSR, one cooperative kernel, grid-wide
//        barrier per frontier round, warp-aggregated frontier appends;
//   segment (segmentation.cpp:20-101)       -> k_kahn: Kahn levelling with
//        in-degree atomics (atomicSub on the remaining-predecessor count), the
//        frontier of round r is exactly layer r; bit-exact with the reference's
//        round-based promotion (proof sketch in DESIGN.md "levels");
//   flatten (layout.cpp:12-83)              -> stable radix sorts: node indices
//        by (network, level) give the (layer, id) positions; kept edges sorted
//        by source id then stably by target position give every row in
//        ascending source-id order; row_ptr by scan.
//
// Populations are one block-diagonal network: ids are offset per network so
// a single pass levels all of them; positions are network-major.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"
#include "sort.cuh"

namespace cg = cooperative_groups;
using namespace asnn_b200;

#define CK(expr)                                                 \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return cuda_fail(dev, _e, #expr); \
    } while (0)
#define RC(expr)           \
    do {                   \
        int _r = (expr);   \
        if (_r) return _r; \
    } while (0)

namespace {

constexpr uint32_t kT = 256;
constexpr uint32_t kUn = 0xFFFFFFFFu;

inline uint32_t nblk(uint64_t n, uint32_t t = kT) { return static_cast<uint32_t>((n + t - 1) / t); }

inline int bits_for(uint64_t v) {  // bits needed to represent values 0..v
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

__device__ __forceinline__ uint32_t seg_of(const uint32_t* __restrict__ prefix, uint32_t n, uint32_t v) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (prefix[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t index_of(const uint32_t* __restrict__ nodes, uint32_t n, uint32_t id,
                                             bool dense) {
    if (dense) return id < n ? id : kUn;
    uint32_t lo = 0, hi = n;  // node_index, network.cpp:57-61
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (nodes[mid] < id) lo = mid + 1;
        else hi = mid;
    }
    return (lo < n && nodes[lo] == id) ? lo : kUn;
}

// ---- id -> node index ----------------------------------------------------------
// si/ti: indices of the endpoints (kUn if unknown).  adj_ok marks edges that
// enter the pred/succ lists: both endpoints known and not a self-loop
// (network.cpp:226-228, segmentation.cpp:26-31).
__global__ void k_map_edges(const uint32_t* __restrict__ nodes, uint32_t N, bool dense,
                            const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                            uint64_t E, uint32_t* __restrict__ si, uint32_t* __restrict__ ti,
                            uint32_t* __restrict__ indeg, uint32_t* __restrict__ outdeg) {
    const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const uint32_t s = index_of(nodes, N, src[e], dense);
    const uint32_t t = index_of(nodes, N, dst[e], dense);
    si[e] = s;
    ti[e] = t;
    if (s != kUn && t != kUn && src[e] != dst[e]) {
        atomicAdd(&indeg[t], 1u);
        atomicAdd(&outdeg[s], 1u);
    }
}

__global__ void k_fill_adj(const uint32_t* __restrict__ si, const uint32_t* __restrict__ ti,
                           const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t E,
                           uint32_t* __restrict__ pred_cur, uint32_t* __restrict__ pred_adj,
                           uint32_t* __restrict__ succ_cur, uint32_t* __restrict__ succ_adj) {
    const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const uint32_t s = si[e], t = ti[e];
    if (s == kUn || t == kUn || src[e] == dst[e]) return;
    pred_adj[atomicAdd(&pred_cur[t], 1u)] = s;
    succ_adj[atomicAdd(&succ_cur[s], 1u)] = t;
}

// Warp-aggregated append of `v` (when `want`) to queue q with counter *cnt.
__device__ __forceinline__ void warp_append(bool want, uint32_t v, uint32_t* __restrict__ q,
                                            uint32_t* cnt) {
    const unsigned m = __ballot_sync(__activemask(), want);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cnt, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(__activemask(), base, leader);
    if (want) q[base + __popc(m & ((1u << lane) - 1u))] = v;
}

__device__ __forceinline__ uint32_t vload(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// compute_required: frontier rounds of backward reachability.  req[] holds
// 1 for members; q0 holds the seeds (outputs), cnt[0] their count.
__global__ void k_bfs_required(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                               uint32_t* __restrict__ req, uint32_t* __restrict__ q0,
                               uint32_t* __restrict__ q1, uint32_t* __restrict__ cnt) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t* cur = q0;
    uint32_t* nxt = q1;
    int par = 0;
    for (;;) {
        const uint32_t n = vload(&cnt[par]);
        for (uint32_t i = gw; i < n; i += nw) {
            const uint32_t v = cur[i];
            const uint32_t b = off[v], e = off[v + 1];
            for (uint32_t k0 = b; k0 < e; k0 += 32) {
                const uint32_t k = k0 + lane;
                bool add = false;
                uint32_t p = 0;
                if (k < e) {
                    p = adj[k];
                    add = atomicExch(&req[p], 1u) == 0u;
                }
                warp_append(add, p, nxt, &cnt[par ^ 1]);
            }
        }
        grid.sync();
        if (vload(&cnt[par ^ 1]) == 0) break;
        if (blockIdx.x == 0 && threadIdx.x == 0) cnt[par] = 0;
        grid.sync();
        uint32_t* t = cur;
        cur = nxt;
        nxt = t;
        par ^= 1;
    }
}

// segment: Kahn rounds.  level[] = 0 for inputs, kUn otherwise; rem[] = the
// in-degree over adjacency edges; req[] the required flags.  Round r
// processes the nodes levelled r-1 and promotes required successors whose
// last predecessor just got a level.  cnt[2] receives the number of layers.
__global__ void k_kahn(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                       uint32_t* __restrict__ rem, const uint32_t* __restrict__ req,
                       uint32_t* __restrict__ level, uint32_t* __restrict__ q0, uint32_t* __restrict__ q1,
                       uint32_t* __restrict__ cnt) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t* cur = q0;
    uint32_t* nxt = q1;
    int par = 0;
    uint32_t round = 1;
    for (;;) {
        const uint32_t n = vload(&cnt[par]);
        for (uint32_t i = gw; i < n; i += nw) {
            const uint32_t a = cur[i];
            const uint32_t b0 = off[a], e = off[a + 1];
            for (uint32_t k0 = b0; k0 < e; k0 += 32) {
                const uint32_t k = k0 + lane;
                bool add = false;
                uint32_t b = 0;
                if (k < e) {
                    b = adj[k];
                    // inputs are in s from the start and never promoted again
                    if (level[b] != 0u) {
                        const uint32_t left = atomicSub(&rem[b], 1u);
                        if (left == 1u && req[b]) {
                            level[b] = round;
                            add = true;
                        }
                    }
                }
                warp_append(add, b, nxt, &cnt[par ^ 1]);
            }
        }
        grid.sync();
        if (vload(&cnt[par ^ 1]) == 0) {
            if (blockIdx.x == 0 && threadIdx.x == 0) cnt[2] = round;  // layers incl. layer 0
            break;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) cnt[par] = 0;
        grid.sync();
        uint32_t* t = cur;
        cur = nxt;
        nxt = t;
        par ^= 1;
        ++round;
    }
}

// Seeds: declared outputs (BFS) or inputs (Kahn), deduplicated through the
// flag array.  For Kahn the flag is level[] (0 = input).
__global__ void k_seed_outputs(const uint32_t* __restrict__ nodes, uint32_t N, bool dense,
                               const uint32_t* __restrict__ outs, uint32_t n_out, uint32_t* __restrict__ req,
                               uint32_t* __restrict__ q, uint32_t* __restrict__ cnt) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_out) return;
    const uint32_t i = index_of(nodes, N, outs[j], dense);
    if (i != kUn && atomicExch(&req[i], 1u) == 0u) q[atomicAdd(cnt, 1u)] = i;
}

__global__ void k_seed_inputs(const uint32_t* __restrict__ nodes, uint32_t N, bool dense,
                              const uint32_t* __restrict__ ins, uint32_t n_in, uint32_t* __restrict__ level,
                              uint32_t* __restrict__ q, uint32_t* __restrict__ cnt) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_in) return;
    const uint32_t i = index_of(nodes, N, ins[j], dense);
    if (i != kUn && atomicCAS(&level[i], kUn, 0u) == kUn) q[atomicAdd(cnt, 1u)] = i;
}

// ---- flatten helpers -----------------------------------------------------------------
// Assigned node indices with their (network, level) sort key.
__global__ void k_pos_keys(const uint32_t* __restrict__ level, const uint32_t* __restrict__ nodes,
                           uint32_t N, const uint32_t* __restrict__ idb_prefix, uint32_t G, int lvl_bits,
                           uint32_t* __restrict__ flag) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) flag[i] = level[i] != kUn ? 1u : 0u;
}

__global__ void k_pos_compact(const uint32_t* __restrict__ level, const uint32_t* __restrict__ nodes,
                              uint32_t N, const uint32_t* __restrict__ idb_prefix, uint32_t G,
                              int lvl_bits, const uint32_t* __restrict__ slot, uint32_t* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N || level[i] == kUn) return;
    const uint32_t g = G > 1 ? seg_of(idb_prefix, G, nodes[i]) : 0u;
    keys[slot[i]] = (g << lvl_bits) | level[i];
    vals[slot[i]] = i;
}

// Position p holds node index order[p]: record pos_of[index], the node id
// local to its network, and count (network, level) cells.
__global__ void k_positions(const uint32_t* __restrict__ order, uint32_t P, const uint32_t* __restrict__ nodes,
                            const uint32_t* __restrict__ level, const uint32_t* __restrict__ idb_prefix,
                            uint32_t G, uint32_t L, uint32_t* __restrict__ pos_of,
                            uint32_t* __restrict__ local_ids, uint32_t* __restrict__ cells) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const uint32_t i = order[p];
    const uint32_t id = nodes[i];
    const uint32_t g = G > 1 ? seg_of(idb_prefix, G, id) : 0u;
    pos_of[i] = p;
    local_ids[p] = id - idb_prefix[g];
    atomicAdd(&cells[static_cast<uint64_t>(g) * L + level[i]], 1u);
}

// Kept edges: target known and levelled (layout.cpp:54-58).  tpos[e] is the
// target position or kUn; dropped counted per network.
__global__ void k_edge_targets(const uint32_t* __restrict__ ti, const uint32_t* __restrict__ dst, uint64_t E,
                               const uint32_t* __restrict__ pos_of, const uint32_t* __restrict__ level,
                               const uint32_t* __restrict__ idb_prefix, uint32_t G,
                               uint32_t* __restrict__ tpos, uint32_t* __restrict__ keep,
                               unsigned long long* __restrict__ dropped) {
    const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const uint32_t t = ti[e];
    const bool ok = t != kUn && level[t] != kUn;
    tpos[e] = ok ? pos_of[t] : kUn;
    keep[e] = ok ? 1u : 0u;
    if (!ok) {
        const uint32_t g = G > 1 ? seg_of(idb_prefix, G, dst[e]) : 0u;
        atomicAdd(&dropped[g], 1ull);
    }
}

__global__ void k_edge_compact(const uint32_t* __restrict__ keep, const uint32_t* __restrict__ slot,
                               const uint32_t* __restrict__ src, uint64_t E, uint32_t* __restrict__ keys,
                               uint32_t* __restrict__ vals) {
    const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= E || !keep[e]) return;
    keys[slot[e]] = src[e];
    vals[slot[e]] = static_cast<uint32_t>(e);
}

__global__ void k_gather_keys(const uint32_t* __restrict__ idx, uint64_t n, const uint32_t* __restrict__ from,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ rowcnt) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t t = from[idx[k]];
    keys[k] = t;
    atomicAdd(&rowcnt[t], 1u);
}

__global__ void k_emit_edges(const uint32_t* __restrict__ idx, uint64_t n, const uint32_t* __restrict__ src,
                             const float* __restrict__ w, const uint32_t* __restrict__ idb_prefix, uint32_t G,
                             uint32_t* __restrict__ in_ids, float* __restrict__ w_out) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t e = idx[k];
    const uint32_t s = src[e];
    const uint32_t g = G > 1 ? seg_of(idb_prefix, G, s) : 0u;
    in_ids[k] = s - idb_prefix[g];
    w_out[k] = w[e];
}

__global__ void k_local_ids(const uint32_t* __restrict__ in, uint32_t n, const uint32_t* __restrict__ prefix,
                            const uint32_t* __restrict__ idb_prefix, uint32_t G, uint32_t* __restrict__ out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t g = G > 1 ? seg_of(prefix, G, j) : 0u;
    out[j] = in[j] - idb_prefix[g];
}

// --------------------------------------------------------------------------------------
// One (possibly combined) network resident on the device.
struct DevNet {
    uint32_t G = 1;
    uint32_t N = 0;
    uint64_t E = 0;
    uint32_t n_in = 0, n_out = 0;
    bool dense = false;
    std::vector<uint32_t> h_idb, h_in_prefix, h_out_prefix, h_node_prefix;  // [G+1]
    std::vector<uint32_t> h_idbound;                                       // [G]
    std::vector<std::vector<uint32_t>> h_inputs, h_outputs;                // per net, local ids
    DevBuf<uint32_t> nodes, src, dst, inputs, outputs, idb_prefix, in_prefix, out_prefix;
    DevBuf<float> w;
    // derived
    DevBuf<uint32_t> si, ti, pred_off, pred_adj, succ_off, succ_adj, req, level;
    uint32_t n_layers = 0;
};

// Host marshalling: G networks -> one id space (ids offset by the running
// id_bound), arrays concatenated, copied to the device.
int upload_networks(asnn_dev* dev, uint32_t G, const asnn_network_desc* nets, DevNet& d) {
    d.G = G;
    d.h_idb.assign(G + 1, 0);
    d.h_in_prefix.assign(G + 1, 0);
    d.h_out_prefix.assign(G + 1, 0);
    d.h_node_prefix.assign(G + 1, 0);
    d.h_idbound.assign(G, 0);
    d.h_inputs.resize(G);
    d.h_outputs.resize(G);
    uint64_t E = 0, N = 0, idb = 0;
    for (uint32_t g = 0; g < G; ++g) {
        const asnn_network_desc& n = nets[g];
        if ((n.n_nodes && !n.nodes) || (n.n_connections && (!n.source || !n.target || !n.weight)) ||
            (n.n_inputs && !n.inputs) || (n.n_outputs && !n.outputs))
            return fail(dev, ASNN_E_INVALID, "null network array");
        for (uint32_t i = 1; i < n.n_nodes; ++i)
            if (n.nodes[i] <= n.nodes[i - 1])
                return fail(dev, ASNN_E_INVALID, "Network.nodes must be sorted ascending and unique");
        const uint32_t bound = n.n_nodes ? n.nodes[n.n_nodes - 1] + 1 : 0;  // layout.cpp:24-26
        d.h_idbound[g] = bound;
        d.h_idb[g + 1] = static_cast<uint32_t>(idb + bound);
        d.h_in_prefix[g + 1] = d.h_in_prefix[g] + n.n_inputs;
        d.h_out_prefix[g + 1] = d.h_out_prefix[g] + n.n_outputs;
        d.h_node_prefix[g + 1] = static_cast<uint32_t>(N + n.n_nodes);
        d.h_inputs[g].assign(n.inputs, n.inputs + n.n_inputs);
        d.h_outputs[g].assign(n.outputs, n.outputs + n.n_outputs);
        E += n.n_connections;
        N += n.n_nodes;
        idb += bound;
        if (idb >= kUn || N >= kUn) return fail(dev, ASNN_E_INVALID, "id space exceeds 2^32-1");
    }
    if (E >= kUn) return fail(dev, ASNN_E_INVALID, "more than 2^32-1 connections");
    d.N = static_cast<uint32_t>(N);
    d.E = E;
    d.n_in = d.h_in_prefix[G];
    d.n_out = d.h_out_prefix[G];
    cudaStream_t st = dev->stream;
    CK(d.nodes.alloc(N));
    CK(d.src.alloc(E));
    CK(d.dst.alloc(E));
    CK(d.w.alloc(E));
    CK(d.inputs.alloc(d.n_in));
    CK(d.outputs.alloc(d.n_out));
    CK(d.idb_prefix.alloc(G + 1));
    CK(d.in_prefix.alloc(G + 1));
    CK(d.out_prefix.alloc(G + 1));
    if (G == 1) {
        const asnn_network_desc& n = nets[0];
        if (N) CK(cudaMemcpyAsync(d.nodes.p, n.nodes, N * 4, cudaMemcpyHostToDevice, st));
        if (E) {
            CK(upload_host(dev, d.src.p, n.source, E * 4, st));
            CK(upload_host(dev, d.dst.p, n.target, E * 4, st));
            CK(upload_host(dev, d.w.p, n.weight, E * 4, st));
        }
        if (d.n_in) CK(cudaMemcpyAsync(d.inputs.p, n.inputs, d.n_in * 4ull, cudaMemcpyHostToDevice, st));
        if (d.n_out) CK(cudaMemcpyAsync(d.outputs.p, n.outputs, d.n_out * 4ull, cudaMemcpyHostToDevice, st));
        d.dense = N == 0 || n.nodes[N - 1] == N - 1;
    } else {
        std::vector<uint32_t> nodes(N), src(E), dst(E), ins(d.n_in), outs(d.n_out);
        std::vector<float> w(E);
        uint64_t e0 = 0;
        bool dense = true;
        for (uint32_t g = 0; g < G; ++g) {
            const asnn_network_desc& n = nets[g];
            const uint32_t off = d.h_idb[g];
            for (uint32_t i = 0; i < n.n_nodes; ++i) nodes[d.h_node_prefix[g] + i] = n.nodes[i] + off;
            dense = dense && (n.n_nodes == 0 || n.nodes[n.n_nodes - 1] == n.n_nodes - 1);
            for (uint64_t e = 0; e < n.n_connections; ++e) {
                src[e0 + e] = n.source[e] + off;
                dst[e0 + e] = n.target[e] + off;
            }
            std::memcpy(&w[e0], n.weight, n.n_connections * 4);
            e0 += n.n_connections;
            for (uint32_t i = 0; i < n.n_inputs; ++i) ins[d.h_in_prefix[g] + i] = n.inputs[i] + off;
            for (uint32_t i = 0; i < n.n_outputs; ++i) outs[d.h_out_prefix[g] + i] = n.outputs[i] + off;
        }
        d.dense = dense;
        if (N) CK(cudaMemcpyAsync(d.nodes.p, nodes.data(), N * 4, cudaMemcpyHostToDevice, st));
        if (E) {
            CK(cudaMemcpyAsync(d.src.p, src.data(), E * 4, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(d.dst.p, dst.data(), E * 4, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(d.w.p, w.data(), E * 4, cudaMemcpyHostToDevice, st));
        }
        if (d.n_in) CK(cudaMemcpyAsync(d.inputs.p, ins.data(), d.n_in * 4ull, cudaMemcpyHostToDevice, st));
        if (d.n_out) CK(cudaMemcpyAsync(d.outputs.p, outs.data(), d.n_out * 4ull, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));  // host staging vectors go out of scope
    }
    CK(cudaMemcpyAsync(d.idb_prefix.p, d.h_idb.data(), (G + 1) * 4ull, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d.in_prefix.p, d.h_in_prefix.data(), (G + 1) * 4ull, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d.out_prefix.p, d.h_out_prefix.data(), (G + 1) * 4ull, cudaMemcpyHostToDevice, st));
    return ASNN_OK;
}

// Endpoint indices + predecessor / successor CSR.
int build_adjacency(asnn_dev* dev, DevNet& d) {
    cudaStream_t st = dev->stream;
    DevBuf<uint32_t> indeg, outdeg;
    CK(d.si.alloc(d.E));
    CK(d.ti.alloc(d.E));
    CK(indeg.alloc(d.N + 1));
    CK(outdeg.alloc(d.N + 1));
    CK(cudaMemsetAsync(indeg.p, 0, (d.N + 1) * 4ull, st));
    CK(cudaMemsetAsync(outdeg.p, 0, (d.N + 1) * 4ull, st));
    if (d.E)
        k_map_edges<<<nblk(d.E), kT, 0, st>>>(d.nodes.p, d.N, d.dense, d.src.p, d.dst.p, d.E, d.si.p,
                                              d.ti.p, indeg.p, outdeg.p);
    CK(cudaGetLastError());
    CK(d.pred_off.alloc(d.N + 1));
    CK(d.succ_off.alloc(d.N + 1));
    uint32_t* d_tot = nullptr;
    DevBuf<uint32_t> tot;
    CK(tot.alloc(2));
    d_tot = tot.p;
    RC(exclusive_scan(dev, indeg.p, d.pred_off.p, d.N + 1, d_tot, st));
    RC(exclusive_scan(dev, outdeg.p, d.succ_off.p, d.N + 1, d_tot + 1, st));
    uint32_t h_tot[2];
    CK(cudaMemcpyAsync(h_tot, d_tot, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(d.pred_adj.alloc(h_tot[0]));
    CK(d.succ_adj.alloc(h_tot[1]));
    // reuse the degree arrays as fill cursors
    CK(cudaMemcpyAsync(indeg.p, d.pred_off.p, (d.N + 1) * 4ull, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(outdeg.p, d.succ_off.p, (d.N + 1) * 4ull, cudaMemcpyDeviceToDevice, st));
    if (d.E)
        k_fill_adj<<<nblk(d.E), kT, 0, st>>>(d.si.p, d.ti.p, d.src.p, d.dst.p, d.E, indeg.p, d.pred_adj.p,
                                             outdeg.p, d.succ_adj.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return ASNN_OK;
}

int coop_grid(asnn_dev* dev, const void* fn, uint32_t* blocks) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kT, 0));
    if (per_sm < 1) return fail(dev, ASNN_E_CUDA, "cooperative kernel does not fit");
    *blocks = static_cast<uint32_t>(per_sm) * static_cast<uint32_t>(dev->sm_count);
    return ASNN_OK;
}

int run_required(asnn_dev* dev, DevNet& d, const uint8_t* host_required) {
    cudaStream_t st = dev->stream;
    CK(d.req.alloc(d.N + 1));
    if (host_required) {
        std::vector<uint32_t> r(d.N);
        for (uint32_t i = 0; i < d.N; ++i) r[i] = host_required[i] ? 1u : 0u;
        CK(cudaMemcpyAsync(d.req.p, r.data(), d.N * 4ull, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        return ASNN_OK;
    }
    CK(cudaMemsetAsync(d.req.p, 0, (d.N + 1) * 4ull, st));
    DevBuf<uint32_t> q0, q1, cnt;
    CK(q0.alloc(d.N + 1));
    CK(q1.alloc(d.N + 1));
    CK(cnt.alloc(4));
    CK(cudaMemsetAsync(cnt.p, 0, 16, st));
    if (d.n_out)
        k_seed_outputs<<<nblk(d.n_out), kT, 0, st>>>(d.nodes.p, d.N, d.dense, d.outputs.p, d.n_out, d.req.p,
                                                     q0.p, cnt.p);
    uint32_t blocks = 0;
    RC(coop_grid(dev, reinterpret_cast<const void*>(k_bfs_required), &blocks));
    void* args[] = {&d.pred_off.p, &d.pred_adj.p, &d.req.p, &q0.p, &q1.p, &cnt.p};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_bfs_required), blocks, kT, args, 0, st));
    CK(cudaStreamSynchronize(st));
    return ASNN_OK;
}

__global__ void k_degree(const uint32_t* __restrict__ off, uint32_t N, uint32_t* __restrict__ deg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) deg[i] = off[i + 1] - off[i];
}

int run_segment(asnn_dev* dev, DevNet& d) {
    cudaStream_t st = dev->stream;
    DevBuf<uint32_t> rem, q0, q1, cnt;
    CK(d.level.alloc(d.N + 1));
    CK(cudaMemsetAsync(d.level.p, 0xFF, (d.N + 1) * 4ull, st));
    CK(rem.alloc(d.N + 1));
    if (d.N) k_degree<<<nblk(d.N), kT, 0, st>>>(d.pred_off.p, d.N, rem.p);
    CK(q0.alloc(d.N + 1));
    CK(q1.alloc(d.N + 1));
    CK(cnt.alloc(4));
    CK(cudaMemsetAsync(cnt.p, 0, 16, st));
    if (d.n_in)
        k_seed_inputs<<<nblk(d.n_in), kT, 0, st>>>(d.nodes.p, d.N, d.dense, d.inputs.p, d.n_in, d.level.p,
                                                   q0.p, cnt.p);
    CK(cudaGetLastError());
    uint32_t blocks = 0;
    RC(coop_grid(dev, reinterpret_cast<const void*>(k_kahn), &blocks));
    void* args[] = {&d.succ_off.p, &d.succ_adj.p, &rem.p, &d.req.p, &d.level.p, &q0.p, &q1.p, &cnt.p};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_kahn), blocks, kT, args, 0, st));
    uint32_t h[4];
    CK(cudaMemcpyAsync(h, cnt.p, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    d.n_layers = h[2];  // depth() = layers including layer 0 (segmentation.cpp:103-105)
    return ASNN_OK;
}

// Positions, per-network layer offsets, CSR of kept edges -> FlatDevice.
int run_flatten(asnn_dev* dev, DevNet& d, std::vector<NetMeta>& metas, FlatDevice& f) {
    cudaStream_t st = dev->stream;
    const uint32_t G = d.G, N = d.N;
    const uint32_t L = std::max<uint32_t>(d.n_layers, 1);
    const int lvl_bits = std::max(1, bits_for(L - 1));
    const int net_bits = G > 1 ? bits_for(G - 1) : 0;
    if (lvl_bits + net_bits > 32) return fail(dev, ASNN_E_INVALID, "too many networks x layers");

    // 1) positions: stable sort of assigned node indices by (network, level)
    DevBuf<uint32_t> flag, slot, keys, vals, tot;
    CK(flag.alloc(N + 1));
    CK(slot.alloc(N + 1));
    CK(tot.alloc(4));
    if (N) k_pos_keys<<<nblk(N), kT, 0, st>>>(d.level.p, d.nodes.p, N, d.idb_prefix.p, G, lvl_bits, flag.p);
    RC(exclusive_scan(dev, flag.p, slot.p, N, tot.p, st));
    uint32_t P = 0;
    CK(cudaMemcpyAsync(&P, tot.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(keys.alloc(P + 1));
    CK(vals.alloc(P + 1));
    if (N)
        k_pos_compact<<<nblk(N), kT, 0, st>>>(d.level.p, d.nodes.p, N, d.idb_prefix.p, G, lvl_bits, slot.p,
                                              keys.p, vals.p);
    CK(cudaGetLastError());
    SortBuffers sb;
    uint32_t *ks = nullptr, *order = nullptr;
    RC(radix_sort_pairs(dev, keys.p, vals.p, P, lvl_bits + net_bits, sb, &ks, &order, st));
    DevBuf<uint32_t> pos_of, cells;
    CK(pos_of.alloc(N + 1));
    CK(f.node_ids.alloc(P + 1));
    CK(cells.alloc(static_cast<size_t>(G) * L));
    CK(cudaMemsetAsync(cells.p, 0, static_cast<size_t>(G) * L * 4, st));
    if (P)
        k_positions<<<nblk(P), kT, 0, st>>>(order, P, d.nodes.p, d.level.p, d.idb_prefix.p, G, L, pos_of.p,
                                            f.node_ids.p, cells.p);
    CK(cudaGetLastError());
    std::vector<uint32_t> h_cells(static_cast<size_t>(G) * L);
    CK(cudaMemcpyAsync(h_cells.data(), cells.p, h_cells.size() * 4, cudaMemcpyDeviceToHost, st));

    // 2) kept edges (target levelled), sorted by source id, then stably by
    //    target position: rows in ascending source-id order (layout.cpp:64-80)
    const uint64_t E = d.E;
    DevBuf<uint32_t> tpos, keep, eslot;
    DevBuf<unsigned long long> dropped;
    CK(tpos.alloc(E + 1));
    CK(keep.alloc(E + 1));
    CK(eslot.alloc(E + 1));
    CK(dropped.alloc(G));
    CK(cudaMemsetAsync(dropped.p, 0, G * 8ull, st));
    if (E)
        k_edge_targets<<<nblk(E), kT, 0, st>>>(d.ti.p, d.dst.p, E, pos_of.p, d.level.p, d.idb_prefix.p, G,
                                               tpos.p, keep.p, dropped.p);
    RC(exclusive_scan(dev, keep.p, eslot.p, E, tot.p, st));
    uint32_t K = 0;
    CK(cudaMemcpyAsync(&K, tot.p, 4, cudaMemcpyDeviceToHost, st));
    std::vector<unsigned long long> h_dropped(G);
    CK(cudaMemcpyAsync(h_dropped.data(), dropped.p, G * 8ull, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    DevBuf<uint32_t> ekeys, evals;
    CK(ekeys.alloc(K + 1));
    CK(evals.alloc(K + 1));
    if (E) k_edge_compact<<<nblk(E), kT, 0, st>>>(keep.p, eslot.p, d.src.p, E, ekeys.p, evals.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    keep.reset();
    eslot.reset();
    SortBuffers eb;
    uint32_t *k1 = nullptr, *v1 = nullptr;
    const uint32_t max_id = d.h_idb[G] ? d.h_idb[G] - 1 : 0;
    RC(radix_sort_pairs(dev, ekeys.p, evals.p, K, std::max(1, bits_for(max_id)), eb, &k1, &v1, st));
    DevBuf<uint32_t> rowcnt;
    CK(rowcnt.alloc(P + 1));
    CK(cudaMemsetAsync(rowcnt.p, 0, (P + 1) * 4ull, st));
    // keys <- target position of each (source-sorted) edge
    uint32_t* kbuf = k1;  // source-sorted keys are no longer needed
    if (K) k_gather_keys<<<nblk(K), kT, 0, st>>>(v1, K, tpos.p, kbuf, rowcnt.p);
    CK(cudaGetLastError());
    uint32_t *k2 = nullptr, *v2 = nullptr;
    {
        // sort needs distinct alternates: use a fresh buffer set
        SortBuffers eb2;
        RC(radix_sort_pairs(dev, kbuf, v1, K, std::max(1, bits_for(P)), eb2, &k2, &v2, st));
        CK(f.row_ptr.alloc(P + 8));  // slack: K-cta bulk copies round up to 16 bytes
        RC(exclusive_scan(dev, rowcnt.p, f.row_ptr.p, P + 1, nullptr, st));
        CK(f.in_ids.alloc(K + 1));
        CK(f.w.alloc(K + 1));
        if (K)
            k_emit_edges<<<nblk(K), kT, 0, st>>>(v2, K, d.src.p, d.w.p, d.idb_prefix.p, G, f.in_ids.p, f.w.p);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
    }
    // declared inputs / outputs, local ids per network
    CK(f.inputs.alloc(d.n_in + 1));
    CK(f.outputs.alloc(d.n_out + 1));
    if (d.n_in)
        k_local_ids<<<nblk(d.n_in), kT, 0, st>>>(d.inputs.p, d.n_in, d.in_prefix.p, d.idb_prefix.p, G,
                                                 f.inputs.p);
    if (d.n_out)
        k_local_ids<<<nblk(d.n_out), kT, 0, st>>>(d.outputs.p, d.n_out, d.out_prefix.p, d.idb_prefix.p, G,
                                                  f.outputs.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));

    // 3) per-network metadata
    metas.assign(G, NetMeta());
    uint64_t ebase = 0;
    std::vector<uint32_t> h_row(1, 0);
    for (uint32_t g = 0; g < G; ++g) {
        NetMeta& m = metas[g];
        uint32_t nl = 1;
        for (uint32_t l = 0; l < L; ++l)
            if (h_cells[static_cast<size_t>(g) * L + l]) nl = l + 1;
        m.n_layers = nl;
        m.layer_offsets.assign(nl + 1, 0);
        for (uint32_t l = 0; l < nl; ++l)
            m.layer_offsets[l + 1] = m.layer_offsets[l] + h_cells[static_cast<size_t>(g) * L + l];
        m.n_pos = m.layer_offsets[nl];
        m.n_sensors = m.layer_offsets[1];
        m.id_bound = d.h_idbound[g];
        m.n_in = d.h_in_prefix[g + 1] - d.h_in_prefix[g];
        m.n_out = d.h_out_prefix[g + 1] - d.h_out_prefix[g];
        m.inputs = d.h_inputs[g];
        m.outputs = d.h_outputs[g];
        m.dropped = h_dropped[g];
        (void)ebase;
    }
    // edges per network from row_ptr at network boundaries
    {
        std::vector<uint32_t> h_rp(P + 1);
        CK(cudaMemcpyAsync(h_rp.data(), f.row_ptr.p, (P + 1) * 4ull, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        uint32_t pb = 0;
        for (uint32_t g = 0; g < G; ++g) {
            metas[g].n_edges = h_rp[pb + metas[g].n_pos] - h_rp[pb];
            pb += metas[g].n_pos;
        }
    }
    return ASNN_OK;
}

// layout.cpp:13-17: outputs of every network must be levelled.  missing[]
// receives the declared-output slots without a layer.
__global__ void k_check_outputs(const uint32_t* __restrict__ nodes, uint32_t N, bool dense,
                                const uint32_t* __restrict__ outs, uint32_t n_out,
                                const uint32_t* __restrict__ level, uint32_t* __restrict__ missing,
                                uint32_t* __restrict__ n_missing) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_out) return;
    const uint32_t i = index_of(nodes, N, outs[j], dense);
    if (i == kUn || level[i] == kUn) {
        const uint32_t k = atomicAdd(n_missing, 1u);
        if (k < 64) missing[k] = j;
    }
}

int check_outputs(asnn_dev* dev, DevNet& d) {
    if (!d.n_out) return ASNN_OK;
    cudaStream_t st = dev->stream;
    DevBuf<uint32_t> miss;
    CK(miss.alloc(65));
    CK(cudaMemsetAsync(miss.p, 0, 65 * 4, st));
    k_check_outputs<<<nblk(d.n_out), kT, 0, st>>>(d.nodes.p, d.N, d.dense, d.outputs.p, d.n_out,
                                                  d.level.p, miss.p + 1, miss.p);
    uint32_t h[65];
    CK(cudaMemcpyAsync(h, miss.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!h[0]) return ASNN_OK;
    std::vector<uint32_t> slots(h + 1, h + 1 + std::min<uint32_t>(h[0], 64));
    std::sort(slots.begin(), slots.end());
    std::string msg = "unassigned output node(s):";
    for (uint32_t j : slots) {
        const uint32_t g = static_cast<uint32_t>(
            std::upper_bound(d.h_out_prefix.begin(), d.h_out_prefix.end(), j) - d.h_out_prefix.begin()) - 1;
        msg += " " + std::to_string(d.h_outputs[g][j - d.h_out_prefix[g]]);
    }
    return fail(dev, ASNN_E_UNASSIGNED_OUTPUT, msg);
}

struct PhaseTimer {
    asnn_dev* dev;
    cudaEvent_t a, b;
    float* slot;
    PhaseTimer(asnn_dev* d, float* s) : dev(d), a(nullptr), b(nullptr), slot(s) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, dev->stream);
    }
    ~PhaseTimer() {
        cudaEventRecord(b, dev->stream);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(slot, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

int preprocess(asnn_dev* dev, uint32_t G, const asnn_network_desc* nets, const uint8_t* host_required,
               DevNet& d, bool want_levels) {
    {
        PhaseTimer t(dev, &dev->timings.upload_ms);
        RC(upload_networks(dev, G, nets, d));
        RC(build_adjacency(dev, d));
    }
    {
        PhaseTimer t(dev, &dev->timings.required_ms);
        RC(run_required(dev, d, host_required));
    }
    if (want_levels) {
        PhaseTimer t(dev, &dev->timings.segment_ms);
        RC(run_segment(dev, d));
    }
    return ASNN_OK;
}

__global__ void k_seed_sources(const uint32_t* __restrict__ pred_off, uint32_t N, uint32_t* __restrict__ level,
                               uint32_t* __restrict__ q, uint32_t* __restrict__ cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N && pred_off[i + 1] == pred_off[i]) {
        level[i] = 0u;
        q[atomicAdd(cnt, 1u)] = i;
    }
}

__global__ void k_count_unplaced(const uint32_t* __restrict__ level, uint32_t N, uint32_t* __restrict__ cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N && level[i] == kUn) atomicAdd(cnt, 1u);
}

int build(asnn_dev* dev, uint32_t G, const asnn_network_desc* nets, asnn_dev_layout** out) {
    if (!dev || !nets || !out) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    *out = nullptr;
    CK(cudaSetDevice(dev->device));
    dev->timings = asnn_timings{};
    DevNet d;
    RC(preprocess(dev, G, nets, nullptr, d, true));
    RC(check_outputs(dev, d));
    std::vector<NetMeta> metas;
    FlatDevice f;
    {
        PhaseTimer t(dev, &dev->timings.flatten_ms);
        // free what flatten no longer needs
        d.pred_adj.reset();
        d.succ_adj.reset();
        d.req.reset();
        d.si.reset();
        RC(run_flatten(dev, d, metas, f));
    }
    d = DevNet();
    return assemble_layout(dev, std::move(metas), std::move(f), out);
}

}  // namespace

// build() for one network whose arrays are already on the device (the
// loader's output): same pipeline, no host round trip of the connections.
int asnn_b200::build_device_network(asnn_dev* dev, DevBuf<uint32_t>&& nodes, uint32_t N, DevBuf<uint32_t>&& src,
                                    DevBuf<uint32_t>&& dst, DevBuf<float>&& w, uint64_t E,
                                    std::vector<uint32_t>&& inputs, std::vector<uint32_t>&& outputs,
                                    asnn_dev_layout** out) {
    cudaStream_t st = dev->stream;
    *out = nullptr;
    dev->timings = asnn_timings{};
    if (E >= kUn) return fail(dev, ASNN_E_INVALID, "more than 2^32-1 connections");
    DevNet d;
    d.G = 1;
    d.N = N;
    d.E = E;
    uint32_t last = 0;
    if (N) CK(cudaMemcpyAsync(&last, nodes.p + (N - 1), 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint32_t bound = N ? last + 1 : 0;  // layout.cpp:24-26
    if (bound == 0 && N) return fail(dev, ASNN_E_INVALID, "id space exceeds 2^32-1");
    d.dense = N == 0 || last == N - 1;
    d.h_idb = {0, bound};
    d.h_idbound = {bound};
    d.h_in_prefix = {0, static_cast<uint32_t>(inputs.size())};
    d.h_out_prefix = {0, static_cast<uint32_t>(outputs.size())};
    d.h_node_prefix = {0, N};
    d.n_in = static_cast<uint32_t>(inputs.size());
    d.n_out = static_cast<uint32_t>(outputs.size());
    d.nodes = std::move(nodes);
    d.src = std::move(src);
    d.dst = std::move(dst);
    d.w = std::move(w);
    CK(d.inputs.alloc(d.n_in));
    CK(d.outputs.alloc(d.n_out));
    if (d.n_in) CK(cudaMemcpyAsync(d.inputs.p, inputs.data(), d.n_in * 4ull, cudaMemcpyHostToDevice, st));
    if (d.n_out) CK(cudaMemcpyAsync(d.outputs.p, outputs.data(), d.n_out * 4ull, cudaMemcpyHostToDevice, st));
    d.h_inputs = {std::move(inputs)};
    d.h_outputs = {std::move(outputs)};
    CK(d.idb_prefix.alloc(2));
    CK(d.in_prefix.alloc(2));
    CK(d.out_prefix.alloc(2));
    CK(cudaMemcpyAsync(d.idb_prefix.p, d.h_idb.data(), 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d.in_prefix.p, d.h_in_prefix.data(), 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d.out_prefix.p, d.h_out_prefix.data(), 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    {
        PhaseTimer t(dev, &dev->timings.upload_ms);
        RC(build_adjacency(dev, d));
    }
    {
        PhaseTimer t(dev, &dev->timings.required_ms);
        RC(run_required(dev, d, nullptr));
    }
    {
        PhaseTimer t(dev, &dev->timings.segment_ms);
        RC(run_segment(dev, d));
    }
    RC(check_outputs(dev, d));
    std::vector<NetMeta> metas;
    FlatDevice f;
    {
        PhaseTimer t(dev, &dev->timings.flatten_ms);
        d.pred_adj.reset();
        d.succ_adj.reset();
        d.req.reset();
        d.si.reset();
        RC(run_flatten(dev, d, metas, f));
    }
    d = DevNet();
    return assemble_layout(dev, std::move(metas), std::move(f), out);
}

// Cycle test of validate (network.cpp:204): Kahn from every node without
// predecessors over all connections; a node left without a level lies on, or
// downstream of, a cycle.  nodes sorted unique; src / dst ids (device).
int asnn_b200::device_cycle_check(asnn_dev* dev, const uint32_t* nodes, uint32_t N, const uint32_t* src,
                                  const uint32_t* dst, uint64_t E, bool* cyclic) {
    cudaStream_t st = dev->stream;
    *cyclic = false;
    if (!N || !E) return ASNN_OK;
    DevNet d;
    d.N = N;
    d.E = E;
    d.dense = false;
    CK(d.nodes.alloc(N));
    CK(d.src.alloc(E));
    CK(d.dst.alloc(E));
    CK(cudaMemcpyAsync(d.nodes.p, nodes, N * 4ull, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(d.src.p, src, E * 4ull, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(d.dst.p, dst, E * 4ull, cudaMemcpyDeviceToDevice, st));
    RC(build_adjacency(dev, d));
    DevBuf<uint32_t> rem, q0, q1, cnt, req, level;
    CK(level.alloc(N + 1));
    CK(cudaMemsetAsync(level.p, 0xFF, (N + 1) * 4ull, st));
    CK(req.alloc(N + 1));
    CK(cudaMemsetAsync(req.p, 0x01, (N + 1) * 4ull, st));  // nonzero: every node may be placed
    CK(rem.alloc(N + 1));
    k_degree<<<nblk(N), kT, 0, st>>>(d.pred_off.p, N, rem.p);
    CK(q0.alloc(N + 1));
    CK(q1.alloc(N + 1));
    CK(cnt.alloc(4));
    CK(cudaMemsetAsync(cnt.p, 0, 16, st));
    k_seed_sources<<<nblk(N), kT, 0, st>>>(d.pred_off.p, N, level.p, q0.p, cnt.p);
    CK(cudaGetLastError());
    uint32_t blocks = 0;
    RC(coop_grid(dev, reinterpret_cast<const void*>(k_kahn), &blocks));
    void* args[] = {&d.succ_off.p, &d.succ_adj.p, &rem.p, &req.p, &level.p, &q0.p, &q1.p, &cnt.p};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_kahn), blocks, kT, args, 0, st));
    CK(cudaMemsetAsync(cnt.p + 3, 0, 4, st));
    k_count_unplaced<<<nblk(N), kT, 0, st>>>(level.p, N, cnt.p + 3);
    uint32_t h = 0;
    CK(cudaMemcpyAsync(&h, cnt.p + 3, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *cyclic = h != 0;
    return ASNN_OK;
}

extern "C" {

int asnn_dev_compute_required(asnn_dev* dev, const asnn_network_desc* net, uint8_t* required) {
    if (!dev || !net || (net->n_nodes && !required)) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    CK(cudaSetDevice(dev->device));
    DevNet d;
    RC(preprocess(dev, 1, net, nullptr, d, false));
    std::vector<uint32_t> r(d.N);
    if (d.N) CK(cudaMemcpy(r.data(), d.req.p, d.N * 4ull, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < d.N; ++i) required[i] = r[i] ? 1 : 0;
    return ASNN_OK;
}

int asnn_dev_segment(asnn_dev* dev, const asnn_network_desc* net, const uint8_t* required, uint32_t* level,
                     uint32_t* n_layers) {
    if (!dev || !net || !n_layers || (net->n_nodes && !level)) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    CK(cudaSetDevice(dev->device));
    DevNet d;
    RC(preprocess(dev, 1, net, required, d, true));
    if (d.N) CK(cudaMemcpy(level, d.level.p, d.N * 4ull, cudaMemcpyDeviceToHost));
    *n_layers = d.n_layers;
    return ASNN_OK;
}

int asnn_dev_build_layout(asnn_dev* dev, const asnn_network_desc* net, asnn_dev_layout** out) {
    return build(dev, 1, net, out);
}

int asnn_dev_build_population(asnn_dev* dev, uint32_t n, const asnn_network_desc* nets,
                              asnn_dev_layout** out) {
    if (n == 0) return fail(dev, ASNN_E_INVALID, "empty population");
    return build(dev, n, nets, out);
}

}  // extern "C"
