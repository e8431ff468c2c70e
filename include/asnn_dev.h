/*
 * asnn_dev.h -- C-ABI of the B200-native ASNN activation engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arxiv/paper_2005_04347, /root/reference/proj):
 *
 *   compute_required (network.cpp:222-255)      -> asnn_dev_compute_required
 *   segment          (segmentation.cpp:20-101)  -> asnn_dev_segment
 *   flatten          (layout.cpp:12-83)         -> asnn_dev_build_layout (+ _download)
 *   eval_parallel, Backend::DeviceCompute
 *                    (eval.hpp:20,37-39; the seam at eval.cpp:51-52)
 *                                               -> per call: asnn_eval_buf_stage + _run
 *                                                  (or asnn_dev_eval_layout); resident:
 *                                                  asnn_dev_upload_layout + asnn_dev_activate
 *   read_outputs     (eval.cpp:82-87)           -> `out` argument of asnn_dev_activate
 *   layer_slice_bounds / max_layer_width / depth
 *                    (layout.cpp:85-91, eval.cpp:89-94, segmentation.cpp:103-105)
 *                                               -> asnn_dev_layout_info / _layer_slice
 *
 * Conventions:
 *  - plain pointers and sizes; every host pointer is caller-owned and only
 *    read (const) or written during the call; nothing is retained;
 *  - errors are status codes (asnn_status), each mapping 1:1 to a reference
 *    exception type (errors.hpp:9-55); asnn_dev_last_error() holds the text;
 *  - one asnn_dev owns one CUDA stream; calls on one handle are serialised by
 *    an internal mutex; use one handle per thread for concurrency;
 *  - every call returns only after its results are visible to the caller
 *    (SPEC.md:329), except the *_device variants, which are stream-ordered.
 * Node ids, layers and positions are uint32; edge counts are uint64.
 */
#ifndef ASNN_DEV_H
#define ASNN_DEV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum asnn_status {
    ASNN_OK = 0,
    ASNN_E_UNAVAILABLE = 1,       /* BackendUnavailable (errors.hpp:33-35; eval.cpp:51-52) */
    ASNN_E_ARITY = 2,             /* InputArityMismatch (errors.hpp:9-11; eval.cpp:26-28) */
    ASNN_E_UNASSIGNED_OUTPUT = 3, /* UnassignedOutput = OutputUnreachable (errors.hpp:14-17;
                                     layout.cpp:13-17) */
    ASNN_E_LAYER_RANGE = 4,       /* LayerOutOfRange (errors.hpp:19-21; layout.cpp:87-89) */
    ASNN_E_INVALID = 5,           /* invalid argument (null pointer, size overflow) */
    ASNN_E_CUDA = 6,              /* CUDA runtime / launch failure */
    ASNN_E_OOM = 7,               /* device or pinned allocation failed */
    ASNN_E_INFEASIBLE = 8,        /* InfeasibleSpec (errors.hpp:23-25; netgen.cpp:29-53) */
    ASNN_E_PARSE = 9,             /* ParseError (errors.hpp:31-35): "line N: ..." */
    ASNN_E_VALIDATION = 10,       /* ValidationError (errors.hpp:37-53): "invalid network\n  ..." */
    ASNN_E_IO = 11                /* IoError (errors.hpp:27-29) */
} asnn_status;

#define ASNN_UNASSIGNED 0xFFFFFFFFu

typedef struct asnn_dev asnn_dev;               /* device + stream + last error      */
typedef struct asnn_dev_layout asnn_dev_layout; /* device-resident level-sorted CSR  */

/* Network (network.hpp:25-32) as plain arrays.  `nodes` sorted ascending and
 * unique; inputs/outputs in declared order; connections as SoA. */
typedef struct asnn_network_desc {
    uint32_t n_nodes;
    const uint32_t* nodes;
    uint32_t n_inputs;
    const uint32_t* inputs;
    uint32_t n_outputs;
    const uint32_t* outputs;
    uint64_t n_connections;
    const uint32_t* source;
    const uint32_t* target;
    const float* weight;
} asnn_network_desc;

/* LayeredLayout (layout.hpp:27-37) in CSR form: node k of the flat array
 * (sorted by (layer, id)) has predecessors in_nodes[row_ptr[k]..row_ptr[k+1])
 * -- ids, in the stored accumulation order -- with parallel in_weights.
 * `outputs` (optional, may be 0/NULL) are the ids read_outputs() projects. */
typedef struct asnn_layout_desc {
    uint32_t total_layers;
    const uint32_t* layer_offsets; /* [total_layers + 1] */
    uint32_t node_count;
    const uint32_t* node_ids;      /* [node_count] */
    const uint64_t* row_ptr;       /* [node_count + 1] */
    const uint32_t* in_nodes;      /* [row_ptr[node_count]] */
    const float* in_weights;       /* [row_ptr[node_count]] */
    uint32_t n_inputs;
    const uint32_t* input_order;   /* [n_inputs] sensor ids, declared order */
    uint32_t id_bound;
    uint32_t n_outputs;
    const uint32_t* outputs;       /* [n_outputs] */
} asnn_layout_desc;

/* Sizes of a device layout (all networks it holds, see build_population). */
typedef struct asnn_layout_info {
    uint32_t n_networks;
    uint32_t total_layers;        /* max over networks */
    uint32_t node_count;          /* assigned nodes, all networks */
    uint64_t edge_count;          /* stored predecessor entries */
    uint64_t dropped_connections; /* layout.cpp:56-58 */
    uint32_t id_bound;            /* sum over networks */
    uint32_t n_inputs;            /* sum over networks */
    uint32_t n_outputs;           /* sum over networks */
    uint32_t max_layer_width;     /* eval.cpp:89-94 */
    uint32_t max_in_degree;
} asnn_layout_info;

/* Per-phase device times of the last build / activate call (CUDA events). */
typedef struct asnn_timings {
    float upload_ms;
    float required_ms;
    float segment_ms;
    float flatten_ms;
    float activate_ms;
} asnn_timings;

/* ---- device handle ------------------------------------------------------ */
int asnn_dev_device_count(int* count);
int asnn_dev_open(int device, asnn_dev** out);       /* ASNN_E_UNAVAILABLE: no GPU */
void asnn_dev_close(asnn_dev* dev);
const char* asnn_dev_last_error(const asnn_dev* dev); /* per handle; "" when none */
const char* asnn_dev_version(void);
/* Run on a caller stream (a cudaStream_t, e.g. torch's current stream);
 * NULL restores the handle's own stream. */
int asnn_dev_set_stream(asnn_dev* dev, void* cuda_stream);
void* asnn_dev_get_stream(asnn_dev* dev);
int asnn_dev_synchronize(asnn_dev* dev);
/* Rows with more predecessors than this stream through the TMA-staged heavy
 * kernel (default 512, or $ASNN_HEAVY_THRESHOLD; 0xFFFFFFFF = never).
 * Numerics are identical either way; this is a scheduling knob. */
int asnn_dev_set_heavy_threshold(asnn_dev* dev, uint32_t min_in_degree);
/* Sweep strategy: 0 = automatic (default, $ASNN_SWEEP_MODE), 1 = one launch
 * per dependency level (for one network with a batch of 64 or a multiple of
 * 128, heavy rows are split into segments that run in the levels of their
 * sources), 2 = one CTA per (network, batch slice) running every level with
 * shared-memory-resident activations whenever they fit, 3 = one launch per
 * level with whole rows only, 4 = (one network) one CTA per batch column
 * keeping only a ring of the newest positions in shared memory and older
 * sources in HBM/L2, with the smallest legal ring (the windowed K-cta, an
 * opt-in experiment: ASNN_CTA_WIN=1), 5 = (one network) the windowed K-chain
 * (chain.cuh WIN: the automatic choice for deep, narrow networks whose
 * one-column slices need more than one wave of CTAs; forced here to exercise
 * it).  Also a scheduling knob: results are identical. */
int asnn_dev_set_sweep_mode(asnn_dev* dev, uint32_t mode);
int asnn_dev_last_timings(const asnn_dev* dev, asnn_timings* out);

/* ---- preprocessing (GPU) ------------------------------------------------
 * compute_required (network.cpp:222-255): required[n_nodes] <- 1 for members,
 * indexed like net->nodes. */
int asnn_dev_compute_required(asnn_dev* dev, const asnn_network_desc* net, uint8_t* required);

/* segment (segmentation.cpp:20-101): level[n_nodes] <- layer of each node
 * (ASNN_UNASSIGNED for the rest), *n_layers <- depth() (>= 1).  `required`
 * may be NULL (then computed on the device). */
int asnn_dev_segment(asnn_dev* dev, const asnn_network_desc* net, const uint8_t* required,
                     uint32_t* level, uint32_t* n_layers);

/* compute_required + segment + flatten on the device; the result stays
 * resident.  ASNN_E_UNASSIGNED_OUTPUT when an output has no layer. */
int asnn_dev_build_layout(asnn_dev* dev, const asnn_network_desc* net, asnn_dev_layout** out);

/* A NEAT population: n_networks independent networks in one layout; their
 * levels run side by side (one block-diagonal DAG). */
int asnn_dev_build_population(asnn_dev* dev, uint32_t n_networks, const asnn_network_desc* nets,
                              asnn_dev_layout** out);

/* Upload a host-flattened layout (what eval_parallel receives, eval.cpp:49).
 * Re-upload on every eval_parallel call: the reference mutates layouts in
 * place between evaluations (asnn_main.cpp:264-278). */
int asnn_dev_upload_layout(asnn_dev* dev, const asnn_layout_desc* layout, asnn_dev_layout** out);

void asnn_dev_free_layout(asnn_dev_layout* layout);

int asnn_dev_layout_info(const asnn_dev_layout* layout, asnn_layout_info* info);

/* layer_slice_bounds (layout.cpp:85-91) of network 0. */
int asnn_dev_layer_slice(const asnn_dev_layout* layout, uint32_t layer, uint32_t* start,
                         uint32_t* count);

/* Download network `net_index`'s flattened layout (flatten parity):
 * arrays sized from asnn_dev_network_info. */
int asnn_dev_network_info(const asnn_dev_layout* layout, uint32_t net_index,
                          asnn_layout_info* info);
int asnn_dev_layout_download(asnn_dev_layout* layout, uint32_t net_index, uint32_t* layer_offsets,
                             uint32_t* node_ids, uint64_t* row_ptr, uint32_t* in_nodes,
                             float* in_weights, uint32_t* input_order);

/* ---- one-call eval_parallel (the per-call drop-in, once.cu) ----------------
 * Replaces eval_parallel(layout, inputs, cfg) with Backend::DeviceCompute
 * (/root/reference/proj/src/eval.cpp:49-80, seam at :51-52) when the layout
 * exists for one call only (the reference passes a host LayeredLayout to
 * every call and may mutate it in between, asnn_main.cpp:264-278).  Nothing
 * is renumbered or kept: the state stays id-indexed as in the reference.
 *
 *   asnn_eval_buf_stage  -- page-locked arrays sized from dims; the caller
 *                           writes the layout's CSR straight into them
 *                           (layout.hpp:13-37: ids, row_ptr, predecessor ids
 *                           in stored order, weights) and, per layer-0 node,
 *                           inputs[id] of make_state (eval.cpp:25-35)
 *   asnn_eval_buf_run    -- one kernel (plus one DMA for larger layouts);
 *                           writes state.outputs [id_bound] (unassigned ids
 *                           0.0f).  ASNN_E_INVALID for malformed layouts
 *                           (layer table, row_ptr or ids out of range).
 * One buffer per calling thread; runs on one handle serialise.  The staged
 * pointers stay valid until the buffer's next stage (which may reallocate)
 * or free; a run may be repeated on the same staging. */
typedef struct asnn_eval_buf asnn_eval_buf;
typedef struct asnn_eval_dims {
    uint32_t total_layers;
    uint32_t node_count;
    uint32_t sensor_count;  /* layer 0 = nodes_per_layer[0] */
    uint32_t id_bound;
    uint64_t edge_count;    /* < 2^32 */
} asnn_eval_dims;
typedef struct asnn_eval_stage {
    uint32_t* layer_offsets; /* [total_layers + 1] */
    uint32_t* node_ids;      /* [node_count] */
    uint32_t* row_ptr;       /* [node_count + 1], 32-bit */
    uint32_t* in_nodes;      /* [edge_count] */
    float* in_weights;       /* [edge_count] */
    float* sensor_inputs;    /* [sensor_count] inputs[node_ids[k]] */
} asnn_eval_stage;
int asnn_eval_buf_create(asnn_dev* dev, asnn_eval_buf** out);
void asnn_eval_buf_free(asnn_eval_buf* buf);
int asnn_eval_buf_stage(asnn_eval_buf* buf, const asnn_eval_dims* dims, asnn_eval_stage* stage);
int asnn_eval_buf_run(asnn_eval_buf* buf, float* state_outputs);
/* kernel variant of the last run: 0 zero-copy into shared memory, 1 DMA +
 * one CTA, 2 DMA + cooperative grid, both with cp.async rings of the next
 * items' slices; 3 / 4 the same without the rings; 5 / 6 an 8-CTA cluster
 * holding the layout in distributed shared memory (per-layer shares / layer
 * ranges) (ASNN_ONCE_MODE forces) */
int asnn_eval_buf_mode(const asnn_eval_buf* buf, uint32_t* mode);
/* The same from a layout descriptor and one input vector (make_state on the
 * host; ASNN_E_ARITY when n_x != n_inputs, eval.cpp:26-28). */
int asnn_dev_eval_layout(asnn_dev* dev, const asnn_layout_desc* layout, const float* x, uint64_t n_x,
                         float* state_outputs);

/* ---- activation -----------------------------------------------------------
 * eval_parallel(DeviceCompute) over a batch: x is [n_vec][n_inputs] per
 * network (networks concatenated), `out` (optional) receives the declared
 * outputs [n_vec][n_outputs] per network (read_outputs order), `state`
 * (optional) the id-indexed op array [n_vec][id_bound] per network
 * (ActivationState.outputs, eval.hpp:14-17; unassigned ids 0.0f).
 * Host pointers; copies happen inside the call.  n_x must equal the total
 * inputs per vector or ASNN_E_ARITY is returned (eval.cpp:26-28). */
int asnn_dev_activate(asnn_dev_layout* layout, const float* x, uint32_t n_vec, uint64_t n_x,
                      float* out, float* state);

/* Batch-1 latency path (serve.cuh): a persistent one-CTA kernel that keeps
 * a single-network layout resident in shared memory and polls a doorbell in
 * page-locked host memory, so an activation costs no launch, copy call or
 * stream synchronisation -- the drop-in per-vector eval_parallel of a small
 * network (eval.cpp:49-80) at the latency of a PCIe round trip plus the
 * sweep.  max_vec (1..64) bounds the vectors per request.
 * ASNN_E_UNAVAILABLE when the layout holds several networks, does not fit
 * one SM's shared memory, or max_vec * n_inputs exceeds 511.  The server
 * is a persistent kernel on its own stream: it occupies one SM until
 * stopped, and a device-wide synchronisation (cudaDeviceSynchronize) waits
 * for it to exit -- synchronise streams instead.  asnn_dev_free_layout stops
 * a live server. */
typedef struct asnn_dev_server asnn_dev_server;
int asnn_dev_server_start(asnn_dev_layout* layout, uint32_t max_vec, asnn_dev_server** out);
/* Same contract as asnn_dev_activate with out != NULL, state == NULL:
 * x[n_vec][n_inputs] (n_x == n_inputs * n_vec, else ASNN_E_ARITY),
 * out[n_vec][n_outputs]; blocks until the outputs are in `out`. */
int asnn_dev_server_activate(asnn_dev_server* server, const float* x, uint32_t n_vec, uint64_t n_x, float* out);
void asnn_dev_server_stop(asnn_dev_server* server);
/* The last activation's host round trip (inputs posted -> outputs seen, ns)
 * and the device's phase times in SM cycles: [0] sensors, [1] layers,
 * [2] outputs issued, [3] waiting for the request (polling). */
int asnn_dev_server_timings(asnn_dev_server* server, double* host_ns, int64_t* device_cycles);

/* Same, with device pointers, stream-ordered on the handle's stream (no
 * synchronisation).  x_dev [n_vec][n_inputs], out_dev [n_vec][n_outputs]. */
int asnn_dev_activate_device(asnn_dev_layout* layout, const float* x_dev, uint32_t n_vec,
                             float* out_dev);

/* One sweep launched kernel by kernel (no graph) with a CUDA event between
 * launches on the handle's stream: ms[k] receives the device time of launch
 * k in order (sensors, each level, output gather); *n_launches its count
 * (ms must hold asnn_dev_activate_plan's `kernels` entries). */
int asnn_dev_profile_sweep(asnn_dev_layout* layout, const float* x_dev, uint32_t n_vec,
                           float* out_dev, float* ms, uint32_t* n_launches);

/* Number of kernels one activate of n_vec vectors launches, and the
 * algorithmic bytes it moves. */
int asnn_dev_activate_plan(asnn_dev_layout* layout, uint32_t n_vec, uint32_t* kernels,
                           uint64_t* alg_bytes, uint64_t* conn_evals);

/* Which sweep strategy an activate of n_vec vectors uses: 0 = per-level
 * launches of whole rows (k_rows / k_level, heavy rows on k_heavy), 1 =
 * per-level launches with heavy rows split into segments across the levels of
 * their sources (k_rows, long segments on k_heavy), 2 = one CTA per (network,
 * batch slice) for the whole sweep (k_cta), 3 = the same with decoupled
 * finish / prefix warps for deep, narrow layers (k_chain, chain.cuh). */
int asnn_dev_sweep_kind(asnn_dev_layout* layout, uint32_t n_vec, uint32_t* kind);

/* Debug: one sweep of n_vec (zero) vectors counting how often each op slot
 * is produced; counts[position][n_vec] (positions in level order, as
 * asnn_dev_layout_download's node_ids).  Every entry must be 1 -- "each slot
 * written exactly once" (proj/tests/test_eval.cpp:199-213).
 * Only the write-count build (build/debug/libasnn_b200_wc.so, make -C
 * paper_2005_04347_b200/csrc wc) counts; the product library returns
 * ASNN_E_UNAVAILABLE. */
int asnn_dev_debug_write_counts(asnn_dev_layout* layout, uint32_t n_vec, uint32_t* counts);

/* The device's sigmoid32 (network.hpp:54-59) over n host floats, for
 * exhaustive parity checks of the epilogue. */
int asnn_dev_sigmoid32(asnn_dev* dev, const float* x, float* y, uint64_t n);

/* The epilogue's fast path against its exact restatement for all 2^32 float
 * inputs, on the device: *mismatches must be 0; *exact_path counts the inputs
 * the rounding test handed to the exact path. */
int asnn_dev_sigmoid_selfcheck(asnn_dev* dev, uint64_t* mismatches, uint64_t* exact_path);

/* Microarchitecture probe: SM cycles per operation of a dependent chain of n
 * ops run by one thread (which: 0 sigmoid32, 1 DFMA, 2 FADD, 3 shared-memory
 * load, 4 double division, 5 exp, 6 empty loop iteration).  Evidence for
 * DESIGN.md's latency model. */
int asnn_dev_latency_probe(asnn_dev* dev, int which, int n, double* cycles_per_op);

/* ---- multi-GPU (north_star item 4) ----------------------------
 * A network's level-synchronous sweep does not shard without a per-level
 * exchange; what shards is the batch (a full layout replica per device, a
 * contiguous balanced slice of the vectors each) and a population (a
 * contiguous balanced slice of the networks per device, all vectors each).
 * Device g's inputs / outputs / state are contiguous slices of the caller's
 * arrays (same layouts as asnn_dev_activate), so the one collective is an
 * all-gather of the declared outputs in device order: ncclAllGather (equal
 * slices) or grouped ncclBroadcast (ragged), NCCL loaded at run time; the
 * copy engines (cudaMemcpyPeerAsync into device 0) when NCCL is absent or a
 * device is listed twice (one-GPU functional mode). */
typedef struct asnn_group asnn_group;               /* one process, G devices   */
typedef struct asnn_group_layout asnn_group_layout; /* a layout sharded over them */

/* Opens one asnn_dev per entry of devices[] (entries may repeat) and, when
 * they are distinct and libnccl loads, one NCCL communicator over them
 * (ncclCommInitAll). */
int asnn_group_open(const int* devices, uint32_t n_devices, asnn_group** out);
void asnn_group_close(asnn_group* group);
const char* asnn_group_last_error(const asnn_group* group);
/* *gather_kind: 0 single device, 1 NCCL, 2 copy engines (see _gather_note). */
int asnn_group_info(const asnn_group* group, uint32_t* n_devices, uint32_t* gather_kind);
const char* asnn_group_gather_note(const asnn_group* group);
/* Member handle i (sweep options, timings); owned by the group. */
asnn_dev* asnn_group_device(asnn_group* group, uint32_t i);
/* Batch sharding: compute_required + segment + flatten on every device
 * concurrently (a replica each), or a host-flattened layout uploaded to each. */
int asnn_group_build_layout(asnn_group* group, const asnn_network_desc* net, asnn_group_layout** out);
int asnn_group_upload_layout(asnn_group* group, const asnn_layout_desc* layout, asnn_group_layout** out);
/* Population sharding: networks [g*P/G, (g+1)*P/G) (balanced) on device g. */
int asnn_group_build_population(asnn_group* group, uint32_t n_networks, const asnn_network_desc* nets,
                                asnn_group_layout** out);
/* The member layout on device i (null for an empty population slice). */
int asnn_group_layout_member(const asnn_group_layout* layout, uint32_t i, asnn_dev_layout** member);
/* Device i's share of an activation of n_vec vectors: vectors it sweeps and
 * the float offsets / counts of its inputs and outputs in the caller's arrays. */
int asnn_group_shard(const asnn_group_layout* layout, uint32_t i, uint32_t n_vec, uint32_t* vecs,
                     uint64_t* x_off, uint64_t* x_count, uint64_t* out_off, uint64_t* out_count);
/* asnn_dev_activate over the group: host x / out / state in the single-device
 * layouts; each device sweeps its slice, the outputs are all-gathered on the
 * devices and read back from device 0; returns when all results are visible. */
int asnn_group_activate(asnn_group_layout* layout, const float* x, uint32_t n_vec, uint64_t n_x,
                        float* out, float* state);
/* Resident path (the benchmark's): stage inputs on the devices once, then
 * `repeats` sweeps + gathers; *ms = device time per repeat, max over devices. */
int asnn_group_stage_inputs(asnn_group_layout* layout, const float* x, uint32_t n_vec, uint64_t n_x);
int asnn_group_sweep(asnn_group_layout* layout, uint32_t repeats, float* ms);
int asnn_group_read_outputs(asnn_group_layout* layout, float* out);
void asnn_group_free_layout(asnn_group_layout* layout);

/* One process per device (a launcher such as torchrun): rank 0 creates the
 * 128-byte id, the launcher's store distributes it, every rank joins; then
 * asnn_dev_allgather enqueues the output all-gather on the handle's stream
 * (stream-ordered after the sweep, no synchronisation).  counts[n_ranks]:
 * floats each rank contributes; recv = their concatenation in rank order;
 * send may lie inside recv at this rank's offset (in place). */
int asnn_comm_unique_id(uint8_t* id128);
int asnn_dev_comm_init(asnn_dev* dev, const uint8_t* id128, int n_ranks, int rank);
int asnn_dev_allgather(asnn_dev* dev, const float* send_dev, float* recv_dev, const uint64_t* counts);

typedef struct asnn_corpus asnn_corpus;

/* ---- loading (io.hpp:23-31) on the device ---------------------------------
 * parse_network (io.cpp:83-156) followed by validate (network.cpp:151-216):
 * text = the bytes of an `asnn 1` file.  On success *out owns the network
 * (read it with asnn_corpus_desc): nodes sorted unique, inputs / outputs in
 * declared order, connections in file order.  ASNN_E_PARSE: the first
 * failing line (*err_line) and the reference's ParseError message
 * ("line N: ...") in asnn_dev_last_error; ASNN_E_VALIDATION: the
 * ValidationError message ("invalid network\n  ..."). */
int asnn_dev_parse_network(asnn_dev* dev, const char* text, uint64_t len, asnn_corpus** out,
                           uint32_t* err_line);
/* load -> levels on the device: parse_network + validate + compute_required +
 * segment + flatten, the parsed arrays never leaving HBM; *out is a resident
 * layout (asnn_dev_activate*).  Errors as asnn_dev_parse_network, then as
 * asnn_dev_build_layout. */
int asnn_dev_load_layout(asnn_dev* dev, const char* text, uint64_t len, asnn_dev_layout** out,
                         uint32_t* err_line);
/* validate (network.cpp:151-216) of an in-memory network on the device: the
 * ValidationReport's messages, in the reference's order, joined by '\n' into
 * report (cap bytes, NUL-terminated, truncated); *n_violations = their count
 * (0 = valid).  nodes must be sorted and unique (make_network's invariant). */
int asnn_dev_validate(asnn_dev* dev, const asnn_network_desc* net, char* report, uint64_t cap,
                      uint32_t* n_violations);
/* normalize (network.cpp:69-85): ids remapped to their positions in nodes
 * (dense 0..N-1), on the device; ASNN_E_INVALID if an id names no node. */
int asnn_dev_normalize(asnn_dev* dev, const asnn_network_desc* net, asnn_corpus** out);
/* read_network (io.cpp:167-173): ASNN_E_IO when the file cannot be read. */
int asnn_dev_read_network(asnn_dev* dev, const char* path, asnn_corpus** out, uint32_t* err_line);
/* parse_weight's from_chars<float> on n tokens buf[off[i], off[i+1]) on the
 * device: status 0 = parsed, 1 = rejected (every token is decided on the
 * device, the exact slow path included); the parser's number kernel, exposed
 * for parity tests. */
int asnn_dev_parse_weights(asnn_dev* dev, const char* buf, const uint64_t* off, uint64_t n, float* out,
                           uint8_t* status);

/* ---- synthetic corpora (host, deterministic) ------------------------------
 * generate(GenSpec) byte-identical to the reference (netgen.cpp:71-157),
 * the MLP-adjacent shape (config 2) and the banded power-law shape
 * (config 4).  A corpus handle owns its arrays; read them with
 * asnn_corpus_desc (pointers valid until asnn_corpus_free). */
int asnn_gen_reference(uint32_t input_count, uint32_t output_count, uint32_t hidden_count,
                       uint64_t connection_count, uint32_t target_depth, float weight_min,
                       float weight_max, uint64_t seed, asnn_corpus** out);
uint64_t asnn_gen_max_connections(uint32_t input_count, uint32_t output_count,
                                  uint32_t hidden_count, uint32_t target_depth);
int asnn_gen_mlp(uint32_t layers, uint32_t width, double p, uint64_t seed, asnn_corpus** out);
int asnn_gen_powerlaw(uint32_t n_nodes, uint32_t bands, uint32_t n_inputs, uint32_t n_outputs,
                      uint64_t target_edges, double alpha, uint64_t seed, asnn_corpus** out);
/* The same two bench shapes generated on the device (gen.cu; counter-based
 * per node, byte-identical to asnn_gen_mlp / asnn_gen_powerlaw): into a host
 * corpus, or straight into a resident layout (compute_required + segment +
 * flatten on the generated device arrays; the network never crosses the
 * host link).  SURVEY.md 8f rank 4; the reference's generate()
 * (netgen.cpp:71-157) cannot make these shapes at this scale. */
int asnn_dev_gen_mlp(asnn_dev* dev, uint32_t layers, uint32_t width, double p, uint64_t seed,
                     asnn_corpus** out);
int asnn_dev_gen_mlp_layout(asnn_dev* dev, uint32_t layers, uint32_t width, double p, uint64_t seed,
                            asnn_dev_layout** out);
int asnn_dev_gen_powerlaw(asnn_dev* dev, uint32_t n_nodes, uint32_t bands, uint32_t n_inputs,
                          uint32_t n_outputs, uint64_t target_edges, double alpha, uint64_t seed,
                          asnn_corpus** out);
int asnn_dev_gen_powerlaw_layout(asnn_dev* dev, uint32_t n_nodes, uint32_t bands, uint32_t n_inputs,
                                 uint32_t n_outputs, uint64_t target_edges, double alpha, uint64_t seed,
                                 asnn_dev_layout** out);
int asnn_corpus_desc(const asnn_corpus* corpus, asnn_network_desc* desc);
void asnn_corpus_free(asnn_corpus* corpus);

#ifdef __cplusplus
}
#endif

#endif /* ASNN_DEV_H */
