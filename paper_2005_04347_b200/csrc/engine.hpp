// engine.hpp -- internal host-side structures of the ASNN engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "asnn_dev.h"

namespace asnn_b200 {

// Stream-ordered allocation: while an AllocStream guard is active on this
// thread (every C-ABI entry point that allocates sets one to the handle's
// stream), DevBuf allocates with cudaMallocAsync on that stream and frees with
// cudaFreeAsync on the same stream -- after all work enqueued there that uses
// the buffer, with no device-wide synchronisation and no unmapping (the pool
// keeps its memory).  Work on other streams joins back before the free
// (fork/join events); asnn_dev_free_layout synchronises the current stream
// first.  Outside a guard: plain cudaMalloc / cudaFree.
inline cudaStream_t& alloc_stream_slot() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}
inline bool& alloc_stream_on() {
    static thread_local bool on = false;
    return on;
}
struct AllocStream {
    cudaStream_t prev;
    bool prev_on;
    explicit AllocStream(cudaStream_t s) : prev(alloc_stream_slot()), prev_on(alloc_stream_on()) {
        alloc_stream_slot() = s;
        alloc_stream_on() = true;
    }
    ~AllocStream() {
        alloc_stream_slot() = prev;
        alloc_stream_on() = prev_on;
    }
};

// Owning device buffer.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;  // stream of a stream-ordered allocation
    bool async = false;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), async(o.async) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p;
            n = o.n;
            s = o.s;
            async = o.async;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    void reset() {
        if (p) {
            if (async) cudaFreeAsync(p, s);
            else cudaFree(p);
        }
        p = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count) {
        reset();
        if (count == 0) count = 1;
        cudaError_t e;
        if (alloc_stream_on()) {
            s = alloc_stream_slot();
            async = true;
            e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s);
        } else {
            async = false;
            e = cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T));
        }
        if (e == cudaSuccess) n = count;
        else p = nullptr;
        return e;
    }
    cudaError_t ensure(size_t count) { return count <= n ? cudaSuccess : alloc(count); }
};

// Pinned host staging buffer.
struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() { reset(); }
    void reset() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    cudaError_t ensure(size_t b) {
        if (b <= bytes) return cudaSuccess;
        reset();
        cudaError_t e = cudaMallocHost(&p, b);
        if (e == cudaSuccess) bytes = b;
        else p = nullptr;
        return e;
    }
};

}  // namespace asnn_b200

struct asnn_dev {
    int device = 0;
    int sm_count = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;  // heavy-row branch of each level (fork/join)
    std::vector<cudaEvent_t> fork_ev, join_ev;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr, ev4 = nullptr;
    std::recursive_mutex mu;
    std::string err;
    uint32_t heavy_threshold = 512;  // in-degree above which rows stream through k_heavy
    uint32_t sweep_mode = 0;         // 0 auto, 1 per-layer launches, 2 K-cta when it fits
    uint32_t option_epoch = 0;       // bumps invalidate cached sweep graphs
    asnn_timings timings{};
    asnn_b200::PinnedBuf pin_x, pin_out;  // pinned staging of pageable host buffers (all layouts)
    asnn_b200::PinnedBuf stage[2];        // double-buffered staging of large pageable transfers
    asnn_b200::PinnedBuf arena;           // small uploads of one layout build, bump-allocated (h2d)
    size_t arena_used = 0;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    // NCCL communicator this device belongs to (group.cu): one rank of a
    // multi-process job (asnn_dev_comm_init) or a member of an asnn_group
    void* comm = nullptr;
    int comm_rank = 0, comm_size = 1;
    asnn_eval_buf* once = nullptr;  // asnn_dev_eval_layout's staging (once.cu)
};

namespace asnn_b200 {

// Large transfers between pageable host memory and the device (the loader's
// text, the parsed corpus): 8 MB chunks through two pinned staging buffers,
// the host side of each chunk copied by up to 8 threads while the other
// chunk's DMA runs.  Small or page-locked buffers take one cudaMemcpyAsync.
// The staged paths return with the host buffer no longer needed (download:
// filled); the direct ones are ordinary stream-ordered copies.
cudaError_t upload_host(asnn_dev* dev, void* dst, const void* src, size_t len, cudaStream_t st);
cudaError_t download_host(asnn_dev* dev, void* dst, const void* src, size_t len, cudaStream_t st);
// A host -> device copy inside a layout build: pageable sources are packed
// into the handle's pinned arena (one host memcpy, then an asynchronous DMA
// instead of the driver's synchronous pageable path); the build synchronises
// before it returns, after which arena_reset() recycles it.  Large or
// non-fitting copies take upload_host.
cudaError_t h2d(asnn_dev* dev, void* dst, const void* src, size_t len, cudaStream_t st);
inline void arena_reset(asnn_dev* dev) { dev->arena_used = 0; }

// In-degree thresholds above which a row goes to the streamed heavy kernel.
constexpr int kNumHeavyThr = 9;
__host__ __device__ constexpr uint32_t heavy_thr(int t) {
    return t == 0 ? 16u : t == 1 ? 32u : t == 2 ? 64u : t == 3 ? 128u : t == 4 ? 256u
         : t == 5 ? 512u : t == 6 ? 1024u : t == 7 ? 4096u : 0xFFFFFFFFu;
}

// One network inside a layout (a population holds many).
struct NetMeta {
    uint32_t pos_base = 0;    // first global position
    uint32_t n_pos = 0;       // assigned nodes
    uint32_t n_sensors = 0;   // layer-0 nodes
    uint32_t n_layers = 0;    // total_layers of this network
    uint32_t id_bound = 0;
    uint32_t n_in = 0, n_out = 0;
    uint32_t in_prefix = 0, out_prefix = 0, idb_prefix = 0;
    uint64_t edge_base = 0, n_edges = 0;
    uint64_t dropped = 0;
    std::vector<uint32_t> layer_offsets;  // local positions, [n_layers + 1]
    std::vector<uint32_t> inputs;         // declared input ids (layout.cpp:23)
    std::vector<uint32_t> outputs;        // declared output ids
};

// Cached CUDA graph of one activation sweep.  The first activation with a
// given (batch, buffers, stream, options) launches directly and only records
// them; the graph is captured when they repeat, so one-shot layouts (the
// per-call eval_parallel drop-in) never pay for capture + instantiation.
struct SweepGraph {
    bool seen = false;
    cudaGraphExec_t exec = nullptr;
    uint32_t n_vec = 0;
    const float* x = nullptr;
    float* out = nullptr;
    float* state = nullptr;
    cudaStream_t stream = nullptr;
    uint32_t epoch = 0;
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
    }
};

}  // namespace asnn_b200

struct asnn_dev_layout {
    asnn_dev* dev = nullptr;
    std::vector<asnn_b200::NetMeta> nets;
    uint32_t total_pos = 0, total_sensors = 0, total_in = 0, total_out = 0, total_idb = 0;
    uint32_t n_levels = 0;  // global levels (max over nets)
    uint32_t max_width = 0, max_deg = 0;
    uint64_t total_edges = 0, dropped = 0;
    std::vector<uint32_t> lvl_off;  // sched offsets per global level, [n_levels + 1]
    std::vector<uint32_t> win_lo, win_hi;  // per level: source position window (win_rows.cuh)
    std::vector<uint32_t> heavy_cnt;  // [kNumHeavyThr][n_levels + 1] rows above heavy_thr(t)

    asnn_b200::DevBuf<uint32_t> row_ptr;    // [total_pos + 1]
    asnn_b200::DevBuf<uint2> edges;         // [total_edges] {src pos, w bits}
    asnn_b200::DevBuf<uint32_t> sched;      // [total_pos] level-major schedule
    asnn_b200::DevBuf<uint4> rtask;         // [total_pos - sensors] {row, first edge, end edge, 0} per sched entry
    asnn_b200::DevBuf<uint4> sinfo;         // [total_sensors]
    asnn_b200::DevBuf<uint4> oinfo;         // [total_out]
    asnn_b200::DevBuf<uint32_t> state_map;  // [total_idb] id -> pos
    asnn_b200::DevBuf<uint32_t> idb_prefix; // [n_nets + 1]
    asnn_b200::DevBuf<uint32_t> node_ids;   // [total_pos]
    asnn_b200::DevBuf<uint32_t> d_meta;     // per-network prefix tables (MetaPtrs)
    asnn_b200::DevBuf<uint32_t> lo_base;    // [n_nets + 1] offsets into lo_cat
    bool sched_ready = false;               // sched / rtask / heavy_cnt built (ensure_schedule)

    // activation workspace
    asnn_b200::DevBuf<float> A;
    asnn_b200::DevBuf<float> x_stage, out_stage;
    asnn_b200::SweepGraph graph;

    // K-cta (whole sweep in one CTA per network x column slice)
    asnn_b200::DevBuf<uint32_t> cta_nets;  // [n_nets][12] CtaNet records
    asnn_b200::DevBuf<uint32_t> lo_cat;    // per net: layer offsets (local positions)
    asnn_b200::DevBuf<uint32_t> le_cat;    // per net: layer offsets as global edge indices
    uint32_t max_pos = 0;                  // largest network (positions)
    uint32_t max_level_edges = 0;          // most edges into one layer of one network
    bool zero_refs = false;                // some predecessor has no position (zero row)
    uint32_t zero_ldA = 0;                 // row pitch the zero row was last cleared at

    // Heavy-row segments (one network; segments.cuh): short ones run in k_rows
    // ahead of the level's rows, long ones in k_heavy
    asnn_b200::DevBuf<uint4> seg;          // {row, first edge, end edge, aux}
    std::vector<uint32_t> seg_short_off;   // [n_levels + 1] short segments of each step
    std::vector<uint32_t> seg_long_off;    // [n_levels + 1] long segments of each step
    uint32_t n_slots = 0;                  // partial-sum slots (heavy rows)
    uint64_t seg_key = ~0ull;              // options they were cut for
    asnn_b200::DevBuf<float> accbuf;       // [n_slots][ldA] partial sums
    // K-cta pipelined consumers: per position, the first stored edge whose
    // source is on the layer just below (k_splits)
    asnn_b200::DevBuf<uint32_t> split;     // [total_pos] absolute edge index
    uint32_t split_d = 0;                  // the prefix depth split[] was computed for
    // K-chain staging plan (chain.cuh, ensure_groups): per group 2 x uint4
    // (chain::GroupPlan), per-network group offsets, per layer 2 x uint4
    // (chain::LayerPlan, lo_cat indexing)
    asnn_b200::DevBuf<uint4> grp;
    asnn_b200::DevBuf<uint32_t> grp_off;   // [n_nets + 1]
    asnn_b200::DevBuf<uint4> lplan;
    uint32_t grp_target = 0, grp_ring = 0;  // group byte target and ring the plan was built for
    std::vector<uint32_t> le_host, lo_base_host;  // host copies of le_cat / lo_base

    asnn_dev_server* server = nullptr;     // live resident server (asnn_dev_server_start)
    // TMA descriptor of A for k_rows_tma (tma_rows.cuh), for (A, ldA) as built
    alignas(64) unsigned char tmA[128] = {};
    const float* tmA_base = nullptr;
    uint32_t tmA_ld = 0;
    ~asnn_dev_layout() { graph.reset(); }
};

namespace asnn_b200 {

// Records `msg` (plus the CUDA error string) as the handle's last error and
// returns the status.
int fail(asnn_dev* dev, int status, const std::string& msg);
int cuda_fail(asnn_dev* dev, cudaError_t e, const char* what);

// Device-side assembly of a layout from flattened per-network arrays that are
// already resident (used by upload, build and population paths).  Takes
// ownership of d_node_ids / d_row_ptr; d_in_ids / d_w are per-edge source ids
// (local to their network) and weights, freed by the caller.
struct FlatDevice {
    DevBuf<uint32_t> node_ids;  // [P]  global pos order
    DevBuf<uint32_t> row_ptr;   // [P+1] global edge offsets
    DevBuf<uint32_t> in_ids;    // [E]
    DevBuf<float> w;            // [E]
    DevBuf<uint32_t> inputs;    // [sum n_in]  declared input ids, per net
    DevBuf<uint32_t> outputs;   // [sum n_out] declared output ids, per net
};
int assemble_layout(asnn_dev* dev, std::vector<NetMeta>&& nets, FlatDevice&& flat,
                    asnn_dev_layout** out);

// compute_required + segment + flatten for one network already on the device
// (preprocess.cu; the loader's output).  Takes ownership of the arrays.
int build_device_network(asnn_dev* dev, DevBuf<uint32_t>&& nodes, uint32_t N, DevBuf<uint32_t>&& src,
                         DevBuf<uint32_t>&& dst, DevBuf<float>&& w, uint64_t E, std::vector<uint32_t>&& inputs,
                         std::vector<uint32_t>&& outputs, asnn_dev_layout** out);

// One activation sweep of a resident layout enqueued on the handle's stream
// (graph-cached; no synchronisation): x_dev [n_vec][inputs], out_dev
// [n_vec][outputs] (may be null), state_dev [n_vec][id_bound] (may be null).
int enqueue_sweep(asnn_dev_layout* L, const float* x_dev, uint32_t n_vec, float* out_dev, float* state_dev);

// Destroys the handle's NCCL communicator, if any (group.cu).
void release_comm(asnn_dev* dev);

// validate's cycle test on device arrays (preprocess.cu): nodes sorted unique,
// connections as (src, dst) ids.
int device_cycle_check(asnn_dev* dev, const uint32_t* nodes, uint32_t N, const uint32_t* src, const uint32_t* dst,
                       uint64_t E, bool* cyclic);

}  // namespace asnn_b200
