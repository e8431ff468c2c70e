// engine.cu -- device handle, layout assembly/upload, activation driver and
// the C-ABI entry points of include/asnn_dev.h (except preprocessing, which
// lives in preprocess.cu and corpora in netgen.cpp).
#include <algorithm>
#include <deque>
#include <mutex>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "engine.hpp"
#include "kernels.cuh"
#include "sort.cuh"

using namespace asnn_b200;

namespace asnn_b200 {

int fail(asnn_dev* dev, int status, const std::string& msg) {
    if (dev) dev->err = msg;
    return status;
}

int cuda_fail(asnn_dev* dev, cudaError_t e, const char* what) {
    const int st = (e == cudaErrorMemoryAllocation) ? ASNN_E_OOM : ASNN_E_CUDA;
    cudaGetLastError();  // clear sticky-free errors
    return fail(dev, st, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace asnn_b200

#define CK(expr)                                              \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_fail(dev, _e, #expr); \
    } while (0)

namespace {

constexpr uint32_t kThreads = 256;

inline uint32_t blocks_for(uint64_t n, uint32_t t = kThreads) {
    return static_cast<uint32_t>((n + t - 1) / t);
}

// g such that prefix[g] <= v < prefix[g+1] (prefix has n+1 entries, n >= 1).
__device__ __forceinline__ uint32_t find_seg(const uint32_t* __restrict__ prefix, uint32_t n,
                                             uint32_t v) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(&prefix[mid]) <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// meta layout on device: 6 arrays of (G+1) u32:
//   0 pos_base, 1 idb_prefix, 2 in_prefix, 3 out_prefix, 4 edge_base, 5 sensor_prefix
struct MetaPtrs {
    const uint32_t* pos;
    const uint32_t* idb;
    const uint32_t* in;
    const uint32_t* out;
    const uint32_t* edge;
    const uint32_t* sens;
    uint32_t G;
};

__global__ void k_state_map(MetaPtrs m, const uint32_t* __restrict__ node_ids, uint32_t P,
                            uint32_t* __restrict__ state_map, uint32_t* __restrict__ bad) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const uint32_t g = find_seg(m.pos, m.G, p);
    const uint32_t idb = m.idb[g + 1] - m.idb[g];
    const uint32_t id = node_ids[p];
    if (id >= idb) {
        atomicOr(bad, 1u);
        return;
    }
    state_map[m.idb[g] + id] = p;
}

// edges[k] = {position of source id (or the zero row P), weight bits}.
__global__ void k_edges(MetaPtrs m, const uint32_t* __restrict__ in_ids, const float* __restrict__ w,
                        uint64_t E, const uint32_t* __restrict__ state_map, uint32_t zero_row,
                        uint2* __restrict__ edges, uint32_t* __restrict__ bad) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= E) return;
    const uint32_t g = find_seg(m.edge, m.G, static_cast<uint32_t>(k));
    const uint32_t idb = m.idb[g + 1] - m.idb[g];
    const uint32_t id = in_ids[k];
    uint32_t pos = zero_row;
    if (id >= idb) atomicOr(bad, 2u);
    else {
        const uint32_t q = state_map[m.idb[g] + id];
        // A predecessor without a position reads its never-written 0.0f slot,
        // exactly like the reference's zero-initialised op array.
        pos = (q == kUnassigned) ? zero_row : q;
        if (q == kUnassigned) atomicOr(bad, 8u);  // not an error: K-cta keeps its guard
    }
    edges[k] = make_uint2(pos, __float_as_uint(w[k]));
}

// kofid[idb + id] = max(i + 1) over declared input index i of that id.
__global__ void k_input_index(MetaPtrs m, const uint32_t* __restrict__ inputs, uint32_t n_in_total,
                              uint32_t* __restrict__ kofid, uint32_t* __restrict__ bad) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_in_total) return;
    const uint32_t g = find_seg(m.in, m.G, j);
    const uint32_t idb = m.idb[g + 1] - m.idb[g];
    const uint32_t id = inputs[j];
    if (id >= idb) {
        atomicOr(bad, 4u);
        return;
    }
    atomicMax(&kofid[m.idb[g] + id], j - m.in[g] + 1);
}

__global__ void k_sinfo(MetaPtrs m, const uint32_t* __restrict__ node_ids,
                        const uint32_t* __restrict__ kofid, uint32_t S, uint4* __restrict__ sinfo) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const uint32_t g = find_seg(m.sens, m.G, s);
    const uint32_t p = m.pos[g] + (s - m.sens[g]);
    const uint32_t k1 = kofid[m.idb[g] + node_ids[p]];
    sinfo[s] = make_uint4(p, m.in[g], m.in[g + 1] - m.in[g], k1 ? k1 - 1 : kUnassigned);
}

__global__ void k_oinfo(MetaPtrs m, const uint32_t* __restrict__ outputs, uint32_t n_out_total,
                        const uint32_t* __restrict__ state_map, uint4* __restrict__ oinfo) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_out_total) return;
    const uint32_t g = find_seg(m.out, m.G, j);
    const uint32_t idb = m.idb[g + 1] - m.idb[g];
    const uint32_t id = outputs[j];
    const uint32_t pos = id < idb ? state_map[m.idb[g] + id] : kUnassigned;
    oinfo[j] = make_uint4(pos, m.out[g], m.out[g + 1] - m.out[g], j - m.out[g]);
}

__global__ void k_max_deg(const uint32_t* __restrict__ row_ptr, uint32_t P, uint32_t* __restrict__ out) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t d = 0;
    if (p < P) d = row_ptr[p + 1] - row_ptr[p];
    for (int o = 16; o; o >>= 1) d = max(d, __shfl_xor_sync(0xFFFFFFFFu, d, o));
    if ((threadIdx.x & 31) == 0 && d) atomicMax(out, d);
}

// Schedule sort keys: (layer << 16) | (0xFFFF - min(in-degree, 0xFFFF)).
__global__ void k_sched_keys(MetaPtrs m, const uint32_t* __restrict__ lo_cat,
                             const uint32_t* __restrict__ lo_base, const uint32_t* __restrict__ row_ptr,
                             uint32_t P, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const uint32_t g = find_seg(m.pos, m.G, p);
    const uint32_t lp = p - m.pos[g];
    const uint32_t nl = lo_base[g + 1] - lo_base[g] - 1;
    const uint32_t lv = find_seg(lo_cat + lo_base[g], nl, lp);
    const uint32_t deg = min(row_ptr[p + 1] - row_ptr[p], 0xFFFFu);
    keys[p] = (lv << 16) | (0xFFFFu - deg);
    vals[p] = p;
}

__global__ void k_heavy_counts(const uint32_t* __restrict__ keys, uint32_t n, uint32_t stride,
                               uint32_t* __restrict__ hv) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t lv = keys[i] >> 16;
    const uint32_t deg = 0xFFFFu - (keys[i] & 0xFFFFu);
#pragma unroll
    for (int t = 0; t < kNumHeavyThr; ++t)
        if (deg > heavy_thr(t)) atomicAdd(&hv[t * stride + lv], 1u);
}

// le_cat[j] = row_ptr[pos_base(g) + lo_cat[j]] for the network g owning j.
__global__ void k_layer_edges(const uint32_t* __restrict__ lo_cat, const uint32_t* __restrict__ lo_base,
                              uint32_t G, const uint32_t* __restrict__ pos_base,
                              const uint32_t* __restrict__ row_ptr, uint32_t n, uint32_t* __restrict__ le) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t g = find_seg(lo_base, G, j);
    le[j] = row_ptr[pos_base[g] + lo_cat[j]];
}

__global__ void k_row64_to_32(const uint64_t* __restrict__ in, uint32_t n, uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<uint32_t>(in[i]);
}

// Padded batch width: powers of two up to 128 columns, multiples of 128
// beyond, so an item (LANES threads x V columns) tiles a row exactly.
uint32_t padded_batch(uint32_t n_vec) {
    if (n_vec <= 1) return 1;
    if (n_vec <= 128) {
        uint32_t p = 1;
        while (p < n_vec) p <<= 1;
        return p;
    }
    return (n_vec + 127) / 128 * 128;
}

// One launch per level: k_level (row items, any batch width) or k_rows (row
// segments + row items, 4 columns per lane).
using LevelFn = void (*)(const uint32_t*, const uint2*, float*, uint32_t, const uint32_t*, uint32_t, uint32_t);
using RowsFn = void (*)(const uint2*, float*, uint32_t, const uint4*, uint32_t, uint32_t, const uint4*, uint32_t,
                        float*);
using WarpRowsFn = void (*)(const uint2*, float*, const uint4*, uint32_t);
using WarpRows4Fn = void (*)(const uint2*, float*, uint32_t, const uint4*, uint32_t, const uint4*, uint32_t, float*);
struct LevelLaunch {
    LevelFn lvl = nullptr;
    RowsFn rows = nullptr;
    WarpRowsFn warp_rows = nullptr;    // batch 1: one warp per row
    WarpRows4Fn warp_rows4 = nullptr;  // batch 4..32: one warp per row (and segment)
    uint32_t lanes = 1;
    uint32_t tiles = 1;
};

// Batch 1: a warp per row (k_warp_rows) unless ASNN_WARP_ROWS=0.
bool warp_rows_enabled() {
    static const bool on = [] {
        const char* s = getenv("ASNN_WARP_ROWS");
        return !(s && s[0] == '0');
    }();
    return on;
}

// ASNN_LEVEL_VARIANT (tuning experiments; profiles/r1_level_variants.txt,
// profiles/r1_light_variants.txt): 5 = k_rows, 8 gathers in flight, 4
// blocks/SM (the default); 6/7/8 = k_rows with 8/12/16 in flight at 3/3/2
// blocks/SM; 0..4 = k_level (8 in flight unconstrained, 8 at 4 blocks/SM,
// 16 at 2, 16 at 3, 4 at 6).
int level_variant() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("ASNN_LEVEL_VARIANT");
        v = s ? atoi(s) : 5;
    }
    return v;
}

template <int LANES>
LevelLaunch wide_level(uint32_t tiles) {
    LevelLaunch l;
    l.lanes = LANES;
    l.tiles = tiles;
    switch (level_variant()) {
        case 0: l.lvl = k_level<4, LANES, 8, 1>; break;
        case 1: l.lvl = k_level<4, LANES, 8, 4>; break;
        case 2: l.lvl = k_level<4, LANES, 16, 2>; break;
        case 3: l.lvl = k_level<4, LANES, 16, 3>; break;
        case 4: l.lvl = k_level<4, LANES, 4, 6>; break;
        case 6: l.rows = k_rows<LANES, 8, 3>; break;
        case 7: l.rows = k_rows<LANES, 12, 3>; break;
        case 8: l.rows = k_rows<LANES, 16, 2>; break;
        case 9: l.rows = k_rows_cp<LANES, 8, 5>; break;
        case 10: l.rows = k_rows_cp<LANES, 6, 6>; break;
        case 11: l.rows = k_rows_cp<LANES, 12, 4>; break;
        case 12: l.rows = k_rows_cp<LANES, 4, 8>; break;
        default: l.rows = k_rows<LANES, 8, 4>; break;
    }
    return l;
}

// Batches of 4..32 columns (the per-GPU slice of a batch sharded over many
// GPUs): k_rows with 16 gathers in flight per lane at 2 blocks/SM -- narrow
// rows need more memory-level parallelism per row.  Config 4's 16- / 8-column
// shards: 9.6 / 9.4 ms, against 12.7 / 11.6 ms with 8 in flight and 13.0 ms
// (8 columns) for one warp per row (k_warp_rows4, ASNN_NARROW_WARP=1).
// ASNN_LEVEL_VARIANT overrides as for wide batches.
template <int LANES>
LevelLaunch narrow_level() {
    static const bool warp = [] {
        const char* s = getenv("ASNN_NARROW_WARP");
        return s && s[0] == '1';
    }();
    if (!warp) {
        if (getenv("ASNN_LEVEL_VARIANT")) return wide_level<LANES>(1);
        LevelLaunch l;
        l.rows = k_rows<LANES, 16, 2>;
        l.lanes = LANES;
        l.tiles = 1;
        return l;
    }
    LevelLaunch l;
    l.warp_rows4 = k_warp_rows4<LANES>;
    l.lanes = 32;
    l.tiles = 1;
    return l;
}

// Programmatic dependent launch between consecutive k_rows levels: the next
// level's blocks are scheduled while the current one drains (config 2: 2.03
// -> 1.97 ms; config 4 unchanged).  ASNN_PDL=0 disables.
bool pdl_enabled() {
    static const bool on = [] {
        const char* s = getenv("ASNN_PDL");
        return !(s && s[0] == '0');
    }();
    return on;
}

LevelLaunch level_launch_for(uint32_t ldA) {
    switch (ldA) {
        case 1: return warp_rows_enabled() ? LevelLaunch{nullptr, nullptr, k_warp_rows, nullptr, 32, 1}
                                           : LevelLaunch{k_level<1, 1>, nullptr, nullptr, nullptr, 1, 1};
        case 2: return {k_level<2, 1>, nullptr, nullptr, nullptr, 1, 1};
        case 4: return narrow_level<1>();
        case 8: return narrow_level<2>();
        case 16: return narrow_level<4>();
        case 32: return narrow_level<8>();
        case 64: return wide_level<16>(1);
        default: return wide_level<32>(ldA / 128);
    }
}

struct HeavyLaunch {
    void (*fn)(const uint32_t*, const uint2*, float*, uint32_t, const uint32_t*, uint32_t, const uint4*, float*);
    uint32_t threads;
    uint32_t smem;
    uint32_t tiles;
};

template <int TC>
HeavyLaunch heavy_launch() {
    const uint32_t smem = heavy::kStages * heavy::kRows * (TC + 1) * 4 + 2 * heavy::kStages * 8;
    // the attribute is per device: remember which ordinals are configured
    static std::atomic<uint64_t> configured{0};
    int device = 0;
    cudaGetDevice(&device);
    const uint64_t bit = 1ull << (device & 63);
    if (!(configured.load() & bit)) {
        cudaFuncSetAttribute(k_heavy<TC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        configured.fetch_or(bit);
    }
    return {k_heavy<TC>, 32u * heavy::kProducers + (TC < 32 ? 32u : static_cast<uint32_t>(TC)), smem, 1};
}

// Rows must be >= 16 bytes for a bulk copy: no heavy path below 4 columns.
HeavyLaunch heavy_launch_for(uint32_t ldA) {
    switch (ldA) {
        case 1:
        case 2: return {nullptr, 0, 0, 0};
        case 4: return heavy_launch<4>();
        case 8: return heavy_launch<8>();
        case 16: return heavy_launch<16>();
        case 32: return heavy_launch<32>();
        case 64: return heavy_launch<64>();
        default: {
            HeavyLaunch h = heavy_launch<128>();
            h.tiles = ldA / 128;
            return h;
        }
    }
}

// Index into heavy_thr() of the smallest listed threshold >= `want` (an
// in-degree), or -1 when the heavy path is off.
int heavy_index_for(uint32_t want) {
    for (int t = 0; t < kNumHeavyThr; ++t)
        if (heavy_thr(t) >= want) return heavy_thr(t) == 0xFFFFFFFFu ? -1 : t;
    return -1;
}

// Default: ASNN_HEAVY_THRESHOLD (an in-degree, or "off"), else 512.
uint32_t default_heavy_threshold() {
    const char* s = getenv("ASNN_HEAVY_THRESHOLD");
    if (s && std::string(s) == "off") return 0xFFFFFFFFu;
    if (s) return static_cast<uint32_t>(strtoul(s, nullptr, 10));
    return 512;
}

// K-cta launch plan for a padded batch width: the largest power-of-two column
// slice whose activations (plus the staged edge buffers) fit in shared memory.
struct CtaPlan {
    bool use = false;
    uint32_t C = 0, V = 1, T = 32, smem = 0, ring_bytes = 0;
    bool pipe = false;        // two consumer groups: finish layer l | prefix of layer l+1
    uint32_t max_items = 0;   // items (node x column group) of the widest layer
    bool global = false;  // activations in A (L2) instead of shared memory
    bool win = false;     // ring of the newest positions in shared memory + A (cta.cuh Win)
    uint32_t win_mask = 0;
    uint32_t stg_edges = 0;  // WIN + pipe: staged prefix sources per layer (0 = direct loads)
    uint32_t chain_nf = 0;   // K-chain (chain.cuh): finish warps (0 = not used)
    bool chain_win = false;  // K-chain with a ring of the newest positions (WIN)
};

// K-chain's prefix groups for NF-warp finish groups: two finish groups + NP
// prefix groups + the producer warp within the 544-thread bound, at most four
// (prefix depth D = NP - 1 <= 3).
constexpr uint32_t chain_np(uint32_t nf) { return nf == 1 ? 8u : nf == 2 ? 4u : nf == 3 ? 3u : 2u; }

constexpr uint32_t kMaxDynSmem = 227 * 1024;

// K-chain staging groups take about 1/6 of the ring each: a handful in flight.
uint32_t chain_group_target(const CtaPlan& p) {
    static const uint32_t div = [] {  // experiments: ASNN_CHAIN_GROUP_DIV (ring / div per group)
        const char* s = getenv("ASNN_CHAIN_GROUP_DIV");
        return s ? std::max(1, atoi(s)) : 6;
    }();
    return std::max<uint32_t>(256, p.ring_bytes / div);
}

// ASNN_CTA_DEBUG (timing experiments only): 2 = no layer staging (read row
// pointers and edges from global memory).
int cta_debug_flags() {
    static int f = -1;
    if (f < 0) {
        const char* s = getenv("ASNN_CTA_DEBUG");
        f = s ? (atoi(s) & 2) : 0;
    }
    return f;
}

CtaPlan cta_plan(const asnn_dev_layout* L, uint32_t ldA) {
    CtaPlan p;
    const uint32_t mode = L->dev->sweep_mode;  // 0 auto, 1/3 layer launches, 2 K-cta when it fits
    if (mode == 1 || mode == 3) return p;
    if (L->n_levels < 2 || L->max_pos == 0) return p;
    // bytes of the largest layer's staged row pointers + edges (16-byte
    // aligned bulk copies: up to 3 / 1 extra leading entries)
    const uint64_t max_layer =
        2 * (((std::min<uint64_t>(L->max_width, 1u << 20) + 1 + 3) * 4 + 15) / 16 * 16) +
        ((std::min<uint64_t>(L->max_level_edges, 1u << 20) + 1) * 8 + 15) / 16 * 16;
    const uint64_t per_sm = 228ull * 1024;
    static const uint32_t cmax_env = [] {
        const char* s = getenv("ASNN_CTA_CMAX");
        return s ? static_cast<uint32_t>(std::max(1, atoi(s))) : 128u;
    }();
    const uint32_t cmax = std::min<uint32_t>(std::min<uint32_t>(ldA, 128), cmax_env);
    // Pipelined consumers (finish group + prefix group) for latency-bound
    // layers of <= 512 items; off with ASNN_CTA_PIPE=0.
    const char* pe = getenv("ASNN_CTA_PIPE");
    const bool want_pipe = !(pe && pe[0] == '0');
    // K-chain (chain.cuh) for one-column-per-item slices of <= 4 warps of
    // items per layer; off with ASNN_CTA_CHAIN=0 (the pipelined K-cta runs).
    static const bool want_chain = [] {
        const char* s = getenv("ASNN_CTA_CHAIN");
        return !(s && s[0] == '0');
    }();
    for (uint32_t C = cmax; C >= 1; C >>= 1) {
        if (ldA % C) continue;
        // activations (+ the zero row) | ring | mbarriers + metas | pipelined
        // consumers' partial sums (2 x items x (V + 1) words)
        const uint64_t as_bytes = (static_cast<uint64_t>(L->max_pos + 1) * C + 3) / 4 * 16;
        const uint64_t vq = C >= 4 ? 4 : 1;
        const uint64_t items_c = static_cast<uint64_t>(L->max_width) * (C / vq);
        const uint64_t nf = want_chain && want_pipe && vq == 1 && items_c <= 128 ? (items_c + 31) / 32 : 0;
        const uint64_t pipe_c = nf ? chain::tail_bytes(static_cast<uint32_t>(nf), chain_np(static_cast<uint32_t>(nf))) -
                                         cta::kMetaBytes
                                   : want_pipe && items_c <= 512 ? 2 * items_c * (vq + 1) * 4 : 0;
        const uint64_t fixed = as_bytes + cta::kMetaBytes + pipe_c;
        if (fixed + 1024 > kMaxDynSmem) {
            if (C == 1) break;
            continue;
        }
        // the ring: up to 32 of the largest layers, within what keeps the
        // CTAs-per-SM the activations alone allow; at least 2 layers when that
        // leaves too little, else whatever remains (big layers read global)
        const uint64_t want = 32 * max_layer;
        // a launch of at most one CTA per SM (a single small network) takes
        // all of the shared memory for its ring
        const uint64_t ctas = static_cast<uint64_t>(ldA / C) * L->nets.size();
        const uint64_t fit = ctas <= static_cast<uint64_t>(L->dev->sm_count)
                                 ? 1
                                 : std::max<uint64_t>(1, per_sm / (fixed + 1024 + std::min<uint64_t>(want, 4096)));
        const uint64_t budget = std::min<uint64_t>(kMaxDynSmem, per_sm / fit - 1024);
        uint64_t ring = budget > fixed ? budget - fixed : 0;
        if (ring < 2 * max_layer) ring = std::min<uint64_t>(2 * max_layer, kMaxDynSmem - fixed);
        ring = std::min(ring, want) / 16 * 16;
        p.C = C;
        p.ring_bytes = static_cast<uint32_t>(std::max<uint64_t>(ring, 16));
        p.smem = static_cast<uint32_t>(fixed + p.ring_bytes);
        p.pipe = pipe_c > 0 && !nf;
        p.chain_nf = static_cast<uint32_t>(nf);
        break;
    }
    // Global (L2-resident) variant for one network whose shared-memory slices
    // would need more than one wave of CTAs: C columns per CTA with the
    // activations in A (which must fit in L2), so ldA / C <= #SMs.
    const uint64_t a_bytes = (static_cast<uint64_t>(L->total_pos) + 1) * ldA * 4;
    const uint32_t sms = static_cast<uint32_t>(L->dev->sm_count);
    const uint64_t smem_waves =
        p.C ? (static_cast<uint64_t>(ldA / p.C) * L->nets.size() +
               sms * std::max<uint64_t>(1, (228ull * 1024) / (p.smem + 1024)) - 1) /
                  (sms * std::max<uint64_t>(1, (228ull * 1024) / (p.smem + 1024)))
             : ~0ull;
    // Off by default: on C3 it measured 5.6 ms against 4.2 ms for the two
    // shared-memory waves (profiles/r1_cta_modes.txt); ASNN_CTA_GLOBAL=1 enables.
    static const bool want_global = [] {
        const char* s = getenv("ASNN_CTA_GLOBAL");
        return s && s[0] == '1';
    }();
    // Windowed variant (cta.cuh Win): a deep network whose whole-slice CTAs
    // would need more than one wave (C3: 256 one-column CTAs of 232 KB, two
    // waves) runs one wave at two CTAs per SM, each keeping only the newest W
    // positions in shared memory and reading older sources from A in L2.
    // ASNN_CTA_WIN=0 disables.
    // Off by default: on C3 it measured 5.7 ms against 2.68 ms for the two
    // shared-memory waves (profiles/r2_c3_window.txt).  ASNN_CTA_WIN=1 enables.
    static const bool want_win = [] {
        const char* s = getenv("ASNN_CTA_WIN");
        return s && s[0] == '1';
    }();
    // Sweep mode 4 (tests): the windowed variant with the smallest legal ring
    // (W >= 2 x the widest layer: a layer's writes never share a slot).
    const bool force_win = mode == 4 && L->nets.size() == 1;
    if (force_win ||
        (want_win && !want_global && L->nets.size() == 1 && smem_waves > 1 && a_bytes <= (96ull << 20))) {
        uint32_t C = 1;
        while (ldA / C > 2 * sms && C < 128) C <<= 1;
        const uint64_t items_c = static_cast<uint64_t>(L->max_width) * C;
        // pipelined consumers + (ASNN_CTA_STAGE=0 disables) the prefix group's
        // staged out-of-ring sources, 2 x the largest layer's edges x C floats
        static const bool want_stage = [] {
            const char* s = getenv("ASNN_CTA_STAGE");
            return !(s && s[0] == '0');
        }();
        const uint64_t stg_c = want_stage && static_cast<uint64_t>(L->max_level_edges) * C * 8 <= 32 * 1024
                                   ? static_cast<uint64_t>(L->max_level_edges) * C * 8 : 0;
        const uint64_t pipe_c = want_pipe && items_c <= 512 ? 2 * items_c * 2 * 4 + stg_c : 0;
        const uint64_t budget = per_sm / 2 - 1024;
        uint64_t ring = std::min<uint64_t>(std::max<uint64_t>(2 * max_layer, 24 * 1024), 32 * max_layer) / 16 * 16;
        uint64_t W = 1;
        if (force_win) {
            while (W < std::max<uint64_t>(32, 2 * static_cast<uint64_t>(L->max_width))) W *= 2;
            // whatever shared memory the ring of positions leaves (layers larger
            // than the staging ring are read from global memory)
            const uint64_t wb = ((W + 1) * C * 4 + 15) / 16 * 16;
            const uint64_t room = kMaxDynSmem > cta::kMetaBytes + pipe_c + wb + 1024
                                      ? kMaxDynSmem - cta::kMetaBytes - pipe_c - wb - 1024 : 0;
            ring = std::max<uint64_t>(16, std::min(ring, room) / 16 * 16);
        }
        static const int w_log2 = [] {
            const char* s = getenv("ASNN_CTA_WIN_LOG2");  // experiments: fixed ring size
            return s ? atoi(s) : 0;
        }();
        const uint64_t fixed = cta::kMetaBytes + pipe_c + ring;
        if (!force_win) {
            if (w_log2 > 0) W = 1ull << w_log2;
            else
                while (fixed + ((2 * W + 1) * C * 4 + 15) / 16 * 16 <= budget) W *= 2;
        }
        if (force_win ||
            (ring >= 2 * max_layer && W >= 4 * static_cast<uint64_t>(L->max_width) && W < L->max_pos)) {
            p.C = C;
            p.chain_nf = 0;
            p.win = true;
            p.win_mask = static_cast<uint32_t>(W - 1);
            p.stg_edges = pipe_c && stg_c ? L->max_level_edges : 0;
            p.ring_bytes = static_cast<uint32_t>(ring);
            p.smem = static_cast<uint32_t>(fixed + ((W + 1) * C * 4 + 15) / 16 * 16);
            p.pipe = pipe_c > 0;
        }
    }
    // Windowed K-chain (chain.cuh WIN): a deep, narrow network whose
    // one-column slices need more than one wave (config 3: 256 CTAs of
    // 232 KB, two waves) runs one wave at two CTAs per SM, each keeping the
    // newest W positions in shared memory and writing every activation
    // through to A (which must sit in L2).  Opt-in (ASNN_CHAIN_WIN=1; sweep
    // mode 5 forces it for the tests): on config 3 it measured 1.23 ms
    // against 0.88 ms for the two full-slice waves -- the prefix warps' L2
    // round trips and two CTAs' warps per SM stretch the per-layer chain from
    // ~430 to ~1200 cycles (profiles/r2_c3_chain_window.txt).
    static const bool want_chain_win = [] {
        const char* s = getenv("ASNN_CHAIN_WIN");
        return s && s[0] == '1';
    }();
    const bool force_cwin = mode == 5 && L->nets.size() == 1 && want_chain;
    if ((force_cwin || (want_chain_win && p.chain_nf && smem_waves > 1)) && L->nets.size() == 1 &&
        a_bytes <= (96ull << 20) && L->max_width <= 128) {
        // the fewest columns per CTA that still fill a wave of two CTAs per SM
        uint32_t C = 1;
        while (ldA / C > 2 * sms && C < 2 && ldA % (2 * C) == 0) C <<= 1;
        const uint64_t items_c = static_cast<uint64_t>(L->max_width) * C;
        if (items_c <= 128) {
            const uint32_t nf = static_cast<uint32_t>((items_c + 31) / 32), np = chain_np(nf);
            const uint64_t D = np - 1;
            uint64_t W = 64;
            while (W < 2 * (D + 2) * static_cast<uint64_t>(L->max_width)) W *= 2;
            const uint64_t wb = (W * C * 4 + 15) / 16 * 16;
            const uint64_t tail = chain::tail_bytes(nf, np);
            static const uint64_t cps = [] {  // experiments: CTAs per SM the ring is sized for
                const char* s = getenv("ASNN_CHAIN_WIN_CTAS");
                return static_cast<uint64_t>(s ? std::max(1, atoi(s)) : 2);
            }();
            const uint64_t budget = std::min<uint64_t>(kMaxDynSmem, per_sm / cps - 1024);
            const uint64_t ring = budget > wb + tail ? std::min<uint64_t>(budget - wb - tail, 32 * max_layer) / 16 * 16
                                                     : 0;
            if (ring >= 2 * max_layer || (force_cwin && ring >= 1024)) {
                p.C = C;
                p.chain_nf = nf;
                p.chain_win = true;
                p.win = false;
                p.pipe = false;
                p.global = false;
                p.win_mask = static_cast<uint32_t>(W - 1);
                p.ring_bytes = static_cast<uint32_t>(ring);
                p.smem = static_cast<uint32_t>(wb + tail + ring);
            }
        }
    }
    if (want_global && L->nets.size() == 1 && !p.chain_win && smem_waves > 1 && a_bytes <= (96ull << 20) &&
        !L->zero_refs) {
        uint32_t C = 1;
        while (ldA / C > sms && C < 128) C <<= 1;
        p.C = C;
        p.chain_nf = 0;
        p.global = true;
        p.ring_bytes = static_cast<uint32_t>(
            std::min<uint64_t>(32 * max_layer, kMaxDynSmem - cta::kMetaBytes) / 16 * 16);
        p.smem = p.ring_bytes + cta::kMetaBytes;
    }
    if (!p.C) return p;
    p.V = p.C >= 4 && !p.win ? 4 : 1;
    const uint64_t items = static_cast<uint64_t>(L->max_width) * (p.C / p.V);
    // consumer threads per CTA: up to 512 (+ the producer warp).  Config 5
    // (1024 column-group items per layer, 2 CTAs/SM): 256 -> 0.90 ms, 512 ->
    // 0.73 ms -- more warps to hide the FP64 sigmoid chains; 768 drops to one
    // CTA per SM (1.14 ms).  ASNN_CTA_TMAX overrides (<= 512, the launch bound).
    static const uint64_t tmax = [] {
        const char* s = getenv("ASNN_CTA_TMAX");
        return s ? std::min<uint64_t>(512, std::max(32, atoi(s)) / 32 * 32) : 512;
    }();
    p.T = static_cast<uint32_t>(std::min<uint64_t>(tmax, std::max<uint64_t>(32, (items + 31) / 32 * 32)));
    if (p.global) p.pipe = false;
    if (p.chain_nf) p.T = 32 * p.chain_nf * (2 + chain_np(p.chain_nf));
    if (p.pipe) {  // finish group + prefix group of up to 8 warps each (one row per
                   // thread up to 256 items: config 1's ~200-row layers, ASNN_CTA_PIPE_MAX)
        static const uint64_t gmax = [] {
            const char* s = getenv("ASNN_CTA_PIPE_MAX");
            return s ? std::min<uint64_t>(256, std::max(32, atoi(s)) / 32 * 32) : 256;
        }();
        p.max_items = static_cast<uint32_t>(items);
        p.T = 2 * static_cast<uint32_t>(std::min<uint64_t>(gmax, (items + 31) / 32 * 32));
    }
    const bool latency_bound = L->nets.size() > 1 || L->n_levels >= 24 ||
                               L->total_edges * static_cast<uint64_t>(ldA) <= (1ull << 22);
    // ... unless a few CTAs would carry a big network alone.  Batch-1
    // measurements (tools/level_probe.py, reference bench corpus): one CTA
    // costs ~1.2 us per layer plus ~0.9 ns per edge-column, a per-level launch
    // over the whole GPU ~7 us per level (57k edges / 10 layers: 54 vs 76 us;
    // 110k edges: 152 vs 75 us).
    const uint64_t ctas = static_cast<uint64_t>(ldA / p.C) * L->nets.size();
    const uint64_t per_wave = static_cast<uint64_t>(L->dev->sm_count) *
                              std::max<uint64_t>(1, (228ull * 1024) / (p.smem + 1024));
    const double cta_us = (1.2 * L->n_levels + static_cast<double>(L->total_edges) / L->nets.size() * p.C / 1100.0) *
                          static_cast<double>((ctas + per_wave - 1) / per_wave);
    const double level_us = 7.0 * L->n_levels;
    p.use = mode == 2 || force_win || (force_cwin && p.chain_win) || (latency_bound && (L->nets.size() > 1 || cta_us <= level_us));
    return p;
}

}  // namespace

// ---------------------------------------------------------------------------
namespace asnn_b200 {

namespace staging {
constexpr size_t kStageChunk = 8u << 20;

void par_memcpy(void* d, const void* s, size_t n) {
    // OpenMP's pool (libgomp is linked for the generators): no per-call thread start
    const int T = static_cast<int>(std::max<size_t>(1, std::min<size_t>(8, n >> 20)));
    const size_t part = ((n + T - 1) / T + 4095) & ~size_t(4095);
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) {
        const size_t a = static_cast<size_t>(t) * part;
        if (a < n) std::memcpy(static_cast<char*>(d) + a, static_cast<const char*>(s) + a, std::min(part, n - a));
    }
}

bool page_locked(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type != cudaMemoryTypeUnregistered;
}

cudaError_t ensure_stage(asnn_dev* dev) {
    for (int b = 0; b < 2; ++b) {
        cudaError_t e = dev->stage[b].ensure(kStageChunk);
        if (e != cudaSuccess) return e;
        if (!dev->stage_ev[b]) {
            e = cudaEventCreateWithFlags(&dev->stage_ev[b], cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}
}  // namespace staging

using namespace staging;

cudaError_t upload_host(asnn_dev* dev, void* dst, const void* src, size_t len, cudaStream_t st) {
    if (len < 2 * kStageChunk || page_locked(src))
        return len ? cudaMemcpyAsync(dst, src, len, cudaMemcpyHostToDevice, st) : cudaSuccess;
    cudaError_t e = ensure_stage(dev);
    if (e != cudaSuccess) return e;
    for (size_t off = 0, i = 0; off < len; off += kStageChunk, ++i) {
        const size_t n = std::min(kStageChunk, len - off);
        const int b = static_cast<int>(i & 1);
        if ((e = cudaEventSynchronize(dev->stage_ev[b])) != cudaSuccess) return e;  // its last DMA done
        par_memcpy(dev->stage[b].p, static_cast<const char*>(src) + off, n);
        if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, dev->stage[b].p, n, cudaMemcpyHostToDevice, st)) !=
            cudaSuccess)
            return e;
        if ((e = cudaEventRecord(dev->stage_ev[b], st)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t h2d(asnn_dev* dev, void* dst, const void* src, size_t len, cudaStream_t st) {
    if (!len) return cudaSuccess;
    const size_t at = (dev->arena_used + 255) & ~size_t(255);
    if (at + len <= dev->arena.bytes) {  // small: one host memcpy beats a pointer-attribute query
        std::memcpy(static_cast<char*>(dev->arena.p) + at, src, len);
        dev->arena_used = at + len;
        return cudaMemcpyAsync(dst, static_cast<char*>(dev->arena.p) + at, len, cudaMemcpyHostToDevice, st);
    }
    return upload_host(dev, dst, src, len, st);
}

cudaError_t download_host(asnn_dev* dev, void* dst, const void* src, size_t len, cudaStream_t st) {
    if (len < 2 * kStageChunk || page_locked(dst))  // stream-ordered, as the caller expects
        return len ? cudaMemcpyAsync(dst, src, len, cudaMemcpyDeviceToHost, st) : cudaSuccess;
    cudaError_t e = ensure_stage(dev);
    if (e != cudaSuccess) return e;
    const size_t chunks = (len + kStageChunk - 1) / kStageChunk;
    for (size_t i = 0; i <= chunks; ++i) {
        if (i < chunks) {  // DMA of chunk i into stage[i & 1] (chunk i - 2 was copied out already)
            const size_t off = i * kStageChunk, n = std::min(kStageChunk, len - off);
            const int b = static_cast<int>(i & 1);
            if ((e = cudaEventSynchronize(dev->stage_ev[b])) != cudaSuccess) return e;
            if ((e = cudaMemcpyAsync(dev->stage[b].p, static_cast<const char*>(src) + off, n,
                                     cudaMemcpyDeviceToHost, st)) != cudaSuccess)
                return e;
            if ((e = cudaEventRecord(dev->stage_ev[b], st)) != cudaSuccess) return e;
        }
        if (i >= 1) {  // host copy of chunk i - 1 while chunk i is in flight
            const size_t j = i - 1, off = j * kStageChunk, n = std::min(kStageChunk, len - off);
            const int b = static_cast<int>(j & 1);
            if ((e = cudaEventSynchronize(dev->stage_ev[b])) != cudaSuccess) return e;
            par_memcpy(static_cast<char*>(dst) + off, dev->stage[b].p, n);
        }
    }
    return cudaSuccess;
}

int assemble_layout(asnn_dev* dev, std::vector<NetMeta>&& nets, FlatDevice&& flat,
                    asnn_dev_layout** result) {
    const uint32_t G = static_cast<uint32_t>(nets.size());
    if (G == 0) return fail(dev, ASNN_E_INVALID, "layout without networks");
    auto* L = new asnn_dev_layout;
    L->dev = dev;
    std::vector<uint32_t> meta(6 * (G + 1), 0);
    uint64_t E = 0;
    for (uint32_t g = 0; g < G; ++g) {
        NetMeta& n = nets[g];
        n.pos_base = meta[0 * (G + 1) + g];
        n.idb_prefix = meta[1 * (G + 1) + g];
        n.in_prefix = meta[2 * (G + 1) + g];
        n.out_prefix = meta[3 * (G + 1) + g];
        n.edge_base = E;
        meta[0 * (G + 1) + g + 1] = n.pos_base + n.n_pos;
        meta[1 * (G + 1) + g + 1] = n.idb_prefix + n.id_bound;
        meta[2 * (G + 1) + g + 1] = n.in_prefix + n.n_in;
        meta[3 * (G + 1) + g + 1] = n.out_prefix + n.n_out;
        meta[4 * (G + 1) + g] = static_cast<uint32_t>(E);
        E += n.n_edges;
        meta[4 * (G + 1) + g + 1] = static_cast<uint32_t>(E);
        meta[5 * (G + 1) + g + 1] = meta[5 * (G + 1) + g] + n.n_sensors;
        L->dropped += n.dropped;
    }
    if (E >= 0xFFFFFFFFull) {
        delete L;
        return fail(dev, ASNN_E_INVALID, "more than 2^32-1 stored edges");
    }

    L->total_pos = meta[0 * (G + 1) + G];
    L->total_idb = meta[1 * (G + 1) + G];
    L->total_in = meta[2 * (G + 1) + G];
    L->total_out = meta[3 * (G + 1) + G];
    L->total_sensors = meta[5 * (G + 1) + G];
    L->total_edges = E;
    cudaStream_t st = dev->stream;

    auto cleanup_fail = [&](int rc) {
        delete L;
        return rc;
    };
    DevBuf<uint32_t> d_meta;
    DevBuf<uint32_t> bad, kofid, maxdeg;
    cudaError_t e;
#define CKL(expr)                                                      \
    do {                                                               \
        e = (expr);                                                    \
        if (e != cudaSuccess) return cleanup_fail(cuda_fail(dev, e, #expr)); \
    } while (0)
    CKL(d_meta.alloc(meta.size()));
    CKL(h2d(dev, d_meta.p, meta.data(), meta.size() * 4, st));
    MetaPtrs m{d_meta.p, d_meta.p + (G + 1), d_meta.p + 2 * (G + 1), d_meta.p + 3 * (G + 1),
               d_meta.p + 4 * (G + 1), d_meta.p + 5 * (G + 1), G};
    CKL(bad.alloc(2));
    CKL(cudaMemsetAsync(bad.p, 0, 8, st));
    CKL(L->state_map.alloc(L->total_idb));
    CKL(cudaMemsetAsync(L->state_map.p, 0xFF, static_cast<size_t>(L->total_idb) * 4, st));
    if (L->total_pos)
        k_state_map<<<blocks_for(L->total_pos), kThreads, 0, st>>>(m, flat.node_ids.p, L->total_pos,
                                                                   L->state_map.p, bad.p);
    CKL(L->edges.alloc(E + 2));  // +2: K-cta bulk copies round up to 16 bytes
    if (E)
        k_edges<<<blocks_for(E), kThreads, 0, st>>>(m, flat.in_ids.p, flat.w.p, E, L->state_map.p,
                                                   L->total_pos, L->edges.p, bad.p);
    CKL(kofid.alloc(L->total_idb));
    CKL(cudaMemsetAsync(kofid.p, 0, static_cast<size_t>(L->total_idb) * 4, st));
    if (L->total_in)
        k_input_index<<<blocks_for(L->total_in), kThreads, 0, st>>>(m, flat.inputs.p, L->total_in,
                                                                    kofid.p, bad.p);
    CKL(L->sinfo.alloc(L->total_sensors));
    if (L->total_sensors)
        k_sinfo<<<blocks_for(L->total_sensors), kThreads, 0, st>>>(m, flat.node_ids.p, kofid.p,
                                                                   L->total_sensors, L->sinfo.p);
    CKL(L->oinfo.alloc(L->total_out));
    if (L->total_out)
        k_oinfo<<<blocks_for(L->total_out), kThreads, 0, st>>>(m, flat.outputs.p, L->total_out,
                                                               L->state_map.p, L->oinfo.p);
    CKL(maxdeg.alloc(1));
    CKL(cudaMemsetAsync(maxdeg.p, 0, 4, st));
    if (L->total_pos)
        k_max_deg<<<blocks_for(L->total_pos), kThreads, 0, st>>>(flat.row_ptr.p, L->total_pos,
                                                                 maxdeg.p);
    CKL(cudaGetLastError());

    // Level-major schedule: global level l runs layer l of every network, its
    // positions ordered by in-degree descending (longest rows first, LPT),
    // ties by position.  A stable radix sort of all positions by
    // (level, ~degree); level-0 sensors sort first and are skipped.
    std::vector<uint32_t> le_host, lo_base_host;
    uint32_t n_levels = 0;
    for (const auto& n : nets) n_levels = std::max(n_levels, n.n_layers);
    L->n_levels = n_levels;
    L->lvl_off.assign(n_levels + 1, 0);
    {
        std::vector<uint32_t> lvl_count(n_levels + 1, 0), lo_cat, lo_base(G + 1, 0);
        for (uint32_t g = 0; g < G; ++g) {
            const auto& n = nets[g];
            for (uint32_t l = 0; l < n.n_layers; ++l) {
                const uint32_t c = n.layer_offsets[l + 1] - n.layer_offsets[l];
                lvl_count[l] += c;
                L->max_width = std::max(L->max_width, c);
            }
            lo_base[g + 1] = lo_base[g] + n.n_layers + 1;
            lo_cat.insert(lo_cat.end(), n.layer_offsets.begin(), n.layer_offsets.end());
        }
        uint32_t acc = 0;
        for (uint32_t l = 1; l < n_levels; ++l) {
            L->lvl_off[l] = acc;
            acc += lvl_count[l];
        }
        if (n_levels) L->lvl_off[n_levels] = acc;
        const uint32_t P = L->total_pos;
        DevBuf<uint32_t> d_lo, d_lob;
        CKL(d_lo.alloc(lo_cat.size()));
        CKL(d_lob.alloc(G + 1));
        if (!lo_cat.empty())
            CKL(h2d(dev, d_lo.p, lo_cat.data(), lo_cat.size() * 4, st));
        CKL(h2d(dev, d_lob.p, lo_base.data(), (G + 1) * 4, st));
        (void)P;
        // K-cta metadata: per-network records and layer boundaries as edge offsets
        std::vector<uint32_t> recs(static_cast<size_t>(G) * 12, 0);
        uint32_t sens = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const NetMeta& n = nets[g];
            uint32_t* r = &recs[static_cast<size_t>(g) * 12];
            r[0] = n.pos_base;
            r[1] = n.n_pos;
            r[2] = n.n_sensors;
            r[3] = sens;
            r[4] = n.in_prefix;
            r[5] = n.n_in;
            r[6] = n.out_prefix;
            r[7] = n.n_out;
            r[8] = lo_base[g];
            r[9] = n.n_layers;
            sens += n.n_sensors;
            L->max_pos = std::max(L->max_pos, n.n_pos);
        }
        CKL(L->cta_nets.alloc(recs.size()));
        CKL(h2d(dev, L->cta_nets.p, recs.data(), recs.size() * 4, st));
        CKL(L->le_cat.alloc(lo_cat.size() + 1));
        if (!lo_cat.empty())
            k_layer_edges<<<blocks_for(lo_cat.size()), kThreads, 0, st>>>(
                d_lo.p, d_lob.p, G, m.pos, flat.row_ptr.p, static_cast<uint32_t>(lo_cat.size()),
                L->le_cat.p);
        CKL(cudaGetLastError());
        le_host.resize(lo_cat.size());
        lo_base_host = lo_base;
        if (!le_host.empty())
            CKL(cudaMemcpyAsync(le_host.data(), L->le_cat.p, le_host.size() * 4, cudaMemcpyDeviceToHost, st));
        L->lo_cat = std::move(d_lo);
        L->lo_base = std::move(d_lob);
    }
    CKL(L->idb_prefix.alloc(G + 1));
    CKL(cudaMemcpyAsync(L->idb_prefix.p, d_meta.p + (G + 1), (G + 1) * 4, cudaMemcpyDeviceToDevice,
                        st));
    uint32_t h_bad[2] = {0, 0};
    CKL(cudaMemcpyAsync(h_bad, bad.p, 8, cudaMemcpyDeviceToHost, st));
    CKL(cudaMemcpyAsync(&L->max_deg, maxdeg.p, 4, cudaMemcpyDeviceToHost, st));
    CKL(cudaStreamSynchronize(st));  // the one synchronisation of a layout build
    arena_reset(dev);
    for (uint32_t g = 0; g < G; ++g)
        for (uint32_t l = 0; l < nets[g].n_layers; ++l)
            L->max_level_edges =
                std::max(L->max_level_edges, le_host[lo_base_host[g] + l + 1] - le_host[lo_base_host[g] + l]);
#undef CKL
    if (h_bad[0] & 7u) {
        delete L;
        return fail(dev, ASNN_E_INVALID,
                    "layout references an id >= id_bound (code " + std::to_string(h_bad[0]) + ")");
    }
    L->zero_refs = (h_bad[0] & 8u) != 0;
    L->le_host = std::move(le_host);
    L->lo_base_host = std::move(lo_base_host);
    L->d_meta = std::move(d_meta);
    L->row_ptr = std::move(flat.row_ptr);
    L->node_ids = std::move(flat.node_ids);
    L->nets = std::move(nets);
    *result = L;
    return ASNN_OK;
}

}  // namespace asnn_b200

// ---------------------------------------------------------------------------
namespace {

template <typename Mark>
int launch_levels(asnn_dev_layout* L, uint32_t ldA, cudaStream_t st, Mark& mark);

// The per-level launch schedule (built on first use: K-cta sweeps -- small,
// deep and population layouts, the per-call drop-in -- never need it).
// Level-major: global level l runs layer l of every network, its positions
// ordered by in-degree descending (longest rows first, LPT), ties by
// position -- a stable radix sort of all positions by (level, ~degree);
// level-0 sensors sort first and are skipped.  Plus the heavy-row counts
// per level for every threshold heavy_thr(t).
bool level_win_enabled() {
    static const bool on = [] {
        const char* s = getenv("ASNN_LEVEL_WIN");
        return s && s[0] == '1';
    }();
    return on;
}

int ensure_schedule(asnn_dev_layout* L) {
    if (L->sched_ready) return ASNN_OK;
    asnn_dev* dev = L->dev;
    cudaStream_t st = dev->stream;
    const uint32_t G = static_cast<uint32_t>(L->nets.size());
    const uint32_t n_levels = L->n_levels;
    const uint32_t P = L->total_pos;
    MetaPtrs m{L->d_meta.p, L->d_meta.p + (G + 1), L->d_meta.p + 2 * (G + 1), L->d_meta.p + 3 * (G + 1),
               L->d_meta.p + 4 * (G + 1), L->d_meta.p + 5 * (G + 1), G};
    DevBuf<uint32_t> keys, vals, hv;
    CK(keys.alloc(P + 1));
    CK(vals.alloc(P + 1));
    if (P)
        k_sched_keys<<<blocks_for(P), kThreads, 0, st>>>(m, L->lo_cat.p, L->lo_base.p, L->row_ptr.p, P, keys.p,
                                                         vals.p);
    CK(cudaGetLastError());
    SortBuffers sb;
    uint32_t *ks = nullptr, *vs = nullptr;
    int lb = 0;
    while ((1u << lb) < n_levels) ++lb;
    int rc = radix_sort_pairs(dev, keys.p, vals.p, P, std::max(1, lb) + 16, sb, &ks, &vs, st);
    if (rc) return rc;
    const uint32_t S = L->total_sensors;
    CK(L->sched.alloc(P - S + 1));
    if (P > S) CK(cudaMemcpyAsync(L->sched.p, vs + S, (P - S) * 4ull, cudaMemcpyDeviceToDevice, st));
    CK(L->rtask.alloc(P - S + 1));
    if (P > S) k_row_tasks<<<blocks_for(P - S), kThreads, 0, st>>>(L->sched.p, L->row_ptr.p, P - S, L->rtask.p);
    const size_t nh = static_cast<size_t>(kNumHeavyThr) * (n_levels + 1);
    CK(hv.alloc(nh));
    CK(cudaMemsetAsync(hv.p, 0, nh * 4, st));
    if (P > S) k_heavy_counts<<<blocks_for(P - S), kThreads, 0, st>>>(ks + S, P - S, n_levels + 1, hv.p);
    CK(cudaGetLastError());
    L->heavy_cnt.assign(nh, 0);
    CK(cudaMemcpyAsync(L->heavy_cnt.data(), hv.p, nh * 4, cudaMemcpyDeviceToHost, st));
    // per-level source windows (k_rows_win), one network
    DevBuf<uint32_t> d_lvl, wmin, wmax;
    L->win_lo.assign(n_levels, 0xFFFFFFFFu);
    L->win_hi.assign(n_levels, 0);
    if (level_win_enabled() && G == 1 && P > S && n_levels) {
        CK(d_lvl.alloc(n_levels + 1));
        CK(wmin.alloc(n_levels));
        CK(wmax.alloc(n_levels));
        CK(cudaMemcpyAsync(d_lvl.p, L->lvl_off.data(), (n_levels + 1) * 4ull, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(wmin.p, 0xFF, n_levels * 4ull, st));
        CK(cudaMemsetAsync(wmax.p, 0, n_levels * 4ull, st));
        k_level_windows<<<blocks_for(P - S), kThreads, 0, st>>>(L->rtask.p, d_lvl.p, n_levels, P - S, L->edges.p,
                                                                 wmin.p, wmax.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(L->win_lo.data(), wmin.p, n_levels * 4ull, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(L->win_hi.data(), wmax.p, n_levels * 4ull, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    L->sched_ready = true;
    return ASNN_OK;
}


// ---- heavy-row segments (segments.cuh) --------------------------------------
// Shortest interrupted segment and longest segment k_rows takes (longer ones
// stream through k_heavy): ASNN_SEG_MIN (default 64), ASNN_SEG_LONG (512).
uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* s = getenv(name);
    return s ? static_cast<uint32_t>(strtoul(s, nullptr, 10)) : dflt;
}

// One network, 4 columns per lane (batch 64 or a multiple of 128), a heavy
// threshold, per-level launches not restricted to whole rows (sweep mode 3),
// and not disabled (ASNN_SEGMENTS=0).
bool seg_eligible(const asnn_dev_layout* L, uint32_t ldA) {
    static const bool enabled = env_u32("ASNN_SEGMENTS", 1) != 0;
    const LevelLaunch ll = level_launch_for(ldA);
    return enabled && L->nets.size() == 1 && L->dev->sweep_mode != 3 && (ll.rows || ll.warp_rows4) &&
           heavy_launch_for(ldA).fn && heavy_index_for(L->dev->heavy_threshold) >= 0 &&
           L->total_pos > L->total_sensors;
}

uint64_t seg_key_for(const asnn_dev_layout* L) {
    return (static_cast<uint64_t>(heavy_index_for(L->dev->heavy_threshold)) << 48) ^
           (static_cast<uint64_t>(env_u32("ASNN_SEG_MIN", 64)) << 24) ^ env_u32("ASNN_SEG_LONG", 512);
}

// Splits every heavy row of the (single) network into segments by the levels
// of its sources; groups them by (short/long, step), longest first.
int ensure_segments(asnn_dev_layout* L) {
    asnn_dev* dev = L->dev;
    cudaStream_t st = dev->stream;
    {
        const int rc = ensure_schedule(L);
        if (rc) return rc;
    }
    const NetMeta& n = L->nets[0];
    const int thr = heavy_index_for(dev->heavy_threshold);
    const uint32_t NL = L->n_levels;
    std::vector<uint32_t> hv_prefix(NL + 1, 0);
    for (uint32_t l = 0; l < NL; ++l)
        hv_prefix[l + 1] = hv_prefix[l] + (l ? L->heavy_cnt[thr * (NL + 1) + l] : 0u);
    const uint32_t H = hv_prefix[NL];
    L->seg_short_off.assign(NL + 1, 0);
    L->seg_long_off.assign(NL + 1, 0);
    L->n_slots = H;
    L->seg_key = seg_key_for(L);
    L->seg.reset();
    if (!H) return ASNN_OK;
    int lb = 0;
    while ((1u << lb) <= NL) ++lb;
    DevBuf<uint32_t> d_prefix, d_lvl_off, lo, hv_level, hv_sched, count, base, keys, vals, step_count;
    DevBuf<uint4> tasks;
    CK(d_prefix.alloc(NL + 1));
    CK(d_lvl_off.alloc(NL + 1));
    CK(lo.alloc(n.layer_offsets.size()));
    CK(hv_level.alloc(H));
    CK(hv_sched.alloc(H));
    CK(count.alloc(H + 1));
    CK(base.alloc(H + 1));
    CK(step_count.alloc(2 * (n.n_layers + 1)));
    CK(cudaMemcpyAsync(d_prefix.p, hv_prefix.data(), (NL + 1) * 4ull, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_lvl_off.p, L->lvl_off.data(), (NL + 1) * 4ull, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(lo.p, n.layer_offsets.data(), n.layer_offsets.size() * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(count.p + H, 0, 4, st));
    CK(cudaMemsetAsync(step_count.p, 0, 2 * (n.n_layers + 1) * 4ull, st));
    k_heavy_rows<<<blocks_for(H), kThreads, 0, st>>>(d_prefix.p, d_lvl_off.p, NL, H, hv_level.p, hv_sched.p);
    SegArgs a{};
    a.row_ptr = L->row_ptr.p;
    a.edges = L->edges.p;
    a.lo = lo.p;
    a.nl = n.n_layers;
    a.sched = L->sched.p;
    a.hv_level = hv_level.p;
    a.hv_sched = hv_sched.p;
    a.n_heavy = H;
    a.min_len = std::max<uint32_t>(1, env_u32("ASNN_SEG_MIN", 64));
    a.long_len = env_u32("ASNN_SEG_LONG", 512);
    a.lb = static_cast<uint32_t>(lb);
    a.count = count.p;
    k_segments<0><<<blocks_for(static_cast<uint64_t>(H) * 32), kThreads, 0, st>>>(a);
    CK(cudaGetLastError());
    int rc = exclusive_scan(dev, count.p, base.p, H + 1, nullptr, st);
    if (rc) return rc;
    uint32_t total = 0;
    CK(cudaMemcpyAsync(&total, base.p + H, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(tasks.alloc(total));
    CK(keys.alloc(total));
    CK(vals.alloc(total));
    a.base = base.p;
    a.tasks = tasks.p;
    a.keys = keys.p;
    a.vals = vals.p;
    a.step_count = step_count.p;
    k_segments<1><<<blocks_for(static_cast<uint64_t>(H) * 32), kThreads, 0, st>>>(a);
    CK(cudaGetLastError());
    SortBuffers sb;
    uint32_t *ks = nullptr, *vs = nullptr;
    rc = radix_sort_pairs(dev, keys.p, vals.p, total, lb + 17, sb, &ks, &vs, st);
    if (rc) return rc;
    CK(L->seg.alloc(total));
    k_gather_tasks<<<blocks_for(total), kThreads, 0, st>>>(tasks.p, vs, total, L->seg.p);
    CK(cudaGetLastError());
    std::vector<uint32_t> sc(2 * (n.n_layers + 1));
    CK(cudaMemcpyAsync(sc.data(), step_count.p, sc.size() * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // sorted order: all short (step ascending), then all long
    uint32_t acc = 0;
    for (uint32_t l = 0; l <= NL; ++l) {
        L->seg_short_off[l] = acc;
        if (l < NL && l <= n.n_layers) acc += sc[l];
    }
    for (uint32_t l = 0; l <= NL; ++l) {
        L->seg_long_off[l] = acc;
        if (l < NL && l <= n.n_layers) acc += sc[(n.n_layers + 1) + l];
    }
    return ASNN_OK;
}

#define RC_(expr)          \
    do {                   \
        int _r = (expr);   \
        if (_r) return _r; \
    } while (0)

// One activation sweep, stream-ordered: sensors, every level, outputs, state.
int launch_sweep(asnn_dev_layout* L, const float* x, uint32_t n_vec, float* out, float* state,
                 cudaStream_t st, std::vector<cudaEvent_t>* evs = nullptr) {
    asnn_dev* dev = L->dev;
    const uint32_t ldA = padded_batch(n_vec);
    size_t ek = 0;
    auto mark = [&]() {
        if (evs && ek < evs->size()) cudaEventRecord((*evs)[ek++], st);
    };
    mark();
    const CtaPlan cp = cta_plan(L, ldA);
    // K-cta writes the declared outputs itself (shared-memory variant, no state)
    const bool cta_out = cp.use && !cp.global && !cp.win && !state && out && L->total_out;
    if (cp.use && cp.chain_nf) {
        using KC = void (*)(const CtaNet*, const uint32_t*, const uint4*, const uint32_t*, const uint4*,
                            const uint32_t*, const uint2*, const uint4*, const uint4*, const float*, uint32_t, float*,
                            uint32_t, uint32_t, uint32_t, uint32_t, int, float*, const uint32_t*, uint32_t);
        static const KC kc[2][2][4] = {
            {{k_chain<1, chain_np(1), false, false>, k_chain<2, chain_np(2), false, false>,
              k_chain<3, chain_np(3), false, false>, k_chain<4, chain_np(4), false, false>},
             {k_chain<1, chain_np(1), true, false>, k_chain<2, chain_np(2), true, false>,
              k_chain<3, chain_np(3), true, false>, k_chain<4, chain_np(4), true, false>}},
            {{k_chain<1, chain_np(1), false, true>, k_chain<2, chain_np(2), false, true>,
              k_chain<3, chain_np(3), false, true>, k_chain<4, chain_np(4), false, true>},
             {k_chain<1, chain_np(1), true, true>, k_chain<2, chain_np(2), true, true>,
              k_chain<3, chain_np(3), true, true>, k_chain<4, chain_np(4), true, true>}}};
        const KC fn = kc[cp.chain_win ? 1 : 0][L->zero_refs ? 1 : 0][cp.chain_nf - 1];
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cp.smem)));
        fn<<<dim3(ldA / cp.C, static_cast<uint32_t>(L->nets.size())), cp.T + 32, cp.smem, st>>>(
            reinterpret_cast<const CtaNet*>(L->cta_nets.p), L->lo_base.p, L->grp.p, L->grp_off.p, L->lplan.p,
            L->row_ptr.p, L->edges.p, L->sinfo.p, L->oinfo.p, x, n_vec, L->A.p, ldA, cp.C, L->max_pos,
            cp.ring_bytes, (state ? 1 : 0) | cta_debug_flags(), cta_out ? out : nullptr, L->split.p, cp.win_mask);
    } else if (cp.use) {
        // the whole sweep (sensors + every layer) of each (network, slice) in one CTA
        auto fn = cp.win ? (cp.pipe ? (L->zero_refs ? k_cta<1, true, false, true, true> : k_cta<1, false, false, true, true>)
                                    : (L->zero_refs ? k_cta<1, true, false, false, true> : k_cta<1, false, false, false, true>))
                  : cp.global ? (cp.V == 4 ? k_cta<4, false, true> : k_cta<1, false, true>)
                  : cp.pipe
                      ? (cp.V == 4 ? (L->zero_refs ? k_cta<4, true, false, true> : k_cta<4, false, false, true>)
                                   : (L->zero_refs ? k_cta<1, true, false, true> : k_cta<1, false, false, true>))
                  : cp.V == 4 ? (L->zero_refs ? k_cta<4, true, false> : k_cta<4, false, false>)
                              : (L->zero_refs ? k_cta<1, true, false> : k_cta<1, false, false>);
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(cp.smem)));
        // cp.T consumer threads + one producer warp
        fn<<<dim3(ldA / cp.C, static_cast<uint32_t>(L->nets.size())), cp.T + 32, cp.smem, st>>>(
            reinterpret_cast<const CtaNet*>(L->cta_nets.p), L->lo_cat.p, L->le_cat.p, L->row_ptr.p,
            L->edges.p, L->sinfo.p, L->oinfo.p, x, n_vec, L->A.p, ldA, cp.C, L->max_pos, cp.ring_bytes,
            (state ? 1 : 0) | cta_debug_flags(), cta_out ? out : nullptr, L->split.p, cp.max_items,
            cp.win_mask, cp.stg_edges);
    } else {
        if (L->total_sensors)
            k_sense<<<blocks_for(static_cast<uint64_t>(L->total_sensors) * ldA), kThreads, 0, st>>>(
                L->sinfo.p, L->total_sensors, x, n_vec, L->A.p, ldA);
        RC_(launch_levels(L, ldA, st, mark));
    }
    if (out && L->total_out && !cta_out) {
        mark();
        k_gather_out<<<blocks_for(static_cast<uint64_t>(L->total_out) * n_vec), kThreads, 0, st>>>(
            L->oinfo.p, L->total_out, L->A.p, ldA, n_vec, out);
    }
    mark();
    if (state && L->total_idb)
        k_state<<<blocks_for(static_cast<uint64_t>(L->total_idb) * n_vec), kThreads, 0, st>>>(
            L->state_map.p, L->idb_prefix.p, static_cast<uint32_t>(L->nets.size()), L->total_idb,
            L->A.p, ldA, n_vec, state);
    CK(cudaGetLastError());
    return ASNN_OK;
}

// Per-layer launches (k_level, plus k_heavy on the aux branch for heavy rows).
// k_rows_win (win_rows.cuh): a level of whole rows whose sources all lie in
// a window of positions small enough for shared memory (two blocks per SM),
// for batches of 128+ columns.  Opt-in (ASNN_LEVEL_WIN=1): on config 2 it
// measured 2.10 ms per sweep against k_rows' 1.93 (profiles/r2_c2_rows_win.txt).
uint32_t rows_win_bytes(const asnn_dev_layout* L, uint32_t l) {
    if (l >= L->win_lo.size() || L->win_lo[l] > L->win_hi[l]) return 0;
    const uint64_t cap = (static_cast<uint64_t>(L->max_deg) + 1) & ~1ull;
    const uint64_t b = static_cast<uint64_t>(L->win_hi[l] - L->win_lo[l] + 1) * winrows::kTile * 4u +
                       winrows::kRowsPerBlock * cap * 8u;
    return b > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(b);
}
bool rows_win_ok(const asnn_dev_layout* L, uint32_t l, uint32_t ldA) {
    const uint32_t b = rows_win_bytes(L, l);
    return level_win_enabled() && ldA >= 128 && ldA % winrows::kTile == 0 && b && b <= 110u * 1024;
}

// k_rows_tma (tma_rows.cuh): the TMA-gather level kernel for ldA a multiple
// of 128; ASNN_LEVEL_VARIANT=13 selects it (experiments).
bool tma_rows_enabled(uint32_t ldA) { return level_variant() == 13 && ldA >= 128 && ldA % 128 == 0; }
// K-rows-bulk (bulk_rows.cuh): 14 = 16 edges per stage, 15 = 8, 16 = 24
bool bulk_rows_enabled(uint32_t ldA) {
    const int v = level_variant();
    return v >= 14 && v <= 16 && ldA % bulkrows::kTile == 0;
}

int ensure_tmap_A(asnn_dev_layout* L, uint32_t ldA) {
    if (L->tmA_base == L->A.p && L->tmA_ld == ldA) return ASNN_OK;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return fail(L->dev, ASNN_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {ldA, static_cast<cuuint64_t>(L->total_pos) + 1};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldA) * 4};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(tmarows::kTile), 1};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(reinterpret_cast<CUtensorMap*>(L->tmA), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, L->A.p, dims,
                              strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(L->dev, ASNN_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    L->tmA_base = L->A.p;
    L->tmA_ld = ldA;
    return ASNN_OK;
}

template <typename Mark>
int launch_levels(asnn_dev_layout* L, uint32_t ldA, cudaStream_t st, Mark& mark) {
    asnn_dev* dev = L->dev;
    const LevelLaunch ll = level_launch_for(ldA);
    const HeavyLaunch hl = heavy_launch_for(ldA);
    const int thr = heavy_index_for(dev->heavy_threshold);
    const bool segs = seg_eligible(L, ldA);
    if (segs && L->seg_key != seg_key_for(L))
        return fail(dev, ASNN_E_INVALID, "internal: row segments not prepared");
    if (dev->fork_ev.size() < L->n_levels) {
        for (size_t i = dev->fork_ev.size(); i < L->n_levels; ++i) {
            cudaEvent_t a, b;
            CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
            dev->fork_ev.push_back(a);
            dev->join_ev.push_back(b);
        }
    }
    int prio = 0;
    cudaStreamGetPriority(dev->aux, &prio);
    auto launch_heavy = [&](uint32_t l, uint32_t count, const uint32_t* sched, const uint4* seg) -> int {
        CK(cudaEventRecord(dev->fork_ev[l], st));
        CK(cudaStreamWaitEvent(dev->aux, dev->fork_ev[l], 0));
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributePriority;
        attr[0].val.priority = prio;
        cfg.gridDim = dim3(count * hl.tiles);
        cfg.blockDim = dim3(hl.threads);
        cfg.dynamicSmemBytes = hl.smem;
        cfg.stream = dev->aux;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, hl.fn, static_cast<const uint32_t*>(L->row_ptr.p),
                              static_cast<const uint2*>(L->edges.p), L->A.p, ldA, sched, hl.tiles, seg,
                              L->accbuf.p));
        return ASNN_OK;
    };
    bool prev_join = false;  // the previous level ended with an event join
    for (uint32_t l = 1; l < L->n_levels; ++l) {
        const uint32_t n = L->lvl_off[l + 1] - L->lvl_off[l];
        // heavy rows of this level: whole rows on k_heavy, or (segmented)
        // segments of heavy rows of this and later levels
        const uint32_t nh = (hl.fn && thr >= 0) ? L->heavy_cnt[thr * (L->n_levels + 1) + l] : 0;
        const uint32_t ns = segs ? L->seg_short_off[l + 1] - L->seg_short_off[l] : 0;
        const uint32_t nlong = segs ? L->seg_long_off[l + 1] - L->seg_long_off[l] : 0;
        if (!n && !ns && !nlong) continue;
        if (L->total_sensors || l > 1) mark();
        const bool fork = segs ? nlong > 0 : nh > 0;
        if (fork) {
            const int rc = segs ? launch_heavy(l, nlong, nullptr, L->seg.p + L->seg_long_off[l])
                                : launch_heavy(l, nh, L->sched.p + L->lvl_off[l], nullptr);
            if (rc) return rc;
        }
        const uint32_t nrows = n - nh;
        if (nrows || ns) {
            const uint64_t items = static_cast<uint64_t>(nrows + ns) * ll.tiles;
            if (ll.warp_rows)
                ll.warp_rows<<<blocks_for(static_cast<uint64_t>(nrows) * 32), kThreads, 0, st>>>(
                    L->edges.p, L->A.p, L->rtask.p + L->lvl_off[l] + nh, nrows);
            else if (ll.warp_rows4)
                ll.warp_rows4<<<blocks_for(static_cast<uint64_t>(nrows + ns) * 32), kThreads, 0, st>>>(
                    L->edges.p, L->A.p, ldA, L->rtask.p + L->lvl_off[l] + nh, nrows,
                    segs ? L->seg.p + L->seg_short_off[l] : nullptr, ns, L->accbuf.p);
            else if (ll.rows && !nh && !ns && !nlong && rows_win_ok(L, l, ldA)) {
                const uint32_t bytes = rows_win_bytes(L, l);
                static bool attr_set = false;
                if (!attr_set) {
                    CK(cudaFuncSetAttribute(k_rows_win, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
                    attr_set = true;
                }
                cudaLaunchConfig_t cfg{};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.gridDim = dim3((ldA / winrows::kTile) *
                                   ((nrows + winrows::kRowsPerBlock - 1) / winrows::kRowsPerBlock));
                cfg.blockDim = dim3(winrows::kThreads);
                cfg.dynamicSmemBytes = bytes;
                cfg.stream = st;
                cfg.attrs = attr;
                cfg.numAttrs = pdl_enabled() && !fork && !prev_join && l > 1 ? 1 : 0;
                CK(cudaLaunchKernelEx(&cfg, k_rows_win, static_cast<const uint2*>(L->edges.p), L->A.p, ldA,
                                      static_cast<const uint4*>(L->rtask.p + L->lvl_off[l]), nrows, L->win_lo[l],
                                      L->win_hi[l] - L->win_lo[l] + 1, (L->max_deg + 1) & ~1u));
            } else if (ll.rows && bulk_rows_enabled(ldA)) {
                const int v = level_variant();
                auto fn = v == 15 ? k_rows_bulk<8> : v == 16 ? k_rows_bulk<24> : k_rows_bulk<16>;
                const uint32_t smem = v == 15   ? bulkrows::smem_bytes<8>()
                                      : v == 16 ? bulkrows::smem_bytes<24>()
                                                : bulkrows::smem_bytes<16>();
                static bool attr_set = false;
                if (!attr_set) {
                    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                    attr_set = true;
                }
                const uint32_t tiles = ldA / bulkrows::kTile;
                cudaLaunchConfig_t cfg{};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.gridDim = dim3(static_cast<uint32_t>(static_cast<uint64_t>(nrows + ns) * tiles));
                cfg.blockDim = dim3(bulkrows::kThreads);
                cfg.dynamicSmemBytes = smem;
                cfg.stream = st;
                cfg.attrs = attr;
                cfg.numAttrs = pdl_enabled() && !fork && !prev_join && l > 1 ? 1 : 0;
                CK(cudaLaunchKernelEx(&cfg, fn, static_cast<const uint2*>(L->edges.p), L->A.p, ldA,
                                      static_cast<const uint4*>(L->rtask.p + L->lvl_off[l] + nh), nrows, tiles,
                                      static_cast<const uint4*>(segs ? L->seg.p + L->seg_short_off[l] : nullptr), ns,
                                      L->accbuf.p));
            } else if (ll.rows && tma_rows_enabled(ldA)) {
                RC_(ensure_tmap_A(L, ldA));
                static bool attr_set = false;
                if (!attr_set) {
                    CK(cudaFuncSetAttribute(k_rows_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(tmarows::smem_bytes())));
                    attr_set = true;
                }
                cudaLaunchConfig_t cfg{};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.gridDim = dim3(static_cast<uint32_t>(std::min<uint64_t>(
                    (items + tmarows::kWarps - 1) / tmarows::kWarps, 2ull * dev->sm_count)));
                cfg.blockDim = dim3(32 * (tmarows::kWarps + 1));
                cfg.dynamicSmemBytes = tmarows::smem_bytes();
                cfg.stream = st;
                cfg.attrs = attr;
                cfg.numAttrs = pdl_enabled() && !fork && !prev_join && l > 1 ? 1 : 0;
                CK(cudaLaunchKernelEx(&cfg, k_rows_tma, *reinterpret_cast<const CUtensorMap*>(L->tmA),
                                      static_cast<const uint2*>(L->edges.p), L->A.p, ldA,
                                      static_cast<const uint4*>(L->rtask.p + L->lvl_off[l] + nh), nrows, ll.tiles,
                                      static_cast<const uint4*>(segs ? L->seg.p + L->seg_short_off[l] : nullptr), ns,
                                      L->accbuf.p, L->total_pos));
            } else if (ll.rows) {
                cudaLaunchConfig_t cfg{};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.gridDim = dim3(blocks_for(items * ll.lanes));
                cfg.blockDim = dim3(kThreads);
                cfg.stream = st;
                cfg.attrs = attr;
                // only after another kernel on this stream (not an event join), and
                // only when every 32-byte sector of A belongs to one row (ldA >= 8):
                // the gathers are ld.global.nc, so no sector a later level reads
                // may share bytes with rows the previous grid is still writing
                cfg.numAttrs = pdl_enabled() && !fork && !prev_join && l > 1 && ldA >= 8 ? 1 : 0;
                CK(cudaLaunchKernelEx(&cfg, ll.rows, static_cast<const uint2*>(L->edges.p), L->A.p, ldA,
                                      static_cast<const uint4*>(L->rtask.p + L->lvl_off[l] + nh), nrows,
                                      ll.tiles,
                                      static_cast<const uint4*>(segs ? L->seg.p + L->seg_short_off[l] : nullptr),
                                      ns, L->accbuf.p));
            }
            else
                ll.lvl<<<blocks_for(items * ll.lanes), kThreads, 0, st>>>(
                    L->row_ptr.p, L->edges.p, L->A.p, ldA, L->sched.p + L->lvl_off[l] + nh,
                    static_cast<uint32_t>(items), ll.tiles);
        }
        if (fork) {
            CK(cudaEventRecord(dev->join_ev[l], dev->aux));
            CK(cudaStreamWaitEvent(st, dev->join_ev[l], 0));
        }
        prev_join = fork;
    }
    CK(cudaGetLastError());
    return ASNN_OK;
}

// K-chain staging plan (chain.cuh).  Groups: consecutive layers packed
// greedily while their row pointers, splits and edges stay within `target`
// bytes (a larger layer is a group alone).  The ring is then simulated on the
// host exactly as a dynamic producer would run it -- byte-granular packing
// with wrap, releases in group order, 32 mbarrier slots, and a group that
// would need the release of the group just before it read from global memory
// (F finishes a group's last layer only with the next group's first prefix)
// -- so the device producer only executes the plan: per group {wait for the
// release of group X, 3 bulk copies}.  Built once per (target, ring).
int ensure_groups(asnn_dev_layout* L, uint32_t target, uint32_t ring) {
    if (L->grp.p && L->grp_target == target && L->grp_ring == ring) return ASNN_OK;
    asnn_dev* dev = L->dev;
    const uint32_t G = static_cast<uint32_t>(L->nets.size());
    std::vector<uint4> gp;                  // per group: 2 x uint4 (chain::GroupPlan)
    std::vector<uint4> lp(2 * (L->le_host.size() + 1), make_uint4(0u, 0u, 0u, 0u));  // per layer
    std::vector<uint32_t> off(G + 1, 0);
    for (uint32_t gi = 0; gi < G; ++gi) {
        const NetMeta& n = L->nets[gi];
        const uint32_t* lo = n.layer_offsets.data();
        const uint32_t* le = L->le_host.data() + L->lo_base_host[gi];
        const uint32_t lb = L->lo_base_host[gi];
        off[gi] = static_cast<uint32_t>(gp.size() / 2);
        // groups of this network
        std::vector<uint32_t> l0s;
        for (uint32_t l = 1; l < n.n_layers;) {
            const uint32_t l0 = l++;
            l0s.push_back(l0);
            while (l < n.n_layers) {
                uint32_t rb, sb, eb;
                chain::group_bytes(n.pos_base + lo[l0], n.pos_base + lo[l + 1], le[l0], le[l + 1], rb, sb, eb);
                if (static_cast<uint64_t>(rb) + sb + eb > target) break;
                ++l;
            }
        }
        l0s.push_back(n.n_layers);
        const uint32_t K = static_cast<uint32_t>(l0s.size()) - 1;
        // ring simulation
        uint32_t w = 0, used = 0;
        std::deque<std::pair<uint32_t, uint32_t>> live;  // (group, extent)
        for (uint32_t k = 0; k < K; ++k) {
            const uint32_t l0 = l0s[k], l1 = l0s[k + 1];
            const uint32_t r0 = n.pos_base + lo[l0], r1 = n.pos_base + lo[l1];
            uint32_t rb, sb, eb;
            chain::group_bytes(r0, r1, le[l0], le[l1], rb, sb, eb);
            const uint32_t size = rb + sb + eb;
            int64_t wait = k >= cta::kSlots ? static_cast<int64_t>(k) - cta::kSlots : -1;  // slot reuse
            while (!live.empty() && static_cast<int64_t>(live.front().first) <= wait) {
                used -= live.front().second;
                live.pop_front();
            }
            bool staged = size <= ring;
            uint32_t at = 0;
            if (staged) {
                for (;;) {
                    if (used == 0) w = 0;
                    const bool wrap = w + size > ring;
                    const uint32_t need = wrap ? ring - w + size : size;
                    if (need <= ring - used) {
                        at = wrap ? 0u : w;
                        w = at + size;
                        used += need;
                        live.emplace_back(k, need);
                        break;
                    }
                    if (live.front().first + 1 >= k) {  // only the previous group holds the space
                        staged = false;
                        break;
                    }
                    wait = std::max<int64_t>(wait, live.front().first);
                    used -= live.front().second;
                    live.pop_front();
                }
            }
            const uint32_t r0a = r0 & ~3u, e0a = le[l0] & ~1u;
            const uint32_t rows_at = at / 4, split_at = (at + rb) / 4, edges_at = (at + rb + sb) / 8;
            gp.push_back(make_uint4(r0a, e0a, eb, static_cast<uint32_t>(wait + 1)));
            gp.push_back(make_uint4(at | (staged ? chain::kPlanStaged : 0u), rb, sb, 0u));
            for (uint32_t l = l0; l < l1; ++l) {
                lp[2 * (lb + l)] = make_uint4(lo[l], lo[l + 1], k | (l + 1 == l1 ? chain::kPlanGroupEnd : 0u),
                                              edges_at);
                lp[2 * (lb + l) + 1] = make_uint4(r0a, e0a, rows_at | (staged ? chain::kPlanStaged : 0u), split_at);
            }
        }
    }
    off[G] = static_cast<uint32_t>(gp.size() / 2);
    if (gp.empty()) gp.push_back(make_uint4(0u, 0u, 0u, 0u));
    L->graph.reset();
    cudaStream_t st = dev->stream;
    CK(L->grp.alloc(gp.size()));
    CK(L->grp_off.alloc(G + 1));
    CK(L->lplan.alloc(lp.size()));
    CK(cudaMemcpyAsync(L->grp.p, gp.data(), gp.size() * sizeof(uint4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(L->grp_off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(L->lplan.p, lp.data(), lp.size() * sizeof(uint4), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // the host vectors go out of scope
    L->grp_target = target;
    L->grp_ring = ring;
    return ASNN_OK;
}

int ensure_workspace(asnn_dev_layout* L, uint32_t n_vec) {
    asnn_dev* dev = L->dev;
    const uint32_t ldA = padded_batch(n_vec);
    if (!cta_plan(L, ldA).use) {
        const int rc = ensure_schedule(L);
        if (rc) return rc;
    }
    // split[] at the prefix depth the plan needs (pipelined K-cta 1, K-chain NP - 1)
    const CtaPlan cpl = cta_plan(L, ldA);
    const uint32_t want_d = cpl.chain_nf ? chain_np(cpl.chain_nf) - 1 : cpl.pipe ? 1u : 0u;
    if (want_d && (!L->split.p || L->split_d != want_d)) {
        L->graph.reset();
        if (!L->split.p) CK(L->split.alloc(L->total_pos + 8));  // slack: K-cta bulk copies round up to 16 bytes
        const uint32_t G = static_cast<uint32_t>(L->nets.size());
        k_splits<<<dim3((L->max_pos + 255) / 256, G), 256, 0, dev->stream>>>(
            reinterpret_cast<const CtaNet*>(L->cta_nets.p), L->lo_cat.p, L->row_ptr.p, L->edges.p, L->split.p,
            want_d);
        CK(cudaGetLastError());
        L->split_d = want_d;
    }
    if (cpl.use && cpl.chain_nf) {
        const int rc = ensure_groups(L, chain_group_target(cpl), cpl.ring_bytes);
        if (rc) return rc;
    }
    if (seg_eligible(L, ldA)) {
        if (L->seg_key != seg_key_for(L)) {
            L->graph.reset();
            const int rc = ensure_segments(L);
            if (rc) return rc;
        }
        if (L->accbuf.n < static_cast<size_t>(L->n_slots) * ldA) {
            L->graph.reset();
            CK(L->accbuf.alloc(static_cast<size_t>(L->n_slots) * ldA));
        }
    }
    // +1 row: the never-written zero row for predecessors without a position.
    const size_t need = (static_cast<size_t>(L->total_pos) + 1) * ldA;
    if (need > L->A.n) {
        L->graph.reset();
        CK(L->A.alloc(need));
        CK(cudaMemsetAsync(L->A.p, 0, need * sizeof(float), L->dev->stream));
        L->zero_ldA = ldA;
    } else if (L->zero_refs && L->zero_ldA != ldA) {
        // A narrower sweep reuses the array: row total_pos at the new pitch
        // overlaps rows an earlier, wider sweep wrote -- clear it again.
        CK(cudaMemsetAsync(L->A.p + static_cast<size_t>(L->total_pos) * ldA, 0, ldA * sizeof(float),
                           L->dev->stream));
        L->zero_ldA = ldA;
    }
    return ASNN_OK;
}

// Sweep through a cached CUDA graph (one launch per sweep instead of one per
// level).  The graph is re-captured when buffers or the stream change.
int run_sweep(asnn_dev_layout* L, const float* x, uint32_t n_vec, float* out, float* state) {
    asnn_dev* dev = L->dev;
    int rc = ensure_workspace(L, n_vec);
    if (rc) return rc;
    cudaStream_t st = dev->stream;
    SweepGraph& g = L->graph;
    const bool same = g.n_vec == n_vec && g.x == x && g.out == out && g.state == state && g.stream == st &&
                      g.epoch == dev->option_epoch;
    if (!(g.exec && same)) {
        if (!(g.seen && same)) {  // first time with these parameters: launch directly
            g.reset();
            g.seen = true;
            g.n_vec = n_vec;
            g.x = x;
            g.out = out;
            g.state = state;
            g.stream = st;
            g.epoch = dev->option_epoch;
            return launch_sweep(L, x, n_vec, out, state, st);
        }
        g.reset();
        // L2 persistence for the front of the activation array: positions are
        // level-sorted, so the earliest layers -- the sources most later rows
        // gather from -- sit at the start of A (ASNN_L2_PERSIST_MB, 0 = off).
        {
            static const long want_mb = [] {
                const char* s = getenv("ASNN_L2_PERSIST_MB");
                return s ? atol(s) : 0L;
            }();
            cudaStreamAttrValue av{};
            if (want_mb > 0) {
                int max_persist = 0;
                cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev->device);
                const size_t bytes = std::min<size_t>(static_cast<size_t>(want_mb) << 20,
                                                      static_cast<size_t>(max_persist));
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes);
                av.accessPolicyWindow.base_ptr = L->A.p;
                av.accessPolicyWindow.num_bytes = std::min(bytes, L->A.n * sizeof(float));
                av.accessPolicyWindow.hitRatio = 1.0f;
                av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            }
            cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av);
            cudaStreamSetAttribute(dev->aux, cudaStreamAttributeAccessPolicyWindow, &av);
            cudaGetLastError();
        }
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        rc = launch_sweep(L, x, n_vec, out, state, st);
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        CK(ce);
        ce = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(ce);
        g.n_vec = n_vec;
        g.x = x;
        g.out = out;
        g.state = state;
        g.stream = st;
        g.epoch = dev->option_epoch;
    }
    CK(cudaGraphLaunch(g.exec, st));
    return ASNN_OK;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Device-visible address of page-locked, mapped host memory (UVA), or null.
void* mapped_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}


}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

const char* asnn_dev_version(void) { return "asnn-b200 0.1 (sm_100a)"; }

int asnn_dev_latency_probe(asnn_dev* dev, int which, int n, double* cycles_per_op) {
    if (!dev || !cycles_per_op || n <= 0) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    CK(cudaSetDevice(dev->device));
    DevBuf<long long> c;
    DevBuf<float> sink;
    CK(c.alloc(1));
    CK(sink.alloc(1));
    void (*fns[])(int, float, long long*, float*) = {k_latency_probe<0>, k_latency_probe<1>,
                                                      k_latency_probe<2>, k_latency_probe<3>,
                                                      k_latency_probe<4>, k_latency_probe<5>,
                                                      k_latency_probe<6>};
    if (which < 0 || which > 6) return fail(dev, ASNN_E_INVALID, "probe index");
    fns[which]<<<1, 32, 0, dev->stream>>>(n, 0.37f, c.p, sink.p);
    CK(cudaGetLastError());
    long long h = 0;
    CK(cudaMemcpyAsync(&h, c.p, 8, cudaMemcpyDeviceToHost, dev->stream));
    CK(cudaStreamSynchronize(dev->stream));
    *cycles_per_op = static_cast<double>(h) / n;
    return ASNN_OK;
}

int asnn_dev_sigmoid_selfcheck(asnn_dev* dev, uint64_t* mismatches, uint64_t* exact_path) {
    if (!dev || !mismatches || !exact_path) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    CK(cudaSetDevice(dev->device));
    DevBuf<unsigned long long> c;
    CK(c.alloc(2));
    CK(cudaMemsetAsync(c.p, 0, 16, dev->stream));
    k_sigmoid_selfcheck<<<dev->sm_count * 8, 256, 0, dev->stream>>>(c.p);
    CK(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, c.p, 16, cudaMemcpyDeviceToHost, dev->stream));
    CK(cudaStreamSynchronize(dev->stream));
    *mismatches = h[0];
    *exact_path = h[1];
    return ASNN_OK;
}

int asnn_dev_sigmoid32(asnn_dev* dev, const float* x, float* y, uint64_t n) {
    if (!dev || (n && (!x || !y))) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    if (!n) return ASNN_OK;
    CK(cudaSetDevice(dev->device));
    DevBuf<float> dx, dy;
    CK(dx.alloc(n));
    CK(dy.alloc(n));
    cudaStream_t st = dev->stream;
    CK(cudaMemcpyAsync(dx.p, x, n * 4, cudaMemcpyHostToDevice, st));
    k_sigmoid_many<<<blocks_for(n), kThreads, 0, st>>>(dx.p, dy.p, n);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(y, dy.p, n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return ASNN_OK;
}

int asnn_dev_device_count(int* count) {
    if (!count) return ASNN_E_INVALID;
    *count = 0;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return ASNN_E_UNAVAILABLE;
    }
    *count = n;
    return n > 0 ? ASNN_OK : ASNN_E_UNAVAILABLE;
}

int asnn_dev_open(int device, asnn_dev** out) {
    if (!out) return ASNN_E_INVALID;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return ASNN_E_UNAVAILABLE;
    }
    if (device < 0 || device >= n) return ASNN_E_UNAVAILABLE;
    auto* dev = new asnn_dev;
    dev->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&dev->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&dev->own_stream, cudaStreamNonBlocking);
    for (cudaEvent_t* ev : {&dev->ev0, &dev->ev1, &dev->ev2, &dev->ev3, &dev->ev4})
        if (e == cudaSuccess) e = cudaEventCreate(ev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete dev;
        return ASNN_E_UNAVAILABLE;
    }
    dev->stream = dev->own_stream;
    // stream-ordered allocations (engine.hpp AllocStream) keep freed memory in
    // the device's default pool instead of returning it at every synchronise
    {
        cudaMemPool_t pool = nullptr;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    dev->heavy_threshold = default_heavy_threshold();
    if (const char* m = getenv("ASNN_SWEEP_MODE")) dev->sweep_mode = static_cast<uint32_t>(atoi(m)) % 5;
    // The heavy-row branch gets the highest stream priority: its CTAs carry
    // the longest dependent-add chains of the layer and must become resident
    // before the light rows fill the machine (ASNN_HEAVY_PRIO=0 disables).
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    {
        const char* hp = getenv("ASNN_HEAVY_PRIO");
        if (hp && atoi(hp) == 0) prio_hi = prio_lo;
    }
    if (cudaStreamCreateWithPriority(&dev->aux, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
        cudaGetLastError();
        delete dev;
        return ASNN_E_UNAVAILABLE;
    }
    *out = dev;
    return ASNN_OK;
}

void asnn_dev_close(asnn_dev* dev) {
    if (!dev) return;
    cudaSetDevice(dev->device);
    cudaStreamSynchronize(dev->stream);
    asnn_eval_buf_free(dev->once);
    release_comm(dev);
    for (cudaEvent_t ev : {dev->ev0, dev->ev1, dev->ev2, dev->ev3, dev->ev4, dev->stage_ev[0], dev->stage_ev[1]})
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : dev->fork_ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : dev->join_ev) cudaEventDestroy(ev);
    if (dev->aux) cudaStreamDestroy(dev->aux);
    if (dev->own_stream) cudaStreamDestroy(dev->own_stream);
    delete dev;
}

const char* asnn_dev_last_error(const asnn_dev* dev) { return dev ? dev->err.c_str() : ""; }

int asnn_dev_set_stream(asnn_dev* dev, void* s) {
    if (!dev) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    dev->stream = s ? static_cast<cudaStream_t>(s) : dev->own_stream;
    return ASNN_OK;
}

void* asnn_dev_get_stream(asnn_dev* dev) { return dev ? dev->stream : nullptr; }

int asnn_dev_set_sweep_mode(asnn_dev* dev, uint32_t mode) {
    if (!dev || mode > 5) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    dev->sweep_mode = mode;
    ++dev->option_epoch;
    return ASNN_OK;
}

int asnn_dev_set_heavy_threshold(asnn_dev* dev, uint32_t min_in_degree) {
    if (!dev) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    dev->heavy_threshold = min_in_degree;
    ++dev->option_epoch;
    return ASNN_OK;
}

int asnn_dev_synchronize(asnn_dev* dev) {
    if (!dev) return ASNN_E_INVALID;
    cudaSetDevice(dev->device);
    CK(cudaStreamSynchronize(dev->stream));
    return ASNN_OK;
}

int asnn_dev_last_timings(const asnn_dev* dev, asnn_timings* out) {
    if (!dev || !out) return ASNN_E_INVALID;
    *out = dev->timings;
    return ASNN_OK;
}

// eval_parallel's input: a host LayeredLayout in CSR form.  The raw arrays
// are copied as-is; id -> position renumbering runs on the device.
int asnn_dev_upload_layout(asnn_dev* dev, const asnn_layout_desc* d, asnn_dev_layout** out) {
    if (!dev || !d || !out) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    *out = nullptr;
    CK(cudaSetDevice(dev->device));
    if (d->total_layers == 0 && d->node_count) return fail(dev, ASNN_E_INVALID, "layers missing");
    if (d->node_count && (!d->layer_offsets || !d->node_ids || !d->row_ptr))
        return fail(dev, ASNN_E_INVALID, "null layout array");
    if (d->total_layers && d->layer_offsets[d->total_layers] != d->node_count)
        return fail(dev, ASNN_E_INVALID, "layer_offsets do not cover node_count");
    const uint64_t E = d->node_count ? d->row_ptr[d->node_count] : 0;
    if (E >= 0xFFFFFFFFull) return fail(dev, ASNN_E_INVALID, "more than 2^32-1 edges");
    if (d->total_layers && d->layer_offsets[0] != 0) return fail(dev, ASNN_E_INVALID, "layer_offsets[0] != 0");
    for (uint32_t k = 0; k < d->total_layers; ++k)
        if (d->layer_offsets[k + 1] < d->layer_offsets[k])
            return fail(dev, ASNN_E_INVALID, "layer_offsets decrease");
    if (d->node_count) {
        if (d->row_ptr[0] != 0) return fail(dev, ASNN_E_INVALID, "row_ptr[0] != 0");
        int64_t bad = 0;
        const int64_t N = d->node_count;
#pragma omp parallel for reduction(| : bad) if (N > (1 << 20))
        for (int64_t i = 0; i < N; ++i) bad |= d->row_ptr[i + 1] < d->row_ptr[i];
        if (bad) return fail(dev, ASNN_E_INVALID, "row_ptr decreases");
    }
    cudaStream_t st = dev->stream;
    // small layouts (the per-call drop-in): every host array through the
    // pinned arena, one asynchronous DMA each
    {
        const uint64_t bytes = 12ull * d->node_count + 8 * E + 4ull * (d->n_inputs + d->n_outputs) +
                               64ull * (d->total_layers + 64);
        arena_reset(dev);
        if (bytes <= (64ull << 20)) CK(dev->arena.ensure(std::max<uint64_t>(bytes + (1 << 16), 1 << 20)));
    }
    CK(cudaEventRecord(dev->ev0, st));
    NetMeta n;
    n.n_pos = d->node_count;
    n.n_layers = d->total_layers;
    n.n_sensors = d->total_layers ? d->layer_offsets[1] : 0;
    n.id_bound = d->id_bound;
    n.n_in = d->n_inputs;
    n.n_out = d->n_outputs;
    n.n_edges = E;
    n.layer_offsets.assign(d->layer_offsets, d->layer_offsets + d->total_layers + 1);
    if (d->n_inputs) n.inputs.assign(d->input_order, d->input_order + d->n_inputs);
    if (d->n_outputs) n.outputs.assign(d->outputs, d->outputs + d->n_outputs);
    FlatDevice f;
    DevBuf<uint64_t> row64;
    CK(f.node_ids.alloc(d->node_count));
    CK(f.row_ptr.alloc(d->node_count + 8));  // slack: K-cta bulk copies round up to 16 bytes
    CK(row64.alloc(d->node_count + 1));
    CK(f.in_ids.alloc(E));
    CK(f.w.alloc(E));
    CK(f.inputs.alloc(d->n_inputs));
    CK(f.outputs.alloc(d->n_outputs));
    if (d->node_count) {
        CK(h2d(dev, f.node_ids.p, d->node_ids, d->node_count * 4ull, st));
        CK(h2d(dev, row64.p, d->row_ptr, (d->node_count + 1) * 8ull, st));
        k_row64_to_32<<<blocks_for(d->node_count + 1), kThreads, 0, st>>>(row64.p, d->node_count + 1,
                                                                           f.row_ptr.p);
    } else {
        CK(cudaMemsetAsync(f.row_ptr.p, 0, 4, st));
    }
    if (E) {
        CK(h2d(dev, f.in_ids.p, d->in_nodes, E * 4, st));
        CK(h2d(dev, f.w.p, d->in_weights, E * 4, st));
    }
    if (d->n_inputs)
        CK(h2d(dev, f.inputs.p, d->input_order, d->n_inputs * 4ull, st));
    if (d->n_outputs)
        CK(h2d(dev, f.outputs.p, d->outputs, d->n_outputs * 4ull, st));
    std::vector<NetMeta> nets;
    nets.push_back(std::move(n));
    int rc = assemble_layout(dev, std::move(nets), std::move(f), out);
    if (rc == ASNN_OK) {
        CK(cudaEventRecord(dev->ev1, st));
        CK(cudaEventSynchronize(dev->ev1));
        cudaEventElapsedTime(&dev->timings.upload_ms, dev->ev0, dev->ev1);
    }
    return rc;
}

void asnn_dev_free_layout(asnn_dev_layout* L) {
    if (!L) return;
    if (L->server) asnn_dev_server_stop(L->server);
    std::lock_guard<std::recursive_mutex> lk(L->dev->mu);
    cudaSetDevice(L->dev->device);
    cudaStreamSynchronize(L->dev->stream);
    delete L;
}

int asnn_dev_layout_info(const asnn_dev_layout* L, asnn_layout_info* info) {
    if (!L || !info) return ASNN_E_INVALID;
    info->n_networks = static_cast<uint32_t>(L->nets.size());
    info->total_layers = L->n_levels;
    info->node_count = L->total_pos;
    info->edge_count = L->total_edges;
    info->dropped_connections = L->dropped;
    info->id_bound = L->total_idb;
    info->n_inputs = L->total_in;
    info->n_outputs = L->total_out;
    info->max_layer_width = L->max_width;
    info->max_in_degree = L->max_deg;
    return ASNN_OK;
}

int asnn_dev_network_info(const asnn_dev_layout* L, uint32_t g, asnn_layout_info* info) {
    if (!L || !info) return ASNN_E_INVALID;
    if (g >= L->nets.size()) return fail(L->dev, ASNN_E_INVALID, "network index out of range");
    const NetMeta& n = L->nets[g];
    info->n_networks = 1;
    info->total_layers = n.n_layers;
    info->node_count = n.n_pos;
    info->edge_count = n.n_edges;
    info->dropped_connections = n.dropped;
    info->id_bound = n.id_bound;
    info->n_inputs = n.n_in;
    info->n_outputs = n.n_out;
    uint32_t w = 0;
    for (uint32_t l = 0; l < n.n_layers; ++l) w = std::max(w, n.layer_offsets[l + 1] - n.layer_offsets[l]);
    info->max_layer_width = w;
    info->max_in_degree = L->max_deg;
    return ASNN_OK;
}

// layer_slice_bounds (layout.cpp:85-91): LayerOutOfRange past the last layer.
int asnn_dev_layer_slice(const asnn_dev_layout* L, uint32_t layer, uint32_t* start, uint32_t* count) {
    if (!L || !start || !count) return ASNN_E_INVALID;
    const NetMeta& n = L->nets[0];
    if (layer >= n.n_layers)
        return fail(L->dev, ASNN_E_LAYER_RANGE,
                    "layer " + std::to_string(layer) + " out of range, total layers " +
                        std::to_string(n.n_layers));
    *start = n.layer_offsets[layer];
    *count = n.layer_offsets[layer + 1] - n.layer_offsets[layer];
    return ASNN_OK;
}

// Flattened layout of one network back in the reference's form (ids, not
// positions), for flatten parity checks.
int asnn_dev_layout_download(asnn_dev_layout* L, uint32_t g, uint32_t* layer_offsets,
                             uint32_t* node_ids, uint64_t* row_ptr, uint32_t* in_nodes,
                             float* in_weights, uint32_t* input_order) {
    if (!L) return ASNN_E_INVALID;
    asnn_dev* dev = L->dev;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    if (g >= L->nets.size()) return fail(dev, ASNN_E_INVALID, "network index out of range");
    CK(cudaSetDevice(dev->device));
    const NetMeta& n = L->nets[g];
    cudaStream_t st = dev->stream;
    std::vector<uint32_t> ids(n.n_pos), rp(n.n_pos + 1);
    std::vector<uint2> ed(n.n_edges);
    if (n.n_pos) {
        CK(cudaMemcpyAsync(ids.data(), L->node_ids.p + n.pos_base, n.n_pos * 4ull, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(rp.data(), L->row_ptr.p + n.pos_base, (n.n_pos + 1) * 4ull, cudaMemcpyDeviceToHost, st));
    }
    if (n.n_edges)
        CK(cudaMemcpyAsync(ed.data(), L->edges.p + n.edge_base, n.n_edges * 8, cudaMemcpyDeviceToHost, st));
    std::vector<uint4> si(L->total_sensors);
    if (L->total_sensors)
        CK(cudaMemcpyAsync(si.data(), L->sinfo.p, L->total_sensors * 16ull, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (layer_offsets) std::copy(n.layer_offsets.begin(), n.layer_offsets.end(), layer_offsets);
    if (node_ids) std::copy(ids.begin(), ids.end(), node_ids);
    if (row_ptr)
        for (uint32_t p = 0; p <= n.n_pos; ++p) row_ptr[p] = rp[p] - rp[0];
    for (uint64_t k = 0; k < n.n_edges; ++k) {
        const uint32_t pos = ed[k].x;
        if (in_nodes)
            in_nodes[k] = (pos >= n.pos_base && pos < n.pos_base + n.n_pos) ? ids[pos - n.pos_base]
                                                                            : ASNN_UNASSIGNED;
        if (in_weights) std::memcpy(&in_weights[k], &ed[k].y, 4);
    }
    if (input_order) std::copy(n.inputs.begin(), n.inputs.end(), input_order);
    (void)si;
    return ASNN_OK;
}

// Kernels one sweep launches (stages = false) or the stages profile_sweep
// brackets with events (stages = true: sensors, one per level, output gather).
static uint32_t sweep_launches(asnn_dev_layout* L, uint32_t n_vec, bool stages, bool with_out = true) {
    uint32_t k = 0;
    const uint32_t ldA = padded_batch(n_vec);
    const CtaPlan cp = cta_plan(L, ldA);
    if (cp.use) {
        // K-cta runs sensors and every layer, and writes the outputs itself
        // unless it is the global-memory variant
        return 1u + (with_out && cp.global && L->total_out ? 1u : 0u);
    } else {
        if (ensure_schedule(L)) return 0;
        const int thr = heavy_index_for(L->dev->heavy_threshold);
        const bool heavy = heavy_launch_for(ldA).fn && thr >= 0;
        const bool segs = seg_eligible(L, ldA);
        if (segs && L->seg_key != seg_key_for(L)) ensure_segments(L);
        k = L->total_sensors ? 1 : 0;
        for (uint32_t l = 1; l < L->n_levels; ++l) {
            const uint32_t n = L->lvl_off[l + 1] - L->lvl_off[l];
            const uint32_t nh = heavy ? L->heavy_cnt[thr * (L->n_levels + 1) + l] : 0;
            const uint32_t ns = segs ? L->seg_short_off[l + 1] - L->seg_short_off[l] : 0;
            const uint32_t nl = segs ? L->seg_long_off[l + 1] - L->seg_long_off[l] : 0;
            if (stages) k += (n || ns || nl) ? 1 : 0;
            else if (segs) k += (n - nh + ns > 0) + (nl > 0);
            else k += (n > nh) + (nh > 0);
        }
    }
    return k + (with_out && L->total_out ? 1 : 0);
}

int asnn_dev_profile_sweep(asnn_dev_layout* L, const float* x_dev, uint32_t n_vec, float* out_dev,
                           float* ms, uint32_t* n_launches) {
    if (!L || !ms || !n_launches) return ASNN_E_INVALID;
    asnn_dev* dev = L->dev;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    CK(cudaSetDevice(dev->device));
    int rc = ensure_workspace(L, n_vec);
    if (rc) return rc;
    const uint32_t k = sweep_launches(L, n_vec, true, out_dev != nullptr);
    std::vector<cudaEvent_t> evs(k + 1);
    for (auto& e : evs) CK(cudaEventCreate(&e));
    rc = launch_sweep(L, x_dev, n_vec, out_dev, nullptr, dev->stream, &evs);
    cudaError_t e = cudaStreamSynchronize(dev->stream);
    for (uint32_t i = 0; i < k && rc == ASNN_OK && e == cudaSuccess; ++i)
        cudaEventElapsedTime(&ms[i], evs[i], evs[i + 1]);
    for (auto& ev : evs) cudaEventDestroy(ev);
    CK(e);
    *n_launches = k;
    return rc;
}

int asnn_dev_activate_plan(asnn_dev_layout* L, uint32_t n_vec, uint32_t* kernels, uint64_t* alg_bytes,
                           uint64_t* conn_evals) {
    if (!L) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(L->dev->mu);
    asnn_b200::AllocStream alloc_on(L->dev->stream);
    const uint32_t k = sweep_launches(L, n_vec, false);
    if (kernels) *kernels = k;
    const uint64_t B = n_vec, E = L->total_edges, N = L->total_pos;
    // 8E (col+w) + 4(N+1) row_ptr + 4EB gathers + 4NB writes + 4 n_in B reads
    if (alg_bytes) *alg_bytes = 8 * E + 4 * (N + 1) + 4 * E * B + 4 * N * B + 4ull * L->total_in * B;
    if (conn_evals) *conn_evals = E * B;
    return ASNN_OK;
}

int asnn_dev_sweep_kind(asnn_dev_layout* L, uint32_t n_vec, uint32_t* kind) {
    if (!L || !kind) return ASNN_E_INVALID;
    const uint32_t ldA = padded_batch(n_vec);
    const CtaPlan cp = cta_plan(L, ldA);
    *kind = cp.use ? (cp.chain_nf ? 3u : 2u) : seg_eligible(L, ldA) ? 1u : 0u;
    return ASNN_OK;
}

int asnn_dev_activate_device(asnn_dev_layout* L, const float* x_dev, uint32_t n_vec, float* out_dev) {
    if (!L) return ASNN_E_INVALID;
    asnn_dev* dev = L->dev;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    if (n_vec == 0) return ASNN_OK;
    CK(cudaSetDevice(dev->device));
    return run_sweep(L, x_dev, n_vec, out_dev, nullptr);
}

}  // extern "C"

int asnn_b200::enqueue_sweep(asnn_dev_layout* L, const float* x_dev, uint32_t n_vec, float* out_dev,
                             float* state_dev) {
    if (!L) return ASNN_E_INVALID;
    asnn_dev* dev = L->dev;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    if (n_vec == 0) return ASNN_OK;
    CK(cudaSetDevice(dev->device));
    return run_sweep(L, x_dev, n_vec, out_dev, state_dev);
}

extern "C" {

// Debug write-count sweep (ASNN_WRITE_COUNT builds only): counts[p][b] = how
// many times op slot (position p, column b < n_vec) was produced in one sweep.
int asnn_dev_debug_write_counts(asnn_dev_layout* L, uint32_t n_vec, uint32_t* counts) {
    if (!L || !counts || n_vec == 0) return ASNN_E_INVALID;
    asnn_dev* dev = L->dev;
#ifndef ASNN_WRITE_COUNT
    return fail(dev, ASNN_E_UNAVAILABLE, "built without ASNN_WRITE_COUNT (make -C csrc wc)");
#else
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    CK(cudaSetDevice(dev->device));
    int rc = ensure_workspace(L, n_vec);
    if (rc) return rc;
    const uint32_t ldA = padded_batch(n_vec);
    const size_t n = (static_cast<size_t>(L->total_pos) + 1) * ldA;
    DevBuf<uint32_t> wc;
    DevBuf<float> x;
    CK(wc.alloc(n));
    CK(x.alloc(static_cast<size_t>(L->total_in) * n_vec + 1));
    CK(cudaMemset(wc.p, 0, n * 4));
    CK(cudaMemset(x.p, 0, (static_cast<size_t>(L->total_in) * n_vec + 1) * 4));
    CK(cudaMemcpyToSymbol(g_wc, &wc.p, sizeof(wc.p)));
    CK(cudaMemcpyToSymbol(g_wc_ld, &ldA, sizeof(ldA)));
    CK(cudaStreamSynchronize(dev->stream));
    rc = launch_sweep(L, x.p, n_vec, nullptr, nullptr, dev->stream);
    CK(cudaStreamSynchronize(dev->stream));
    uint32_t* null_wc = nullptr;
    CK(cudaMemcpyToSymbol(g_wc, &null_wc, sizeof(null_wc)));
    if (rc) return rc;
    std::vector<uint32_t> h(n);
    CK(cudaMemcpy(h.data(), wc.p, n * 4, cudaMemcpyDeviceToHost));
    for (size_t p = 0; p < L->total_pos; ++p)
        std::memcpy(counts + p * n_vec, h.data() + p * ldA, n_vec * 4);
    return ASNN_OK;
#endif
}

// eval_parallel(DeviceCompute) + read_outputs over a batch of host vectors.
int asnn_dev_activate(asnn_dev_layout* L, const float* x, uint32_t n_vec, uint64_t n_x, float* out,
                      float* state) {
    if (!L) return ASNN_E_INVALID;
    asnn_dev* dev = L->dev;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    // eval.cpp:26-28 -- arity check (per vector, all networks).
    if (n_x != static_cast<uint64_t>(L->total_in) * n_vec)
        return fail(dev, ASNN_E_ARITY,
                    "expected " + std::to_string(static_cast<uint64_t>(L->total_in) * n_vec) +
                        " input values, got " + std::to_string(n_x));
    if (n_vec == 0) return ASNN_OK;
    if (!x && n_x) return fail(dev, ASNN_E_INVALID, "null input");
    CK(cudaSetDevice(dev->device));
    cudaStream_t st = dev->stream;
    const size_t xb = static_cast<size_t>(n_x) * 4;
    const size_t ob = static_cast<size_t>(L->total_out) * n_vec * 4;
    CK(L->x_stage.ensure(n_x ? n_x : 1));
    CK(L->out_stage.ensure(static_cast<size_t>(L->total_out) * n_vec + 1));
    DevBuf<float> state_dev;
    if (state) CK(state_dev.alloc(static_cast<size_t>(L->total_idb) * n_vec));
    // zero-copy: page-locked, mapped inputs / outputs used in place by the
    // sweep's kernels (one graph launch, no copy operations; K-cta's reads and
    // writes overlap the other CTAs' sweeps)
    if (!state) {
        void* xd = xb ? mapped_device_ptr(x) : nullptr;
        void* od = (out && ob) ? mapped_device_ptr(out) : nullptr;
        if ((xd || !xb) && (od || !(out && ob))) {
            // no events on this latency-critical path: activate_ms is the
            // call's wall time (it includes the launch and the wait)
            const auto t0 = std::chrono::steady_clock::now();
            int rc = run_sweep(L, static_cast<const float*>(xd), n_vec, static_cast<float*>(od), nullptr);
            if (rc) return rc;
            CK(cudaStreamSynchronize(st));
            dev->timings.activate_ms =
                std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
            return ASNN_OK;
        }
    }
    CK(cudaEventRecord(dev->ev0, st));
    if (xb) {
        const float* src = x;
        if (!is_pinned(x)) {
            CK(dev->pin_x.ensure(xb));
            std::memcpy(dev->pin_x.p, x, xb);
            src = static_cast<const float*>(dev->pin_x.p);
        }
        CK(cudaMemcpyAsync(L->x_stage.p, src, xb, cudaMemcpyHostToDevice, st));
    }
    int rc = run_sweep(L, L->x_stage.p, n_vec, out ? L->out_stage.p : nullptr,
                       state ? state_dev.p : nullptr);
    if (rc) return rc;
    bool stage_out = false;
    if (out && ob) {
        if (is_pinned(out)) {
            CK(cudaMemcpyAsync(out, L->out_stage.p, ob, cudaMemcpyDeviceToHost, st));
        } else {
            CK(dev->pin_out.ensure(ob));
            CK(cudaMemcpyAsync(dev->pin_out.p, L->out_stage.p, ob, cudaMemcpyDeviceToHost, st));
            stage_out = true;
        }
    }
    if (state)
        CK(cudaMemcpyAsync(state, state_dev.p, static_cast<size_t>(L->total_idb) * n_vec * 4,
                           cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(dev->ev1, st));
    CK(cudaEventSynchronize(dev->ev1));
    if (stage_out) std::memcpy(out, dev->pin_out.p, ob);
    cudaEventElapsedTime(&dev->timings.activate_ms, dev->ev0, dev->ev1);
    return ASNN_OK;
}


// ---------------------------------------------------------------------------
// Resident server (serve.cuh): the batch-1 latency path.
struct asnn_dev_server {
    asnn_dev_layout* L = nullptr;
    cudaStream_t st = nullptr;
    ServeCtl* ctl = nullptr;    // phase stamps (page-locked, mapped)
    uint64_t* in_h = nullptr;   // [1 + max_vec * n_in] flagged records (page-locked, mapped)
    uint64_t* out_h = nullptr;  // [max_vec * n_out]
    uint32_t max_vec = 1, n_in = 0, n_out = 0, seq = 0;
    double last_ns = 0;  // host round trip of the last activation (records out -> records back)
    std::mutex mu;
};

namespace {
void server_release(asnn_dev_server* s) {
    if (s->st) cudaStreamDestroy(s->st);
    if (s->ctl) cudaFreeHost(s->ctl);
    if (s->in_h) cudaFreeHost(s->in_h);
    if (s->out_h) cudaFreeHost(s->out_h);
    delete s;
}
inline void put_rec(uint64_t* p, uint32_t v, uint32_t seq) {
    *reinterpret_cast<volatile uint64_t*>(p) = static_cast<uint64_t>(seq) << 32 | v;
}
// host side of a request: every input slot (unused ones zero) and the header
// carry seq, so each device thread's poll of its own record completes
void server_post(asnn_dev_server* s, const float* x, uint32_t n_vec, uint32_t hdr) {
    const uint32_t q = ++s->seq;
    const uint32_t used = n_vec * s->n_in, slots = s->max_vec * s->n_in;
    for (uint32_t k = 0; k < slots; ++k) {
        uint32_t v = 0;
        if (k < used) std::memcpy(&v, x + k, 4);
        put_rec(s->in_h + 1 + k, v, q);
    }
    put_rec(s->in_h, hdr, q);
}
}  // namespace

int asnn_dev_server_start(asnn_dev_layout* L, uint32_t max_vec, asnn_dev_server** out) {
    if (!L || !out || max_vec == 0 || max_vec > 64) return ASNN_E_INVALID;
    *out = nullptr;
    asnn_dev* dev = L->dev;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    if (L->server) return fail(dev, ASNN_E_INVALID, "layout already has a live server");
    if (L->nets.size() != 1) return fail(dev, ASNN_E_UNAVAILABLE, "the resident server takes one network");
    const NetMeta& n = L->nets[0];
    const uint32_t bytes = serve::smem_bytes(n.n_pos, L->total_edges, n.n_sensors, n.n_out, n.n_layers, max_vec);
    if (bytes > kMaxDynSmem - 4096)
        return fail(dev, ASNN_E_UNAVAILABLE,
                    "network too large for one SM's shared memory (" + std::to_string(bytes) + " bytes)");
    if (static_cast<uint64_t>(max_vec) * L->total_in > 511)
        return fail(dev, ASNN_E_UNAVAILABLE, "more than 511 input values per request");
    CK(cudaSetDevice(dev->device));
    auto* s = new asnn_dev_server;
    s->L = L;
    s->max_vec = max_vec;
    s->n_in = L->total_in;
    s->n_out = L->total_out;
    cudaError_t e;
    auto bail = [&](cudaError_t err, const char* what) {
        server_release(s);
        return cuda_fail(dev, err, what);
    };
    const size_t in_n = 1 + static_cast<size_t>(max_vec) * s->n_in, out_n = std::max<size_t>(1, max_vec * s->n_out);
    if ((e = cudaHostAlloc(&s->ctl, sizeof(ServeCtl), cudaHostAllocMapped)) != cudaSuccess) return bail(e, "ctl");
    if ((e = cudaHostAlloc(&s->in_h, 8 * in_n, cudaHostAllocMapped)) != cudaSuccess) return bail(e, "in");
    if ((e = cudaHostAlloc(&s->out_h, 8 * out_n, cudaHostAllocMapped)) != cudaSuccess) return bail(e, "out");
    std::memset(s->ctl, 0, sizeof(ServeCtl));
    std::memset(s->in_h, 0, 8 * in_n);
    std::memset(s->out_h, 0, 8 * out_n);
    void *ctl_d, *in_d, *out_d;
    if ((e = cudaHostGetDevicePointer(&ctl_d, s->ctl, 0)) != cudaSuccess) return bail(e, "ctl map");
    if ((e = cudaHostGetDevicePointer(&in_d, s->in_h, 0)) != cudaSuccess) return bail(e, "in map");
    if ((e = cudaHostGetDevicePointer(&out_d, s->out_h, 0)) != cudaSuccess) return bail(e, "out map");
    if ((e = cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking)) != cudaSuccess) return bail(e, "stream");
    // the layout's arrays are complete on the handle's stream before the server starts
    if ((e = cudaStreamSynchronize(dev->stream)) != cudaSuccess) return bail(e, "sync");
    auto fn = L->zero_refs ? k_serve<true> : k_serve<false>;
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes))) !=
        cudaSuccess)
        return bail(e, "smem attribute");
    // batch 1: a finish half and a prefix half (serve.cuh)
    const uint32_t T = std::min<uint32_t>(
        512, std::max<uint32_t>({64, (max_vec == 1 ? 2 : 1) * ((L->max_width * max_vec + 31) / 32 * 32),
                                 static_cast<uint32_t>((in_n + 31) / 32 * 32)}));
    fn<<<1, T, bytes, s->st>>>(reinterpret_cast<const CtaNet*>(L->cta_nets.p), L->lo_cat.p, L->row_ptr.p,
                               L->edges.p, L->sinfo.p, L->oinfo.p, static_cast<ServeCtl*>(ctl_d),
                               static_cast<const uint2*>(in_d), static_cast<uint2*>(out_d), max_vec);
    if ((e = cudaGetLastError()) != cudaSuccess) return bail(e, "k_serve launch");
    L->server = s;
    *out = s;
    return ASNN_OK;
}

int asnn_dev_server_activate(asnn_dev_server* s, const float* x, uint32_t n_vec, uint64_t n_x, float* out) {
    if (!s) return ASNN_E_INVALID;
    asnn_dev* dev = s->L->dev;
    std::lock_guard<std::mutex> lk(s->mu);
    if (n_x != static_cast<uint64_t>(s->n_in) * n_vec) {
        std::lock_guard<std::recursive_mutex> lk2(dev->mu);
        return fail(dev, ASNN_E_ARITY,
                    "expected " + std::to_string(static_cast<uint64_t>(s->n_in) * n_vec) + " input values, got " +
                        std::to_string(n_x));
    }
    if (n_vec == 0) return ASNN_OK;
    if (n_vec > s->max_vec || (!x && n_x) || (!out && s->n_out)) {
        std::lock_guard<std::recursive_mutex> lk2(dev->mu);
        return fail(dev, ASNN_E_INVALID, "batch larger than the server's max_vec, or null buffer");
    }
    const auto t0 = std::chrono::steady_clock::now();
    server_post(s, x, n_vec, n_vec);
    const uint32_t q = s->seq;
    const uint32_t m = n_vec * s->n_out;
    const volatile uint64_t* rec = s->out_h;
    // spin on the device's flagged outputs; every 64k polls check the kernel is alive
    uint64_t spins = 0;
    for (uint32_t j = 0; j < m; ++j) {
        uint64_t r;
        while (((r = rec[j]) >> 32) != q) {
            if ((++spins & 0xFFFF) == 0) {
                const cudaError_t e = cudaStreamQuery(s->st);
                if (e != cudaErrorNotReady) {
                    std::lock_guard<std::recursive_mutex> lk2(dev->mu);
                    return cuda_fail(dev, e == cudaSuccess ? cudaErrorLaunchFailure : e, "resident server stopped");
                }
            }
#if defined(__x86_64__)
            __builtin_ia32_pause();
#endif
        }
        const uint32_t v = static_cast<uint32_t>(r);
        std::memcpy(out + j, &v, 4);
    }
    s->last_ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
    return ASNN_OK;
}

int asnn_dev_server_timings(asnn_dev_server* s, double* host_ns, int64_t* device_cycles) {
    if (!s) return ASNN_E_INVALID;
    std::lock_guard<std::mutex> lk(s->mu);
    if (host_ns) *host_ns = s->last_ns;
    if (device_cycles) {
        volatile ServeCtl* c = s->ctl;
        device_cycles[0] = c->t_sens;
        device_cycles[1] = c->t_layers;
        device_cycles[2] = c->t_out;
        device_cycles[3] = c->t_wait;
        device_cycles[4] = c->t_dbg0;
        device_cycles[5] = c->t_dbg1;
        device_cycles[6] = c->t_dbg2;
        device_cycles[7] = c->t_dbg3;
    }
    return ASNN_OK;
}

void asnn_dev_server_stop(asnn_dev_server* s) {
    if (!s) return;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        server_post(s, nullptr, 0, kServeStop);
        cudaStreamSynchronize(s->st);
    }
    if (s->L) s->L->server = nullptr;
    server_release(s);
}

}  // extern "C"
