// once.cu -- eval_parallel of a layout that lives for ONE call (the per-call
// drop-in, eval.cpp:49-80 behind the seam at :51-52).
//
// The reference hands every eval_parallel call a host LayeredLayout and the
// caller may mutate it between calls (asnn_main.cpp:264-278), so nothing can
// be kept on the device across calls.  The resident path (engine.cu:
// upload_layout -> renumbering, schedules, CUDA graphs) pays ~200 us of fixed
// cost for structures that only amortise over many sweeps; this path keeps
// the reference's own id-indexed state and runs the whole call as
//
//   caller writes the CSR straight into page-locked staging (asnn_eval_buf_stage)
//   -> mode 0 [small, or deep and fitting one SM]: one CTA pulls the staged
//               layout over PCIe into shared memory (zero-copy cp.async) and
//               sweeps the layers there, __syncthreads between layers
//   -> mode 5 [medium, <= 24 layers] / mode 6 [medium, deeper]: an 8-CTA
//               cluster pulls its shares of the staged layout over PCIe into
//               distributed shared memory, every CTA keeping a copy of the
//               state (DSMEM stores); shares of every layer and a cluster
//               barrier per layer (5), or ranges of whole layers and a
//               barrier per range (6)
//   -> mode 1 [state fits one SM]: one DMA, then one CTA with the state in
//               shared memory and cp.async rings of the next items
//   -> mode 2 / 4 [large, shallow / deep]: one DMA, then one cooperative grid
//               with the state in L2, grid.sync() between layers (with / without
//               the rings); mode 3 = mode 1 without the rings (experiments)
//   -> state.outputs written by the kernel into mapped host memory.
//
// Arithmetic is activate_node (eval.cpp:16-23): the stored predecessor order,
// __fmul_rn / __fadd_rn (no contraction), sigmoid32 bit for bit; sensors
// (layer 0) take sigmoid32(inputs[id]) where the caller did make_state
// (eval.cpp:25-35) and staged inputs[id] per sensor.  Malformed layouts
// (ids or predecessors >= id_bound, row_ptr out of order) are flagged by the
// kernel without any out-of-bounds access and reported as ASNN_E_INVALID.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "engine.hpp"

using namespace asnn_b200;
namespace cg = cooperative_groups;

namespace {

constexpr uint32_t kSmemCap = 227 * 1024;

// Byte offsets of the staged arrays inside the blob (16-byte aligned).
struct OnceOff {
    uint32_t lo, ids, rp, src, w, sx, bytes;
};

struct OnceArgs {
    const uint8_t* blob;  // staged layout: mapped host (mode 0) or device copy
    OnceOff off;
    float* op;            // [idb] state in global memory (mode 2)
    float* out;           // [idb] state.outputs, mapped host memory
    uint32_t* err;        // mapped host flag
    uint32_t L, N, idb, ns;
    uint32_t E;
};

__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p, bool global_ro) {
    return global_ro ? __ldg(p) : *p;
}

// kMode 0: blob in mapped host memory, copied into shared memory by the CTA
//          (followed by the state); everything after the copy is on-chip.
// kMode 1: blob in device memory (one DMA); state in shared memory.
// kMode 2: blob in device memory; state in global memory (L2), grid-wide.
template <int kMode>
__global__ void __launch_bounds__(1024) k_once(const OnceArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nthr = gridDim.x * blockDim.x;
    const uint32_t op_bytes = (a.idb * 4 + 15) & ~15u;
    float* op = kMode == 2 ? a.op : reinterpret_cast<float*>(smem);
    const uint8_t* base = a.blob;
    if constexpr (kMode == 0) {
        // zero-copy pull of the staged layout: independent 16-byte loads
        const uint4* s = reinterpret_cast<const uint4*>(a.blob);
        uint4* d = reinterpret_cast<uint4*>(smem + op_bytes);
        for (uint32_t i = threadIdx.x; i < a.off.bytes / 16; i += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(d + i))),
                         "l"(s + i)
                         : "memory");
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
        base = smem + op_bytes;
    }
    constexpr bool ro = kMode != 0;
    const uint32_t* lo = reinterpret_cast<const uint32_t*>(base + a.off.lo);
    const uint32_t* ids = reinterpret_cast<const uint32_t*>(base + a.off.ids);
    const uint32_t* rp = reinterpret_cast<const uint32_t*>(base + a.off.rp);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(base + a.off.src);
    const float* w = reinterpret_cast<const float*>(base + a.off.w);
    const float* sx = reinterpret_cast<const float*>(base + a.off.sx);

    auto sync = [] {
        if constexpr (kMode == 2) cg::this_grid().sync();
        else __syncthreads();
    };
    // the state read another CTA wrote: L2 only (L1 is not coherent)
    auto rd = [&](uint32_t u) -> float {
        if constexpr (kMode == 2) return __ldcg(op + u);
        else return op[u];
    };

    for (uint32_t i = tid; i < a.idb; i += nthr) op[i] = 0.0f;  // make_state: outputs zero
    sync();
    uint32_t bad = 0;
    // layer 0: sensors, sigmoid32(inputs[id]) (eval.cpp:17)
    for (uint32_t i = tid; i < a.ns; i += nthr) {
        const uint32_t id = ld_u32(ids + i, ro);
        const float v = sigmoid32(ro ? __ldg(sx + i) : sx[i]);
        if (id < a.idb) op[id] = v;
        else bad = 1;
    }
    for (uint32_t l = 1; l < a.L; ++l) {
        sync();
        const uint32_t b = ld_u32(lo + l, ro), e = ld_u32(lo + l + 1, ro);
        for (uint32_t i = b + tid; i < e; i += nthr) {
            const uint32_t id = ld_u32(ids + i, ro);
            uint32_t k = ld_u32(rp + i, ro);
            uint32_t ke = ld_u32(rp + i + 1, ro);
            if (ke < k || ke > a.E) {
                bad = 1;
                ke = k;
            }
            float s = 0.0f;
            if constexpr (kMode == 2) {
                // state and edges in L2: predicated batches of 8, one dependent
                // round of L2 reads per 8 predecessors, the tail included
                for (; k < ke; k += 8) {
                    uint32_t u[8];
                    float wv[8], v[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const bool in = k + j < ke;
                        u[j] = in ? __ldg(src + k + j) : 0u;
                        wv[j] = in ? __ldg(w + k + j) : 0.0f;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const bool in = k + j < ke;
                        bad |= in && u[j] >= a.idb;
                        v[j] = in && u[j] < a.idb ? rd(u[j]) : 0.0f;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (k + j < ke) s = __fadd_rn(s, __fmul_rn(wv[j], v[j]));
                }
            }
            // predecessors in the stored order; four loads ahead of the chain
            for (; k + 4 <= ke; k += 4) {
                uint32_t u[4];
                float wv[4], v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    u[j] = ld_u32(src + k + j, ro);
                    wv[j] = ro ? __ldg(w + k + j) : w[k + j];
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    bad |= u[j] >= a.idb;
                    v[j] = u[j] < a.idb ? rd(u[j]) : 0.0f;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) s = __fadd_rn(s, __fmul_rn(wv[j], v[j]));
            }
            for (; k < ke; ++k) {
                const uint32_t u = ld_u32(src + k, ro);
                const float wk = ro ? __ldg(w + k) : w[k];
                bad |= u >= a.idb;
                s = __fadd_rn(s, __fmul_rn(wk, u < a.idb ? rd(u) : 0.0f));
            }
            const float y = sigmoid32(s);
            if (id < a.idb) op[id] = y;
            else bad = 1;
        }
    }
    sync();
    for (uint32_t i = tid; i < a.idb; i += nthr) a.out[i] = kMode == 2 ? __ldcg(op + i) : op[i];
    if (bad) *reinterpret_cast<volatile uint32_t*>(a.err) = 1u;
}

// ---- pipelined sweep (modes 1 and 2) ---------------------------------------
// The layers are cut into items of T consecutive nodes (one node per thread).
// A CTA walks its items (mode 1: all of them; mode 2: chunk k of layer l goes
// to CTA k mod G) with a seven-slot ring of row_ptr / id slices and a
// four-slot ring of edge slices in shared memory, filled by cp.async: while
// item t is summed, items t+1..t+3's edges and t+1..t+6's row_ptr / ids are in
// flight (one cp.async group per item, waited two items behind; the staged
// layout is first prefetched into L2), so the dependent
// chain of an item touches shared memory only (and the state: shared in mode
// 1, L2 in mode 2).  Items whose edges exceed a slot read them from global
// memory instead.  The layer table sits in shared memory when it fits.
__device__ __forceinline__ void cpa4(void* d, const void* s) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(d))),
                 "l"(s)
                 : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_2() { asm volatile("cp.async.wait_group 2;" ::: "memory"); }

struct Item {
    uint32_t l, k;  // layer, chunk within the layer; l >= L: none
};

constexpr uint32_t kLoSmem = 4096;  // layer-table entries kept in shared memory
// prefetch distances (items): edges kDE ahead, row_ptr / ids kDM ahead; an
// item's copies must land within kDE - 1 items (cp.async.wait_group kDE - 1)
constexpr uint32_t kDE = 3, kDM = kDE + 3, kES = kDE + 1, kMS = kDM + 1;

__host__ __device__ constexpr uint32_t pipe_ring_bytes(uint32_t T, uint32_t L) {
    return 4 * (kMS * (T + 1) + kMS * T + 1) + 4 * ((L + 1 <= kLoSmem ? L + 1 : 0) + 3) / 4 * 4;
}

template <bool kGrid>
__global__ void __launch_bounds__(512) k_once_pipe(const OnceArgs a, uint32_t ecap, uint32_t tsh) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t T = 1u << tsh, t = threadIdx.x;  // blockDim.x == T
    const uint32_t G = kGrid ? gridDim.x : 1u, c = kGrid ? blockIdx.x : 0u;
    const uint32_t op_bytes = kGrid ? 0u : (a.idb * 4 + 15) & ~15u;
    float* op = kGrid ? a.op : reinterpret_cast<float*>(smem);
    uint32_t* rp_s = reinterpret_cast<uint32_t*>(smem + op_bytes);  // [kMS][T + 1]
    uint32_t* id_s = rp_s + kMS * (T + 1);                            // [kMS][T]
    uint32_t* lo_s = id_s + kMS * T + 1;                              // [L + 1] when it fits
    const bool lo_in_smem = a.L + 1 <= kLoSmem;
    uint32_t* es = lo_s + (lo_in_smem ? (a.L + 1 + 3) / 4 * 4 : 0);   // [kES][ecap] sources
    float* ew = reinterpret_cast<float*>(es + kES * ecap);            // [kES][ecap] weights
    const uint32_t* lo_g = reinterpret_cast<const uint32_t*>(a.blob + a.off.lo);
    const uint32_t* ids = reinterpret_cast<const uint32_t*>(a.blob + a.off.ids);
    const uint32_t* rp = reinterpret_cast<const uint32_t*>(a.blob + a.off.rp);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.blob + a.off.src);
    const float* w = reinterpret_cast<const float*>(a.blob + a.off.w);
    const float* sx = reinterpret_cast<const float*>(a.blob + a.off.sx);
    const uint32_t gt = c * T + t, nthr = G * T;
    // the staged layout into L2 first (one DMA put it in HBM): the rings'
    // copies then wait on L2, not DRAM
    for (uint32_t o = gt * 16384u; o < a.off.bytes; o += nthr * 16384u)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.blob + o), "r"(min(16384u, a.off.bytes - o))
                     : "memory");
    if (lo_in_smem)
        for (uint32_t i = t; i <= a.L; i += T) lo_s[i] = __ldg(lo_g + i);
    __syncthreads();
    const uint32_t* lo = lo_in_smem ? lo_s : lo_g;

    auto nch = [&](uint32_t l) { return (lo[l + 1] - lo[l] + T - 1) >> tsh; };
    auto norm = [&](Item it) {
        while (it.l < a.L && it.k >= nch(it.l)) {
            ++it.l;
            it.k = c;
        }
        return it;
    };
    auto next = [&](Item it) { return it.l < a.L ? norm(Item{it.l, it.k + G}) : it; };
    auto span = [&](Item it, uint32_t& b, uint32_t& n) {
        b = lo[it.l] + (it.k << tsh);
        n = min(T, lo[it.l + 1] - b);
    };
    auto meta = [&](Item it, uint32_t slot) {
        if (it.l >= a.L) return;
        uint32_t b, n;
        span(it, b, n);
        for (uint32_t j = t; j <= n; j += T) cpa4(rp_s + slot * (T + 1) + j, rp + b + j);
        for (uint32_t j = t; j < n; j += T) cpa4(id_s + slot * T + j, ids + b + j);
    };
    // edges of an item whose row_ptr slice is in `slot`; false: read globally
    auto staged = [&](Item it, uint32_t slot, uint32_t& e0, uint32_t& m) {
        uint32_t b, n;
        span(it, b, n);
        e0 = rp_s[slot * (T + 1)];
        const uint32_t e1 = rp_s[slot * (T + 1) + n];
        m = e1 - e0;
        return e1 >= e0 && e1 <= a.E && e1 - e0 <= ecap;
    };
    auto edges = [&](Item it, uint32_t slot, uint32_t eslot) {
        if (it.l >= a.L) return;
        uint32_t e0, m;
        if (!staged(it, slot, e0, m)) return;
        for (uint32_t j = t; j < m; j += T) {
            cpa4(es + eslot * ecap + j, src + e0 + j);
            cpa4(ew + eslot * ecap + j, w + e0 + j);
        }
    };
    auto layer_sync = [&] {
        if constexpr (kGrid) cg::this_grid().sync();
        else __syncthreads();
    };
    auto rd = [&](uint32_t u) -> float {
        if constexpr (kGrid) return __ldcg(op + u);
        else return op[u];
    };

    // items t .. t+kDM of this CTA
    Item i0 = norm(Item{1, c});
    Item i1 = next(i0), i2 = next(i1), i3 = next(i2), i4 = next(i3), i5 = next(i4);
    meta(i0, 0);
    meta(i1, 1);
    meta(i2, 2);
    meta(i3, 3);
    meta(i4, 4);
    meta(i5, 5);
    cpa_commit();
    for (uint32_t i = gt; i < a.idb; i += nthr) op[i] = 0.0f;  // make_state: outputs zero
    layer_sync();
    uint32_t bad = 0;
    for (uint32_t i = gt; i < a.ns; i += nthr) {  // layer 0: sensors (eval.cpp:17)
        const uint32_t id = __ldg(ids + i);
        const float v = sigmoid32(__ldg(sx + i));
        if (id < a.idb) op[id] = v;
        else bad = 1;
    }
    cpa_wait_all();
    layer_sync();
    edges(i0, 0, 0);
    edges(i1, 1, 1);
    edges(i2, 2, 2);
    cpa_commit();
    // layers with no item of this CTA before its first one
    if constexpr (kGrid)
        for (uint32_t l = 1; l < min(i0.l, a.L); ++l) layer_sync();
    cpa_wait_all();
    __syncthreads();
    // ring slots of item t: s0 (row_ptr / ids, of kMS = 7) and e_cur (edges, of kES = 4)
    for (uint32_t s0 = 0, e_cur = 0; i0.l < a.L;
         s0 = s0 == kMS - 1 ? 0 : s0 + 1, e_cur = e_cur == kES - 1 ? 0 : e_cur + 1) {
        const Item i6 = next(i5);
        meta(i6, s0 == 0 ? kMS - 1 : s0 - 1);                                  // (t + 6) mod 7
        edges(i3, s0 + 3 >= kMS ? s0 + 3 - kMS : s0 + 3, e_cur == 0 ? kES - 1 : e_cur - 1);  // t + 3
        cpa_commit();
        {
            uint32_t b, n, e0, m;
            span(i0, b, n);
            const bool st = staged(i0, s0, e0, m);
            if (t < n) {
                const uint32_t id = id_s[s0 * T + t];
                uint32_t k = rp_s[s0 * (T + 1) + t], ke = rp_s[s0 * (T + 1) + t + 1];
                if (ke < k || ke > a.E || (st && (k < e0))) {
                    bad = 1;
                    ke = k;
                }
                float sum = 0.0f;
                if (st) {
                    // state in L2 (mode 2): batches of 8 predicated loads, so a
                    // row's gathers cost one dependent L2 read per 8
                    // predecessors, the partial batch included (no add for the
                    // masked slots); mode 1 only runs its tail through it
                    const uint32_t* es_ = es + e_cur * ecap - e0;
                    const float* ew_ = ew + e_cur * ecap - e0;
                    constexpr int U = 8;
                    if constexpr (!kGrid) {
                        // state in shared memory: plain batches of 4 and a scalar tail
                        for (; k + 4 <= ke; k += 4) {
                            uint32_t u[4];
                            float wv[4], v[4];
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                u[j] = es_[k + j];
                                wv[j] = ew_[k + j];
                            }
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                bad |= u[j] >= a.idb;
                                v[j] = u[j] < a.idb ? rd(u[j]) : 0.0f;
                            }
#pragma unroll
                            for (int j = 0; j < 4; ++j) sum = __fadd_rn(sum, __fmul_rn(wv[j], v[j]));
                        }
                    }
                    for (; k < ke; k += U) {
                        uint32_t u[U];
                        float wv[U], v[U];
#pragma unroll
                        for (int j = 0; j < U; ++j) {
                            const bool in = k + j < ke;
                            u[j] = in ? es_[k + j] : 0u;
                            wv[j] = in ? ew_[k + j] : 0.0f;
                        }
#pragma unroll
                        for (int j = 0; j < U; ++j) {
                            const bool in = k + j < ke;
                            bad |= in && u[j] >= a.idb;
                            v[j] = in && u[j] < a.idb ? rd(u[j]) : 0.0f;
                        }
#pragma unroll
                        for (int j = 0; j < U; ++j)
                            if (k + j < ke) sum = __fadd_rn(sum, __fmul_rn(wv[j], v[j]));
                    }
                } else {
                    for (; k < ke; ++k) {
                        const uint32_t u = __ldg(src + k);
                        bad |= u >= a.idb;
                        sum = __fadd_rn(sum, __fmul_rn(__ldg(w + k), u < a.idb ? rd(u) : 0.0f));
                    }
                }
                const float y = sigmoid32(sum);
                if (id < a.idb) op[id] = y;
                else bad = 1;
            }
        }
        if constexpr (kGrid) {
            const uint32_t to = i1.l < a.L ? i1.l : a.L;
            for (uint32_t l = i0.l; l < to; ++l) layer_sync();
        }
        cpa_wait_2();  // copies issued two items ago and earlier; the last two items' fly on
        __syncthreads();
        i0 = i1;
        i1 = i2;
        i2 = i3;
        i3 = i4;
        i4 = i5;
        i5 = i6;
    }
    cpa_wait_all();
    __syncthreads();
    for (uint32_t i = gt; i < a.idb; i += nthr) a.out[i] = kGrid ? __ldcg(op + i) : op[i];
    if (bad) *reinterpret_cast<volatile uint32_t*>(a.err) = 1u;
}

// ---- mode 5: a cluster of CTAs holding the layout in distributed shared memory
// Each of the kC CTAs of one thread-block cluster owns a contiguous 1/kC of
// every layer's nodes.  At start every CTA pulls its share of the staged
// layout (ids, row_ptr, predecessor ids / weights, sensor inputs) straight
// from page-locked host memory into its own shared memory (cp.async, no DMA
// operation); it keeps a full copy of the id-indexed state.  Per layer each
// CTA sums its nodes from shared memory and stores every result into all kC
// copies of the state (st.shared::cluster through DSMEM), then one cluster
// barrier.  The host plans the shares: per (CTA, layer) {first node, nodes,
// first edge, edges, node offset, edge offset} in shared memory.
constexpr uint32_t kC = 8;

struct PlanEnt {
    uint32_t a, n, ea, m, noff, eoff, pad0, pad1;
};

struct LayerRanges {
    uint32_t b[kC + 1];  // mode 6: CTA r owns layers [b[r], b[r+1]); b[0] == kNoRanges: mode 5
};
constexpr uint32_t kNoRanges = 0xFFFFFFFFu;

__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(256) k_once_cluster(const OnceArgs a, const PlanEnt* plan,
                                                                                 uint32_t n_loc, uint32_t e_loc,
                                                                                 const LayerRanges rg) {
    extern __shared__ __align__(16) uint8_t smem[];
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t r = cl.block_rank(), t = threadIdx.x, T = blockDim.x;
    const uint32_t op_bytes = (a.idb * 4 + 15) & ~15u;
    float* op = reinterpret_cast<float*>(smem);
    PlanEnt* pl = reinterpret_cast<PlanEnt*>(smem + op_bytes);             // [L]
    uint32_t* lid = reinterpret_cast<uint32_t*>(pl + a.L);                  // [n_loc]
    uint32_t* lrp = lid + n_loc;                                            // [n_loc + L]
    uint32_t* les = lrp + n_loc + a.L;                                      // [e_loc]
    float* lew = reinterpret_cast<float*>(les + e_loc);                     // [e_loc]
    float* lsx = lew + e_loc;                                               // [layer-0 share]
    const uint32_t* ids = reinterpret_cast<const uint32_t*>(a.blob + a.off.ids);
    const uint32_t* rp = reinterpret_cast<const uint32_t*>(a.blob + a.off.rp);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.blob + a.off.src);
    const float* w = reinterpret_cast<const float*>(a.blob + a.off.w);
    const float* sx = reinterpret_cast<const float*>(a.blob + a.off.sx);

    for (uint32_t i = t; i < a.L * 8; i += T)
        cpa4(reinterpret_cast<uint32_t*>(pl) + i, reinterpret_cast<const uint32_t*>(plan + static_cast<size_t>(r) * a.L) + i);
    cpa_commit();
    for (uint32_t i = t; i < a.idb; i += T) op[i] = 0.0f;  // make_state: outputs zero
    cpa_wait_all();
    __syncthreads();
    // this CTA's share of the layout, over PCIe into shared memory
    for (uint32_t l = 0; l < a.L; ++l) {
        const PlanEnt e = pl[l];
        for (uint32_t j = t; j < e.n; j += T) {
            cpa4(lid + e.noff + j, ids + e.a + j);
            if (l == 0) cpa4(lsx + j, sx + e.a + j);
        }
        if (l > 0) {
            for (uint32_t j = t; j <= e.n; j += T) cpa4(lrp + e.noff + l + j, rp + e.a + j);
            for (uint32_t j = t; j < e.m; j += T) {
                cpa4(les + e.eoff + j, src + e.ea + j);
                cpa4(lew + e.eoff + j, w + e.ea + j);
            }
        }
    }
    cpa_commit();
    cpa_wait_all();
    cl.sync();  // every copy of the state zeroed before any remote store
    uint32_t bad = 0;
    // this CTA's nodes of layer l; every result goes into all kC copies
    auto layer = [&](uint32_t l, bool bcast) {
        const PlanEnt e = pl[l];
        for (uint32_t j = t; j < e.n; j += T) {
            const uint32_t id = lid[e.noff + j];
            float y;
            if (l == 0) {
                y = sigmoid32(lsx[j]);  // eval.cpp:17
            } else {
                uint32_t k = lrp[e.noff + l + j], ke = lrp[e.noff + l + j + 1];
                if (ke < k || k < e.ea || ke > e.ea + e.m) {
                    bad = 1;
                    ke = k = e.ea;
                }
                const uint32_t* s_ = les + e.eoff - e.ea;
                const float* w_ = lew + e.eoff - e.ea;
                float sum = 0.0f;
                for (; k + 4 <= ke; k += 4) {
                    uint32_t u[4];
                    float wv[4], v[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        u[q] = s_[k + q];
                        wv[q] = w_[k + q];
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        bad |= u[q] >= a.idb;
                        v[q] = u[q] < a.idb ? op[u[q]] : 0.0f;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) sum = __fadd_rn(sum, __fmul_rn(wv[q], v[q]));
                }
                for (; k < ke; ++k) {
                    const uint32_t u = s_[k];
                    bad |= u >= a.idb;
                    sum = __fadd_rn(sum, __fmul_rn(w_[k], u < a.idb ? op[u] : 0.0f));
                }
                y = sigmoid32(sum);
            }
            if (id < a.idb) {
                op[id] = y;
                if (bcast)
#pragma unroll
                    for (uint32_t q = 1; q < kC; ++q) cl.map_shared_rank(op, (r + q) % kC)[id] = y;
            } else {
                bad = 1;
            }
        }
    };
    if (rg.b[0] == kNoRanges) {
        // mode 5: every CTA takes 1/kC of every layer, one cluster barrier per layer
        for (uint32_t l = 0; l < a.L; ++l) {
            layer(l, true);
            cl.sync();
        }
    } else {
        // mode 6: CTA r runs its own contiguous range of layers (__syncthreads
        // between them, every result also stored into the other copies as it
        // is made); one cluster barrier per range hands the state on
        for (uint32_t q = 0; q < kC; ++q) {
            if (q == r)
                for (uint32_t l = rg.b[r]; l < rg.b[r + 1]; ++l) {
                    layer(l, true);
                    __syncthreads();
                }
            cl.sync();
        }
    }
    const uint32_t per = (a.idb + kC - 1) / kC, b0 = r * per, b1 = min(a.idb, b0 + per);
    for (uint32_t i = b0 + t; i < b1; i += T) a.out[i] = op[i];
    if (bad) *reinterpret_cast<volatile uint32_t*>(a.err) = 1u;
}

uint32_t align16(uint64_t b) { return static_cast<uint32_t>((b + 15) & ~15ull); }

// cudaFuncSetAttribute once per (kernel, device, size growth): the per-call
// path pays no attribute calls after the first of each size class
cudaError_t set_smem(const void* fn, int device, uint32_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, uint32_t>> set;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : set)
        if (e.first.first == fn && e.first.second == device) {
            if (e.second >= bytes) return cudaSuccess;
            const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            if (r == cudaSuccess) e.second = bytes;
            return r;
        }
    const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (r == cudaSuccess) set.push_back({{fn, device}, bytes});
    return r;
}

// device address of page-locked host memory, cached per allocation
template <class T>
cudaError_t mapped(const void* h, const void*& h_cached, T*& d_cached) {
    if (h == h_cached && d_cached) return cudaSuccess;
    void* d = nullptr;
    const cudaError_t r = cudaHostGetDevicePointer(&d, const_cast<void*>(h), 0);
    if (r == cudaSuccess) {
        h_cached = h;
        d_cached = static_cast<T*>(d);
    }
    return r;
}

}  // namespace

struct asnn_eval_buf {
    asnn_dev* dev = nullptr;
    asnn_eval_dims dims{};
    OnceOff off{};
    bool staged = false;
    PinnedBuf blob;            // page-locked (mapped) staging of the layout
    PinnedBuf plan;            // mode 5: per (CTA, layer) shares (mapped)
    uint8_t* dblob = nullptr;  // device copy (modes 1, 2)
    size_t dblob_bytes = 0;
    float* op = nullptr;       // global state (mode 2)
    size_t op_n = 0;
    float* out_h = nullptr;    // mapped state.outputs
    size_t out_n = 0;
    uint32_t* err_h = nullptr;
    uint32_t last_mode = 0;
    // device addresses of the mapped buffers (cached per allocation)
    const void *blob_h = nullptr, *plan_h = nullptr, *out_hc = nullptr, *err_hc = nullptr;
    const uint8_t* blob_d = nullptr;
    const void* plan_d = nullptr;
    float* out_d = nullptr;
    uint32_t* err_d = nullptr;
    ~asnn_eval_buf() {
        if (dblob) cudaFree(dblob);
        if (op) cudaFree(op);
        if (out_h) cudaFreeHost(out_h);
        if (err_h) cudaFreeHost(err_h);
    }
};

#define CK(expr)                                                 \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return cuda_fail(dev, _e, #expr); \
    } while (0)

extern "C" {

int asnn_eval_buf_create(asnn_dev* dev, asnn_eval_buf** out) {
    if (!dev || !out) return ASNN_E_INVALID;
    *out = nullptr;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    CK(cudaSetDevice(dev->device));
    auto* b = new asnn_eval_buf;
    b->dev = dev;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&b->err_h), 16, cudaHostAllocMapped);
    if (e != cudaSuccess) {
        b->err_h = nullptr;
        delete b;
        return cuda_fail(dev, e, "eval buffer flag");
    }
    *b->err_h = 0;
    *out = b;
    return ASNN_OK;
}

void asnn_eval_buf_free(asnn_eval_buf* b) {
    if (!b) return;
    std::lock_guard<std::recursive_mutex> lk(b->dev->mu);
    cudaSetDevice(b->dev->device);
    cudaStreamSynchronize(b->dev->stream);
    delete b;
}

int asnn_eval_buf_stage(asnn_eval_buf* b, const asnn_eval_dims* d, asnn_eval_stage* s) {
    if (!b || !d || !s) return ASNN_E_INVALID;
    asnn_dev* dev = b->dev;
    b->staged = false;
    if (d->edge_count >= 0xFFFFFFFFull) return fail(dev, ASNN_E_INVALID, "more than 2^32-1 edges");
    if (d->sensor_count > d->node_count) return fail(dev, ASNN_E_INVALID, "sensor_count > node_count");
    if (d->total_layers == 0 && d->node_count) return fail(dev, ASNN_E_INVALID, "layers missing");
    OnceOff o{};
    uint64_t at = 0;
    auto take = [&](uint64_t bytes) {
        const uint32_t r = static_cast<uint32_t>(at);
        at += align16(bytes);
        return r;
    };
    o.lo = take(4ull * (d->total_layers + 1));
    o.ids = take(4ull * d->node_count);
    o.rp = take(4ull * (d->node_count + 1));
    o.sx = take(4ull * d->sensor_count);
    o.src = take(4ull * d->edge_count);
    o.w = take(4ull * d->edge_count);
    if (at >= (1ull << 32)) return fail(dev, ASNN_E_INVALID, "layout too large for one call");
    o.bytes = static_cast<uint32_t>(at);
    {
        // page-locked staging is mapped for the zero-copy kernel (UVA)
        cudaSetDevice(dev->device);
        cudaError_t e = b->blob.ensure(std::max<uint64_t>(at, 64));
        if (e != cudaSuccess) return cuda_fail(dev, e, "eval staging");
    }
    uint8_t* p = static_cast<uint8_t*>(b->blob.p);
    s->layer_offsets = reinterpret_cast<uint32_t*>(p + o.lo);
    s->node_ids = reinterpret_cast<uint32_t*>(p + o.ids);
    s->row_ptr = reinterpret_cast<uint32_t*>(p + o.rp);
    s->in_nodes = reinterpret_cast<uint32_t*>(p + o.src);
    s->in_weights = reinterpret_cast<float*>(p + o.w);
    s->sensor_inputs = reinterpret_cast<float*>(p + o.sx);
    b->dims = *d;
    b->off = o;
    b->staged = true;
    return ASNN_OK;
}

int asnn_eval_buf_run(asnn_eval_buf* b, float* state_outputs) {
    if (!b) return ASNN_E_INVALID;
    asnn_dev* dev = b->dev;
    if (!b->staged) return fail(dev, ASNN_E_INVALID, "nothing staged");
    const asnn_eval_dims d = b->dims;
    if (d.id_bound && !state_outputs) return fail(dev, ASNN_E_INVALID, "null state");
    const uint8_t* hp = static_cast<const uint8_t*>(b->blob.p);
    const uint32_t* lo = reinterpret_cast<const uint32_t*>(hp + b->off.lo);
    const uint32_t* rp = reinterpret_cast<const uint32_t*>(hp + b->off.rp);
    // layer table on the host (L + 1 reads): the kernel indexes with it
    uint32_t max_w = 0;
    if (d.total_layers) {
        if (lo[0] != 0) return fail(dev, ASNN_E_INVALID, "layer_offsets[0] != 0");
        for (uint32_t l = 0; l < d.total_layers; ++l) {
            if (lo[l + 1] < lo[l]) return fail(dev, ASNN_E_INVALID, "layer_offsets decrease");
            max_w = std::max(max_w, lo[l + 1] - lo[l]);
        }
        if (lo[d.total_layers] != d.node_count)
            return fail(dev, ASNN_E_INVALID, "layer_offsets do not cover node_count");
        if (lo[1] != d.sensor_count) return fail(dev, ASNN_E_INVALID, "layer 0 size != sensor_count");
    }
    if (d.node_count && (rp[0] != 0 || rp[d.node_count] != d.edge_count))
        return fail(dev, ASNN_E_INVALID, "row_ptr does not span the edges");

    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    CK(cudaSetDevice(dev->device));
    cudaStream_t st = dev->stream;
    const uint32_t idb = d.id_bound;
    if (idb == 0) {
        if (d.node_count) return fail(dev, ASNN_E_INVALID, "malformed layout: nodes with id_bound 0");
        return ASNN_OK;
    }
    if (b->out_n < idb) {
        if (b->out_h) cudaFreeHost(b->out_h);
        b->out_h = nullptr;
        b->out_n = 0;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&b->out_h), 4ull * idb, cudaHostAllocMapped));
        b->out_n = idb;
    }
    // write the state straight into the caller's buffer when it is page-locked
    float* out_dev = nullptr;
    {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, state_outputs) == cudaSuccess && pa.type == cudaMemoryTypeHost)
            out_dev = static_cast<float*>(pa.devicePointer);
        cudaGetLastError();
    }
    const bool direct = out_dev != nullptr;
    if (!direct) {
        CK(mapped(b->out_h, b->out_hc, b->out_d));
        out_dev = b->out_d;
    }
    CK(mapped(b->err_h, b->err_hc, b->err_d));
    uint32_t* err_dev = b->err_d;
    *reinterpret_cast<volatile uint32_t*>(b->err_h) = 0;

    const uint32_t op_bytes = align16(4ull * idb);
    const uint32_t blob = b->off.bytes;
    // mode: 0 = zero-copy into shared memory, 1 = DMA + one CTA (state in
    // shared memory, pipelined), 2 = DMA + cooperative grid (state in L2,
    // pipelined); 3 / 4 = 1 / 2 without the cp.async rings (experiments)
    uint32_t t1sh = 6;  // one-CTA item width: a power of two in [64, 512] covering the widest layer
    while (t1sh < 9 && (1u << t1sh) < max_w) ++t1sh;
    const uint32_t T1 = 1u << t1sh;
    const uint32_t ring1 = pipe_ring_bytes(T1, d.total_layers);
    const uint32_t fit1 = kSmemCap - 1024 > op_bytes + ring1 ? (kSmemCap - 1024 - op_bytes - ring1) / (8 * kES) : 0;
    // cluster plans.  Mode 5: each CTA takes a contiguous 1/kC of every layer
    // (one cluster barrier per layer: shallow layouts).  Mode 6: each CTA
    // takes a contiguous range of layers, split by bytes (one barrier per
    // range: deep layouts).  Feasible when every share plus a full state fits
    // shared memory.
    uint32_t n_max = 0, e_max = 0, s_max = 0, smem5 = 0;
    bool fit5 = false;
    LayerRanges rg{};
    rg.b[0] = kNoRanges;
    const uint64_t plan_bytes = static_cast<uint64_t>(kC) * d.total_layers * sizeof(PlanEnt);
    // one CTA pulls the whole layout: small layouts, and deep ones that fit
    // (its per-layer step is the cheapest; wide shallow ones pull faster with 8 CTAs)
    const bool fit0 = op_bytes + static_cast<uint64_t>(blob) <= kSmemCap - 1024 &&
                      (blob <= (96u << 10) || d.total_layers > 24);
    const char* force = getenv("ASNN_ONCE_MODE");
    const int forced = force ? atoi(force) : -1;
    const bool ranges = forced == 6 || (forced != 5 && d.total_layers > 24);
    if ((!fit0 || forced == 5 || forced == 6) && d.total_layers && plan_bytes <= (64u << 10) &&
        op_bytes + d.total_layers * sizeof(PlanEnt) < kSmemCap) {
        CK(b->plan.ensure(plan_bytes));
        PlanEnt* pe = static_cast<PlanEnt*>(b->plan.p);
        bool ok = true;
        for (uint32_t l = 1; l < d.total_layers && ok; ++l)
            ok = rp[lo[l + 1]] >= rp[lo[l]] && rp[lo[l + 1]] <= d.edge_count;  // else the other variants report it
        if (ok && ranges) {
            // layers [rg.b[r], rg.b[r+1]) to CTA r: close a range once it holds
            // 1/kC of the bytes (ids, row_ptr, edges)
            auto cost = [&](uint32_t l) -> uint64_t {
                const uint64_t n = lo[l + 1] - lo[l];
                return 8 * n + 4 + (l ? 8ull * (rp[lo[l + 1]] - rp[lo[l]]) : 4 * n);
            };
            uint64_t total = 0;
            for (uint32_t l = 0; l < d.total_layers; ++l) total += cost(l);
            const uint64_t target = (total + kC - 1) / kC;
            uint32_t r = 0;
            uint64_t cur = 0;
            rg.b[0] = 0;
            for (uint32_t l = 0; l < d.total_layers; ++l) {
                const uint64_t c = cost(l);
                if (cur > 0 && cur + c > target && r + 1 < kC) {
                    rg.b[++r] = l;
                    cur = 0;
                }
                cur += c;
            }
            for (uint32_t q = r + 1; q <= kC; ++q) rg.b[q] = d.total_layers;
        }
        for (uint32_t r = 0; r < kC && ok; ++r) {
            uint32_t noff = 0, eoff = 0;
            for (uint32_t l = 0; l < d.total_layers; ++l) {
                const uint32_t wl = lo[l + 1] - lo[l];
                uint32_t a0, a1;
                if (ranges) {
                    const bool mine = l >= rg.b[r] && l < rg.b[r + 1];
                    a0 = 0;
                    a1 = mine ? wl : 0;
                } else {
                    const uint32_t ch = (wl + kC - 1) / kC;
                    a0 = std::min(wl, r * ch);
                    a1 = std::min(wl, (r + 1) * ch);
                }
                PlanEnt& e = pe[static_cast<size_t>(r) * d.total_layers + l];
                e = PlanEnt{lo[l] + a0, a1 - a0, 0, 0, noff, eoff, 0, 0};
                if (l > 0) {
                    e.ea = rp[e.a];
                    const uint32_t eb = rp[e.a + e.n];
                    if (eb < e.ea || eb > d.edge_count) {
                        ok = false;
                        break;
                    }
                    e.m = eb - e.ea;
                } else {
                    s_max = std::max(s_max, e.n);
                }
                noff += e.n;
                eoff += e.m;
            }
            n_max = std::max(n_max, noff);
            e_max = std::max(e_max, eoff);
        }
        const uint64_t need = op_bytes + d.total_layers * sizeof(PlanEnt) + 4ull * n_max +
                              4ull * (n_max + d.total_layers) + 8ull * e_max + 4ull * s_max;
        fit5 = ok && need <= kSmemCap - 1024;
        smem5 = static_cast<uint32_t>(need);
    }
    uint32_t mode;
    if (fit0) mode = 0;
    else if (fit5) mode = ranges ? 6 : 5;
    else if (fit1 >= 1024 && d.edge_count <= (256u << 10)) mode = 1;
    else mode = d.total_layers <= 32 ? 2 : 4;  // deep: grid-wide syncs bind, the rings do not pay
    if (forced >= 0) {
        const int f = forced;
        if ((f == 1 && fit1 >= 256) || f == 2) mode = static_cast<uint32_t>(f);
        if (f == 3 && op_bytes <= kSmemCap - 1024) mode = 3;
        if (f == 4) mode = 4;
        if ((f == 5 || f == 6) && fit5) mode = static_cast<uint32_t>(f);
    }
    b->last_mode = mode;

    OnceArgs a{};
    a.off = b->off;
    a.out = out_dev;
    a.err = err_dev;
    a.L = d.total_layers;
    a.N = d.node_count;
    a.idb = idb;
    a.ns = d.sensor_count;
    a.E = static_cast<uint32_t>(d.edge_count);
    if (mode == 0 || mode == 5 || mode == 6) {
        CK(mapped(b->blob.p, b->blob_h, b->blob_d));
        a.blob = b->blob_d;
    } else {
        if (b->dblob_bytes < blob) {
            if (b->dblob) cudaFree(b->dblob);
            b->dblob = nullptr;
            b->dblob_bytes = 0;
            CK(cudaMalloc(&b->dblob, blob));
            b->dblob_bytes = blob;
        }
        CK(cudaMemcpyAsync(b->dblob, b->blob.p, blob, cudaMemcpyHostToDevice, st));
        a.blob = b->dblob;
    }
    if (mode == 2 || mode == 4) {
        if (b->op_n < idb) {
            if (b->op) cudaFree(b->op);
            b->op = nullptr;
            b->op_n = 0;
            CK(cudaMalloc(&b->op, 4ull * idb));
            b->op_n = idb;
        }
        a.op = b->op;
        constexpr uint32_t kT = 256, kEcap = 2048;
        const void* fn = mode == 2 ? reinterpret_cast<const void*>(k_once_pipe<true>)
                                   : reinterpret_cast<const void*>(k_once<2>);
        const uint32_t smem = mode == 2 ? pipe_ring_bytes(kT, d.total_layers) + kES * kEcap * 8 : 0;
        CK(set_smem(fn, dev->device, smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kT, smem));
        if (per_sm < 1) return fail(dev, ASNN_E_CUDA, "cooperative kernel does not fit");
        const uint32_t cap = static_cast<uint32_t>(per_sm) * static_cast<uint32_t>(dev->sm_count);
        const uint32_t want = mode == 2 ? (max_w + kT - 1) / kT
                                        : std::max<uint32_t>((max_w + kT - 1) / kT, (idb + 8 * kT - 1) / (8 * kT));
        const uint32_t blocks = std::max<uint32_t>(1, std::min(cap, want));
        uint32_t ecap = kEcap, tsh = 8;
        void* args2[] = {&a, &ecap, &tsh};
        void* args4[] = {&a};
        CK(cudaLaunchCooperativeKernel(fn, blocks, kT, mode == 2 ? args2 : args4, smem, st));
    } else if (mode == 5 || mode == 6) {
        CK(mapped(b->plan.p, b->plan_h, b->plan_d));
        CK(set_smem(reinterpret_cast<const void*>(k_once_cluster), dev->device, smem5));
        k_once_cluster<<<kC, 256, smem5, st>>>(a, static_cast<const PlanEnt*>(b->plan_d), n_max, e_max, rg);
        CK(cudaGetLastError());
    } else if (mode == 1) {
        const uint32_t ecap = std::min<uint32_t>(fit1, 1u << 16);
        const uint32_t smem = op_bytes + ring1 + ecap * 8 * kES;
        CK(set_smem(reinterpret_cast<const void*>(k_once_pipe<false>), dev->device, smem));
        k_once_pipe<false><<<1, T1, smem, st>>>(a, ecap, t1sh);
        CK(cudaGetLastError());
    } else {
        const uint32_t smem = op_bytes + (mode == 0 ? blob : 0);
        const uint32_t T = std::min<uint32_t>(1024, std::max<uint32_t>(128, (max_w + 31) / 32 * 32));
        auto fn = mode == 0 ? k_once<0> : k_once<1>;
        CK(set_smem(reinterpret_cast<const void*>(fn), dev->device, smem));
        fn<<<1, T, smem, st>>>(a);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));
    if (*reinterpret_cast<volatile uint32_t*>(b->err_h))
        return fail(dev, ASNN_E_INVALID, "malformed layout: node id, predecessor id or row_ptr out of range");
    if (!direct) {
        // state back into the caller's (pageable) array, all host threads for large states
        const int64_t nb = (static_cast<int64_t>(idb) + 16383) / 16384;
#pragma omp parallel for schedule(static) if (nb > 4)
        for (int64_t i = 0; i < nb; ++i) {
            const uint64_t o = static_cast<uint64_t>(i) * 16384;
            std::memcpy(state_outputs + o, b->out_h + o, 4ull * std::min<uint64_t>(16384, idb - o));
        }
    }
    return ASNN_OK;
}

int asnn_eval_buf_mode(const asnn_eval_buf* b, uint32_t* mode) {
    if (!b || !mode) return ASNN_E_INVALID;
    *mode = b->last_mode;
    return ASNN_OK;
}

// Convenience: a layout descriptor + input vector (make_state on the host,
// eval.cpp:25-35), staged and run through a temporary buffer.
int asnn_dev_eval_layout(asnn_dev* dev, const asnn_layout_desc* d, const float* x, uint64_t n_x,
                         float* state_outputs) {
    if (!dev || !d) return ASNN_E_INVALID;
    if (n_x != d->n_inputs)
        return fail(dev, ASNN_E_ARITY,
                    "expected " + std::to_string(d->n_inputs) + " input values, got " + std::to_string(n_x));
    if (n_x && !x) return fail(dev, ASNN_E_INVALID, "null input");
    if (d->node_count && (!d->layer_offsets || !d->node_ids || !d->row_ptr))
        return fail(dev, ASNN_E_INVALID, "null layout array");
    if (d->total_layers && d->layer_offsets[d->total_layers] != d->node_count)
        return fail(dev, ASNN_E_INVALID, "layer_offsets do not cover node_count");
    const uint64_t E = d->node_count ? d->row_ptr[d->node_count] : 0;
    for (uint32_t i = 0; i < d->n_inputs; ++i)
        if (d->input_order[i] >= d->id_bound) return fail(dev, ASNN_E_INVALID, "input id >= id_bound");
    // the handle's own buffer, held under the handle's lock for the whole call
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    if (!dev->once) {
        int rc0 = asnn_eval_buf_create(dev, &dev->once);
        if (rc0) return rc0;
    }
    asnn_eval_buf* b = dev->once;
    int rc = ASNN_OK;
    asnn_eval_dims dims{};
    dims.total_layers = d->total_layers;
    dims.node_count = d->node_count;
    dims.sensor_count = d->total_layers ? d->layer_offsets[1] : 0;
    dims.id_bound = d->id_bound;
    dims.edge_count = E;
    asnn_eval_stage s{};
    rc = asnn_eval_buf_stage(b, &dims, &s);
    if (rc == ASNN_OK) {
        if (d->total_layers) std::memcpy(s.layer_offsets, d->layer_offsets, 4ull * (d->total_layers + 1));
        if (d->node_count) std::memcpy(s.node_ids, d->node_ids, 4ull * d->node_count);
        for (uint64_t i = 0; i <= d->node_count && d->node_count; ++i) {
            if (d->row_ptr[i] > E || (i && d->row_ptr[i] < d->row_ptr[i - 1]))
                return fail(dev, ASNN_E_INVALID, "row_ptr decreases");
            s.row_ptr[i] = static_cast<uint32_t>(d->row_ptr[i]);
        }
        if (E) {
            std::memcpy(s.in_nodes, d->in_nodes, 4 * E);
            std::memcpy(s.in_weights, d->in_weights, 4 * E);
        }
        // make_state: inputs[input_order[i]] = x[i], the last duplicate wins
        std::vector<float> in(d->id_bound, 0.0f);
        for (uint32_t i = 0; i < d->n_inputs; ++i) in[d->input_order[i]] = x[i];
        for (uint32_t k = 0; k < dims.sensor_count; ++k) {
            const uint32_t id = d->node_ids[k];
            s.sensor_inputs[k] = id < d->id_bound ? in[id] : 0.0f;
        }
        rc = asnn_eval_buf_run(b, state_outputs);
    }
    return rc;
}

}  // extern "C"
