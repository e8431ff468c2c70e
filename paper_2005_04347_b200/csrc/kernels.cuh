// kernels.cuh -- activation kernels of the ASNN engine (sm_100a).
//
// Data layout in HBM:
//   positions  p = 0..P-1 : every assigned node of every network, network-major,
//                           then (layer, id) -- the reference's flat order
//                           (layout.cpp:28-50);
//   row_ptr[P+1]  (u32)   : destination-major CSR of incoming edges;
//   edges[E]      (uint2) : {source position, weight bits}, each row in the
//                           reference's accumulation order (ascending source
//                           id, layout.cpp:64-80);
//   A[P][ldA]     (f32)   : activations, one row per position, one column per
//                           input vector (ldA = padded batch), so a source row
//                           gather across the batch is one coalesced 128-bit
//                           load per thread.
#pragma once

#include "common.cuh"

namespace asnn_b200 {

constexpr uint32_t kUnassigned = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// K-sense: sensors (layer 0).  eval.cpp:17 + make_state eval.cpp:25-35:
// A[pos][b] = sigmoid32(x_b[k]) where k is the declared input index feeding
// the sensor id (last duplicate wins).  sinfo = {pos, in_prefix, n_in, k}.
__global__ void k_sense(const uint4* __restrict__ sinfo, uint32_t n_sensors,
                        const float* __restrict__ x, uint32_t n_vec, float* __restrict__ A,
                        uint32_t ldA) {
    // vector-major (sensor fastest): a vector's inputs are contiguous in x
    const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t b64 = idx / n_sensors;
    const uint32_t s = static_cast<uint32_t>(idx - b64 * n_sensors);
    const uint32_t b = static_cast<uint32_t>(b64);
    if (b64 >= ldA) return;
    const uint4 si = sinfo[s];
    float xv = 0.0f;
    if (b < n_vec && si.w != kUnassigned)
        xv = x[static_cast<uint64_t>(n_vec) * si.y + static_cast<uint64_t>(b) * si.z + si.w];
    A[static_cast<uint64_t>(si.x) * ldA + b] = sigmoid32(xv);
    wc_note(si.x, b, 1);
}

// ---------------------------------------------------------------------------
// K-act-lane: one launch per dependency level.  activate_node (eval.cpp:16-23)
// for every (node, column tile) item of the level:
//   LANES threads own one item; thread `lane` owns V consecutive batch
//   columns; edges are loaded cooperatively (one 8-byte {col, w} per lane,
//   coalesced) and broadcast with __shfl; each of the U in-flight source-row
//   gathers is one V-wide vector load; the sum runs sequentially in the
//   stored edge order with fp32 mul then fp32 add (bit-exact).
// sched lists the level's positions (heaviest first); item -> (sched[item /
// tiles], item % tiles).
template <int V, int LANES, int UU>
struct LevelCfg {
    static constexpr int U = UU;                          // gathers in flight per thread
    static constexpr int CH = LANES < U ? U : LANES;      // edges per chunk
    static constexpr int PER = CH / LANES;                // edges held per lane
};

template <int V, int LANES, int U = 8, int MINB = 1>
__global__ void __launch_bounds__(256, MINB)
k_level(const uint32_t* __restrict__ row_ptr, const uint2* __restrict__ edges,
        float* __restrict__ A, uint32_t ldA, const uint32_t* __restrict__ sched,
        uint32_t n_items, uint32_t tiles) {
    using C = LevelCfg<V, LANES, U>;
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t item = gt / LANES;
    if (item >= n_items) return;  // uniform across the LANES group
    const uint32_t lane = threadIdx.x % LANES;
    const uint32_t ni = item / tiles;
    const uint32_t tile = item - ni * tiles;
    const uint32_t node = __ldg(&sched[ni]);
    const uint32_t col = tile * (LANES * V) + lane * V;
    const unsigned gmask =
        LANES == 32 ? 0xFFFFFFFFu
                    : (((1u << LANES) - 1u) << ((threadIdx.x & 31u) / LANES * LANES));
    const uint32_t beg = __ldg(&row_ptr[node]);
    const uint32_t end = __ldg(&row_ptr[node + 1]);
    const float* __restrict__ Acol = A + col;

    float acc[V];
#pragma unroll
    for (int c = 0; c < V; ++c) acc[c] = 0.0f;

    for (uint32_t base = beg; base < end; base += C::CH) {
        uint2 e[C::PER];
#pragma unroll
        for (int r = 0; r < C::PER; ++r) {
            const uint32_t k = base + r * LANES + lane;
            e[r] = k < end ? __ldg(&edges[k]) : make_uint2(0u, 0u);
        }
        const uint32_t n = min(static_cast<uint32_t>(C::CH), end - base);
#pragma unroll
        for (int j0 = 0; j0 < C::CH; j0 += C::U) {
            if (static_cast<uint32_t>(j0) >= n) break;
            float v[C::U][V];
            float wj[C::U];
#pragma unroll
            for (int u = 0; u < C::U; ++u) {
                const int j = j0 + u;
                uint32_t s, wb;
                if constexpr (LANES == 1) {
                    s = e[j].x;
                    wb = e[j].y;
                } else {
                    s = __shfl_sync(gmask, e[j / LANES].x, j % LANES, LANES);
                    wb = __shfl_sync(gmask, e[j / LANES].y, j % LANES, LANES);
                }
                wj[u] = __uint_as_float(wb);
                if (static_cast<uint32_t>(j) < n) {
                    load_cols<V>(v[u], Acol + static_cast<uint64_t>(s) * ldA);
                } else {
#pragma unroll
                    for (int c = 0; c < V; ++c) v[u][c] = 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < C::U; ++u) {
                if (static_cast<uint32_t>(j0 + u) < n) {
#pragma unroll
                    for (int c = 0; c < V; ++c) acc[c] = mac(acc[c], wj[u], v[u][c]);
                }
            }
        }
    }
    sigmoid32_v<V>(acc);
    store_cols<V>(A + static_cast<uint64_t>(node) * ldA + col, acc);
    wc_note(node, col, V);
}

// ---------------------------------------------------------------------------
// K-rows: the lean form of K-act-lane for 4 columns per lane (batch >= 64).
// Same arithmetic as k_level, fewer instructions per gathered row: every
// lane reads the edge record itself (all lanes of the group hit the same L1
// line: one broadcast load, no shuffles), the edge line two batches ahead is
// prefetched into L1, and each of the U source-row gathers is one 128-bit
// load straight into registers.  Per edge and lane: 1 L1 load, 1 address
// IMAD, 1 gather, 4 FMUL + 4 FADD.
//
// Items: the first n_seg are row segments (uint4 {row, first edge, end edge,
// aux}, common.cuh / segments.cuh: a heavy row's edges split across the
// levels whose sources they need, the partial sum carried in accbuf), then
// n_rows whole rows (the same record with aux = 0, in schedule order); each
// item runs on `tiles` column tiles.
template <int LANES, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
k_rows(const uint2* __restrict__ edges, float* __restrict__ A, uint32_t ldA,
       const uint4* __restrict__ rows, uint32_t n_rows, uint32_t tiles, const uint4* __restrict__ seg,
       uint32_t n_seg, float* __restrict__ accbuf) {
    // programmatic dependent launch (engine.cu pdl_enabled): the next level's grid may
    // become resident while this one drains; it reads only the static task
    // record and edges before griddepcontrol.wait (a no-op otherwise)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t item = gt / LANES;
    const uint32_t ni = item / tiles;
    if (ni >= n_seg + n_rows) return;  // uniform across the LANES group
    const uint32_t lane = threadIdx.x % LANES;
    const uint32_t tile = item - ni * tiles;
    // one 16-byte task record per item (no sched -> row_ptr dependent loads)
    const uint4 t = ni < n_seg ? __ldg(&seg[ni]) : __ldg(&rows[ni - n_seg]);
    const uint32_t node = t.x, beg = t.y, end = t.z, aux = t.w;
    asm volatile("prefetch.global.L1 [%0];" ::"l"(edges + beg));
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t col = tile * (LANES * 4) + lane * 4;
    const uint32_t stride = ldA * 4u;
    const char* __restrict__ Acol = reinterpret_cast<const char*>(A + col);
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    if (aux & kAccLoad) {
        const float4 p = *reinterpret_cast<const float4*>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col);
        a0 = p.x, a1 = p.y, a2 = p.z, a3 = p.w;
    }
    for (uint32_t k = beg; k < end; k += U) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(edges + k + 2 * U));
        float4 v[U];
        float w[U];
        const uint32_t n = min(static_cast<uint32_t>(U), end - k);
        if (n == U) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint2 e = __ldg(&edges[k + u]);
                w[u] = __uint_as_float(e.y);
                v[u] = __ldg(reinterpret_cast<const float4*>(Acol + static_cast<uint64_t>(e.x) * stride));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                a0 = mac(a0, w[u], v[u].x);
                a1 = mac(a1, w[u], v[u].y);
                a2 = mac(a2, w[u], v[u].z);
                a3 = mac(a3, w[u], v[u].w);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (static_cast<uint32_t>(u) < n) {
                    const uint2 e = __ldg(&edges[k + u]);
                    w[u] = __uint_as_float(e.y);
                    v[u] = __ldg(reinterpret_cast<const float4*>(Acol + static_cast<uint64_t>(e.x) * stride));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (static_cast<uint32_t>(u) < n) {
                    a0 = mac(a0, w[u], v[u].x);
                    a1 = mac(a1, w[u], v[u].y);
                    a2 = mac(a2, w[u], v[u].z);
                    a3 = mac(a3, w[u], v[u].w);
                }
            }
        }
    }
    if (aux & kAccStore) {
        *reinterpret_cast<float4*>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col) =
            make_float4(a0, a1, a2, a3);
    } else {
        float o[4] = {a0, a1, a2, a3};
        sigmoid32_v<4>(o);
        *reinterpret_cast<float4*>(A + static_cast<uint64_t>(node) * ldA + col) = make_float4(o[0], o[1], o[2], o[3]);
        wc_note(node, col, 4);
    }
}

// ---------------------------------------------------------------------------
// K-rows-cp: k_rows with the source-row gathers staged through shared memory
// by cp.async instead of registers (L2-bound levels: config 2's 2 MB level
// slabs).  Every lane keeps D gathers of its 16-byte column quad in flight
// in its own ring slot column (it reads back only what it copied itself, so
// no synchronisation beyond cp.async.wait_group), the edge records
// prefetched into L1 two rounds ahead; the data registers k_rows spends on the U
// in-flight gathers are freed, so more warps per SM keep more bytes in
// flight.  Same items, same in-order __fmul_rn / __fadd_rn chain, bitwise
// identical to k_rows.
__device__ __forceinline__ void rows_cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

template <int LANES, int D, int MINB>
__global__ void __launch_bounds__(256, MINB)
k_rows_cp(const uint2* __restrict__ edges, float* __restrict__ A, uint32_t ldA,
          const uint4* __restrict__ rows, uint32_t n_rows, uint32_t tiles, const uint4* __restrict__ seg,
          uint32_t n_seg, float* __restrict__ accbuf) {
    __shared__ __align__(16) float4 ring[D][256];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t item = gt / LANES;
    const uint32_t ni = item / tiles;
    if (ni >= n_seg + n_rows) return;  // uniform across the LANES group
    const uint32_t lane = threadIdx.x % LANES;
    const uint32_t tile = item - ni * tiles;
    const uint4 t = ni < n_seg ? __ldg(&seg[ni]) : __ldg(&rows[ni - n_seg]);
    const uint32_t node = t.x, beg = t.y, end = t.z, aux = t.w;
    const uint32_t col = tile * (LANES * 4) + lane * 4;
    const uint32_t stride = ldA * 4u;
    const char* __restrict__ Acol = reinterpret_cast<const char*>(A + col);
    float4* my = &ring[0][threadIdx.x];
    asm volatile("prefetch.global.L1 [%0];" ::"l"(edges + beg));
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float w[D];
    // prologue: the first D gathers in flight
#pragma unroll
    for (int u = 0; u < D; ++u) {
        if (beg + u < end) {
            const uint2 e = __ldg(&edges[beg + u]);
            w[u] = __uint_as_float(e.y);
            rows_cp16(my + u * 256, Acol + static_cast<uint64_t>(e.x) * stride);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    if (aux & kAccLoad) {
        const float4 p = *reinterpret_cast<const float4*>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col);
        a0 = p.x, a1 = p.y, a2 = p.z, a3 = p.w;
    }
    for (uint32_t base = beg; base < end; base += D) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(edges + base + 2 * D));
#pragma unroll
        for (int u = 0; u < D; ++u) {
            const uint32_t k = base + u;
            asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");  // edge k's row landed
            if (k < end) {
                const float4 v = my[u * 256];
                a0 = mac(a0, w[u], v.x);
                a1 = mac(a1, w[u], v.y);
                a2 = mac(a2, w[u], v.z);
                a3 = mac(a3, w[u], v.w);
            }
            // refill slot u with edge k + D
            if (k + D < end) {
                const uint2 e = __ldg(&edges[k + D]);
                w[u] = __uint_as_float(e.y);
                rows_cp16(my + u * 256, Acol + static_cast<uint64_t>(e.x) * stride);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (aux & kAccStore) {
        *reinterpret_cast<float4*>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col) =
            make_float4(a0, a1, a2, a3);
    } else {
        float o[4] = {a0, a1, a2, a3};
        sigmoid32_v<4>(o);
        *reinterpret_cast<float4*>(A + static_cast<uint64_t>(node) * ldA + col) = make_float4(o[0], o[1], o[2], o[3]);
        wc_note(node, col, 4);
    }
}

// ---------------------------------------------------------------------------
// K-warp-rows: one warp per row for a single input vector (batch 1, the
// reference's eval_parallel call).  The 32 lanes load 32 consecutive edges
// and their source activations at once (32 gathers in flight per row instead
// of one thread's 8), form the products w * x in parallel (each an IEEE fp32
// multiply, exactly as in the sequential loop), and the warp then adds them
// in stored order through __shfl -- the reference's sequence of fp32 adds,
// now 4 cycles per edge behind one memory round trip per 32 edges; the next
// 32 edges' loads are issued before the current ones are summed.  Items are
// rtask records ({row, first edge, end edge, 0}) in schedule order.
__global__ void __launch_bounds__(256)
k_warp_rows(const uint2* __restrict__ edges, float* __restrict__ A, const uint4* __restrict__ rows,
            uint32_t n_rows) {
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (wid >= n_rows) return;  // warp-uniform
    const uint4 t = __ldg(&rows[wid]);
    const uint32_t beg = t.y, end = t.z;
    auto product = [&](uint32_t k) -> float {
        if (k >= end) return 0.0f;
        const uint2 e = __ldg(&edges[k]);
        return __fmul_rn(__uint_as_float(e.y), __ldg(&A[e.x]));
    };
    float acc = 0.0f;
    float p = product(beg + lane);
    for (uint32_t base = beg; base < end; base += 32) {
        const float pn = product(base + 32 + lane);  // next chunk in flight
        const uint32_t n = min(32u, end - base);
        if (n == 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc = __fadd_rn(acc, __shfl_sync(0xFFFFFFFFu, p, j));
        } else {
            for (uint32_t j = 0; j < n; ++j) acc = __fadd_rn(acc, __shfl_sync(0xFFFFFFFFu, p, j));
        }
        p = pn;
    }
    if (lane == 0) {
        A[t.x] = sigmoid32(acc);
        wc_note(t.x, 0, 1);
    }
}

// ---------------------------------------------------------------------------
// K-warp-rows4: one warp per item for narrow batches (ldA = 4 * LANES = 4 ..
// 32 columns: the per-GPU slice of a batch sharded over many GPUs).  The warp
// is LANES column quads x P = 32 / LANES edge phases: lane (phase p, quad c)
// loads edge k + p, gathers its 16-byte quad of the source row and forms the
// four IEEE products; the row's sums then run in stored order over the
// phases through __shfl (every lane of quad c keeps the same running sums).
// P gathers per row are in flight instead of 8, and one row per warp gives
// many waves per level where row-per-group kernels would leave a partial
// second wave.  Items: the first n_seg are row segments (common.cuh), then
// rows (rtask records).
template <int LANES>
__global__ void __launch_bounds__(256)
k_warp_rows4(const uint2* __restrict__ edges, float* __restrict__ A, uint32_t ldA, const uint4* __restrict__ rows,
             uint32_t n_rows, const uint4* __restrict__ seg, uint32_t n_seg, float* __restrict__ accbuf) {
    static_assert(LANES >= 1 && LANES <= 8 && (LANES & (LANES - 1)) == 0, "1..8 column quads");
    constexpr uint32_t P = 32 / LANES;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= n_seg + n_rows) return;  // warp-uniform
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t c = lane % LANES, ph = lane / LANES;
    const uint4 t = wid < n_seg ? __ldg(&seg[wid]) : __ldg(&rows[wid - n_seg]);
    const uint32_t beg = t.y, end = t.z, aux = t.w;
    const uint32_t col = c * 4;
    const uint32_t stride = ldA * 4u;
    const char* __restrict__ Acol = reinterpret_cast<const char*>(A + col);
    auto load = [&](uint32_t k, float (&pr)[4]) {
        if (k < end) {
            const uint2 e = __ldg(&edges[k]);
            const float w = __uint_as_float(e.y);
            const float4 v = __ldg(reinterpret_cast<const float4*>(Acol + static_cast<uint64_t>(e.x) * stride));
            pr[0] = __fmul_rn(w, v.x);
            pr[1] = __fmul_rn(w, v.y);
            pr[2] = __fmul_rn(w, v.z);
            pr[3] = __fmul_rn(w, v.w);
        } else {
            pr[0] = pr[1] = pr[2] = pr[3] = 0.0f;
        }
    };
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (aux & kAccLoad) {
        const float4 p = *reinterpret_cast<const float4*>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col);
        acc[0] = p.x, acc[1] = p.y, acc[2] = p.z, acc[3] = p.w;
    }
    float cur[4], nxt[4];
    load(beg + ph, cur);
    for (uint32_t base = beg; base < end; base += P) {
        load(base + P + ph, nxt);  // the next P edges in flight
        const uint32_t n = min(P, end - base);
        if (n == P) {
#pragma unroll
            for (uint32_t j = 0; j < P; ++j)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __shfl_sync(0xFFFFFFFFu, cur[q], j * LANES + c));
        } else {
            for (uint32_t j = 0; j < n; ++j)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __shfl_sync(0xFFFFFFFFu, cur[q], j * LANES + c));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
    }
    if (ph != 0) return;
    if (aux & kAccStore) {
        *reinterpret_cast<float4*>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col) =
            make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
        sigmoid32_v<4>(acc);
        *reinterpret_cast<float4*>(A + static_cast<uint64_t>(t.x) * ldA + col) =
            make_float4(acc[0], acc[1], acc[2], acc[3]);
        wc_note(t.x, col, 4);
    }
}

// ---------------------------------------------------------------------------
// K-act-heavy: one CTA per (high in-degree node, column tile).  The serial
// fp32 sum of a node cannot be split without changing its rounding, so the
// row is streamed instead: two producer warps copy predecessor rows with
// cp.async (LDGSTS, 16 bytes per lane, completion signalled on an mbarrier
// per stage) into a ring of shared-memory stages -- hundreds of rows in
// flight -- and one consumer thread per batch column runs the reference's
// in-order mul-then-add chain out of shared memory (~4 cycles per edge, the
// FADD latency).  Heavy rows thus cost their dependent-add chain, not d round
// trips to HBM.  (One TMA bulk copy per 256-byte row measured ~70 cycles per
// row per SM on B200, 17x slower than LDGSTS for this row size.)
namespace heavy {
constexpr int kRows = 32;     // rows per stage
constexpr int kStages = 12;   // ring depth: 384 rows in flight
constexpr int kProducers = 2; // producer warps (stage c belongs to warp c % 2)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Arrives on `b` once all of this thread's prior cp.async have landed.
__device__ __forceinline__ void cp_async_arrive(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
}  // namespace heavy

// TC = columns per tile (4..128, a multiple of 4); block = 64 producer threads
// + max(TC, 32) consumers; dynamic smem = stages x rows x (TC + 1) floats.
template <int TC>
__global__ void __launch_bounds__(32 * heavy::kProducers + (TC < 32 ? 32 : TC))
k_heavy(const uint32_t* __restrict__ row_ptr, const uint2* __restrict__ edges, float* __restrict__ A,
        uint32_t ldA, const uint32_t* __restrict__ sched, uint32_t tiles, const uint4* __restrict__ seg,
        float* __restrict__ accbuf) {
    using namespace heavy;
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);                         // [S][R][TC]
    float* wts = ring + kStages * kRows * TC;                             // [S][R]
    uint64_t* full = reinterpret_cast<uint64_t*>(wts + kStages * kRows);  // [S]
    uint64_t* empty = full + kStages;                                     // [S]
    constexpr int kConsumerWarps = (TC + 31) / 32;
    constexpr int kPieces = TC / 4;  // 16-byte pieces per row

    const uint32_t item = blockIdx.x;
    const uint32_t tile = item % tiles;
    // a whole row sched[i], or a row segment seg[i] (common.cuh)
    uint32_t node, beg, end, aux = 0;
    if (seg) {
        const uint4 t = seg[item / tiles];
        node = t.x, beg = t.y, end = t.z, aux = t.w;
    } else {
        node = sched[item / tiles];
        beg = row_ptr[node], end = row_ptr[node + 1];
    }
    const uint32_t n_chunks = (end - beg + kRows - 1) / kRows;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 33);  // 32 cp.async arrivals + the weights arrive
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp >= kConsumerWarps) {
        // ---- producer warps: chunk c belongs to warp kConsumerWarps + c % kProducers ----
        const int p = warp - kConsumerWarps;
        const float* base = A + static_cast<uint64_t>(tile) * TC;
        constexpr int kAhead = 8;  // this warp's chunks whose edges are in flight
        uint2 pre[kAhead];
#pragma unroll
        for (int i = 0; i < kAhead; ++i) {
            const uint32_t k = beg + (p + i * kProducers) * kRows + lane;
            pre[i] = k < end ? __ldg(&edges[k]) : make_uint2(0u, 0u);
        }
        for (uint32_t i0 = 0;; i0 += kAhead) {
            bool done = false;
#pragma unroll
            for (int i = 0; i < kAhead; ++i) {
                const uint32_t c = p + (i0 + i) * kProducers;
                if (c >= n_chunks) {
                    done = true;
                    break;
                }
                const uint2 cur = pre[i];
                const uint32_t k = beg + (c + kAhead * kProducers) * kRows + lane;
                pre[i] = k < end ? __ldg(&edges[k]) : make_uint2(0u, 0u);
                const int s = c % kStages;
                if (c >= kStages) mbar_wait(&empty[s], ((c / kStages) - 1) & 1);
                const uint32_t rows = min(static_cast<uint32_t>(kRows), end - beg - c * kRows);
                float* dst = ring + s * kRows * TC;
#pragma unroll
                for (int j = 0; j < kPieces; ++j) {
                    const int q = j * 32 + lane;    // piece index within the stage
                    const int r = q / kPieces;      // row
                    const int pc = q - r * kPieces; // 16-byte piece of the row
                    const uint32_t col = __shfl_sync(0xFFFFFFFFu, cur.x, r);
                    if (static_cast<uint32_t>(r) < rows)
                        cp_async16(dst + r * TC + pc * 4, base + static_cast<uint64_t>(col) * ldA + pc * 4);
                }
                cp_async_arrive(&full[s]);
                wts[s * kRows + lane] = __uint_as_float(cur.y);
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
            if (done) break;
        }
    } else {
        // ---- consumers: thread = one batch column of the tile ----
        const int col = threadIdx.x;
        float acc = 0.0f;
        if ((aux & kAccLoad) && col < TC)
            acc = accbuf[static_cast<uint64_t>(aux & kSlotMask) * ldA + tile * TC + col];
        for (uint32_t c = 0; c < n_chunks; ++c) {
            const int s = c % kStages;
            mbar_wait(&full[s], (c / kStages) & 1);
            const uint32_t rows = min(static_cast<uint32_t>(kRows), end - beg - c * kRows);
            const float* r = ring + s * kRows * TC;
            const float* ws = wts + s * kRows;
            if (col < TC) {
                if (rows == kRows) {
#pragma unroll
                    for (int j = 0; j < kRows; ++j) acc = mac(acc, ws[j], r[j * TC + col]);
                } else {
                    for (uint32_t j = 0; j < rows; ++j) acc = mac(acc, ws[j], r[j * TC + col]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (col < TC) {
            if (aux & kAccStore) accbuf[static_cast<uint64_t>(aux & kSlotMask) * ldA + tile * TC + col] = acc;
            else {
                A[static_cast<uint64_t>(node) * ldA + tile * TC + col] = sigmoid32(acc);
                wc_note(node, tile * TC + col, 1);
            }
        }
    }
}

#include "cta.cuh"
#include "chain.cuh"
#include "serve.cuh"
#include "tma_rows.cuh"
#include "bulk_rows.cuh"
#include "win_rows.cuh"
#include "segments.cuh"

// Latency probes (one thread, dependent chains, clock64), op templated and the
// loop unrolled 8x so the loop branch is amortised:
//   0 sigmoid32, 1 DFMA, 2 FADD, 3 shared-memory load chain, 4 double
//   division, 5 exp, 6 an empty loop iteration (branch + counter).
template <int W>
__device__ __forceinline__ void probe_op(float& f, double& d, uint32_t& p, const uint32_t* chain) {
    if constexpr (W == 0) f = sigmoid32(f);
    else if constexpr (W == 1) d = __fma_rn(d, 1.0000001, 1e-9);
    else if constexpr (W == 2) f = __fadd_rn(f, 1e-7f);
    else if constexpr (W == 3) p = chain[p & 255];
    else if constexpr (W == 4) d = __ddiv_rn(1.0, __dadd_rn(1.0, d));
    else if constexpr (W == 5) d = exp_glibc(__dmul_rn(-d, 1e-3), kExpTab);
}

template <int W>
__global__ void k_latency_probe(int n, float seed, long long* cycles, float* sink) {
    __shared__ uint32_t chain[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) chain[i] = (i * 97 + 13) & 255;
    __syncthreads();
    if (threadIdx.x) return;
    float f = seed;
    double d = seed;
    uint32_t p = static_cast<uint32_t>(seed * 100);
    const long long t0 = clock64();
    if constexpr (W == 6) {
        for (int i = 0; i < n; ++i) asm volatile("" : "+r"(p));
    } else {
        for (int i = 0; i < n; i += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) probe_op<W>(f, d, p, chain);
        }
    }
    const long long t1 = clock64();
    *cycles = t1 - t0;
    *sink = f + static_cast<float>(d) + static_cast<float>(p);
}

// Every float bit pattern through sigmoid32 (fast path + rounding test) and
// sigmoid32_exact: counts[0] = bitwise mismatches (a NaN matches any NaN),
// counts[1] = inputs the rounding test sent to the exact path.
__global__ void k_sigmoid_selfcheck(unsigned long long* counts) {
    unsigned long long bad = 0, slow = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (1ull << 32);
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float x = __uint_as_float(static_cast<uint32_t>(i));
        bool exact;
        const float f = sigmoid32_path(x, exact);
        const float g = sigmoid32_exact(x);
        const bool same = __float_as_uint(f) == __float_as_uint(g) || (f != f && g != g);
        bad += same ? 0 : 1;
        slow += exact ? 1 : 0;
    }
    for (int o = 16; o; o >>= 1) {
        bad += __shfl_xor_sync(0xFFFFFFFFu, bad, o);
        slow += __shfl_xor_sync(0xFFFFFFFFu, slow, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&counts[0], bad);
        atomicAdd(&counts[1], slow);
    }
}

__global__ void k_sigmoid_many(const float* __restrict__ x, float* __restrict__ y, uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) y[i] = sigmoid32(x[i]);
}

// ---------------------------------------------------------------------------
// K-gather-out: read_outputs (eval.cpp:82-87) for the whole batch.
// oinfo = {pos (or kUnassigned), out_prefix, n_out, k}; out is [net][b][k].
__global__ void k_gather_out(const uint4* __restrict__ oinfo, uint32_t n_total,
                             const float* __restrict__ A, uint32_t ldA, uint32_t n_vec,
                             float* __restrict__ out) {
    // vector-major (output fastest): a vector's outputs are contiguous in out
    const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t b64 = idx / n_total;
    const uint32_t o = static_cast<uint32_t>(idx - b64 * n_total);
    const uint32_t b = static_cast<uint32_t>(b64);
    if (b64 >= n_vec) return;
    const uint4 oi = oinfo[o];
    const float v = oi.x == kUnassigned ? 0.0f : A[static_cast<uint64_t>(oi.x) * ldA + b];
    out[static_cast<uint64_t>(n_vec) * oi.y + static_cast<uint64_t>(b) * oi.z + oi.w] = v;
}

// K-state: the id-indexed ActivationState.outputs (eval.hpp:14-17) for every
// vector; ids without a layer stay 0.0f (eval.cpp:30-31).
__global__ void k_state(const uint32_t* __restrict__ state_map, const uint32_t* __restrict__ idb_prefix,
                        uint32_t n_nets, uint32_t total_idb, const float* __restrict__ A,
                        uint32_t ldA, uint32_t n_vec, float* __restrict__ state) {
    const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t f = idx / n_vec;
    const uint32_t b = static_cast<uint32_t>(idx - f * n_vec);
    if (f >= total_idb) return;
    uint32_t lo = 0, hi = n_nets;  // net g: idb_prefix[g] <= f < idb_prefix[g+1]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (idb_prefix[mid] <= f) lo = mid;
        else hi = mid;
    }
    const uint32_t base = idb_prefix[lo];
    const uint32_t idb = idb_prefix[lo + 1] - base;
    const uint32_t pos = state_map[f];
    const float v = pos == kUnassigned ? 0.0f : A[static_cast<uint64_t>(pos) * ldA + b];
    state[static_cast<uint64_t>(n_vec) * base + static_cast<uint64_t>(b) * idb + (f - base)] = v;
}

}  // namespace asnn_b200
