// tma_rows.cuh -- K-rows-TMA: one dependency level of a wide batch (ldA a
// multiple of 128 columns, config 2) with the source-row gathers done by the
// Blackwell TMA engine (cp.async.bulk.tensor.2d ... tile::gather4: four
// 512-byte rows of A, given their row indices, into shared memory with one
// instruction) instead of per-lane register loads.
//
// Why: k_rows keeps its gathers in flight in registers (8 float4 per lane,
// 64 registers, <= 32 warps/SM) -- ~110 KB in flight per SM, and config 2's
// levels run at ~45% of the measured L2 gather ceiling
// (profiles/r2_c2_l2.txt: 10.6 of 22-24 TB/s).  Here the bytes in flight are
// bounded by shared memory: S stages x 2 KB per block, two blocks per SM.
//
// Block = 4 consumer warps (thread c owns column c of the item's 128-column
// tile) + 1 producer warp.  Work item = (row task or short segment, tile),
// walked persistently (item = blockIdx.x + k * gridDim.x).  The producer's
// lanes load 32 edge records of the current item at a time (prefetching the
// next window), lane 0 writes each group's 4 weights to shared memory and
// issues the gather4 of its 4 source rows (missing edges of a row's last group
// gather the row's first source with weight 0: +0.0f appended to a sum changes at most
// the sign of a zero result, which sigmoid32 ignores -- and a parked partial
// sum only meets further additions).  Consumers add the products in stored
// order (eval.cpp:20-21), then sigmoid32 (or park the partial sum of a
// segment in accbuf, segments.cuh), exactly as k_rows.
// Included by kernels.cuh inside namespace asnn_b200.
#pragma once

#include <cuda.h>  // CUtensorMap

namespace tmarows {
constexpr int kTile = 128;      // columns per item (4 per consumer lane)
constexpr int kWarps = 4;       // consumer warps per block, one item each at a time
constexpr int kSub = 10;        // ring stages per consumer warp (2 KB each)
constexpr uint32_t kStageBytes = 4 * kTile * 4;
constexpr uint32_t smem_bytes() { return kWarps * kSub * (kStageBytes + 16 + 16); }

__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint64_t* bar, int32_t col, int32_t r0,
                                        int32_t r1, int32_t r2, int32_t r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(heavy::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(heavy::smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
}  // namespace tmarows

// Block = kWarps consumer warps + 1 producer warp.  Consumer warp w of block b
// takes items (b * kWarps + w) + k * gridDim.x * kWarps; lane w of the
// producer warp feeds it through its own kSub-stage sub-ring, loading each
// group's four edge records itself (two 16-byte loads) -- no shuffles, and the
// four streams run independently.
__global__ void __launch_bounds__(32 * (tmarows::kWarps + 1), 2)
k_rows_tma(const __grid_constant__ CUtensorMap tmA, const uint2* __restrict__ edges, float* __restrict__ A,
           uint32_t ldA, const uint4* __restrict__ rtask, uint32_t nrows, uint32_t tiles,
           const uint4* __restrict__ seg, uint32_t ns, float* __restrict__ accbuf, uint32_t zero_row) {
    using namespace tmarows;
    extern __shared__ __align__(128) unsigned char tr_smem[];
    float* stage = reinterpret_cast<float*>(tr_smem);                                   // [W][S][4][128]
    float4* wts = reinterpret_cast<float4*>(tr_smem + kWarps * kSub * kStageBytes);   // [W][S]
    uint64_t* full = reinterpret_cast<uint64_t*>(wts + kWarps * kSub);                // [W][S]
    uint64_t* empty = full + kWarps * kSub;                                            // [W][S]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t items = static_cast<uint64_t>(nrows + ns) * tiles;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWarps;
    if (tid < kWarps * kSub) {
        heavy::mbar_init(&full[tid], 1);
        heavy::mbar_init(&empty[tid], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // the previous level's grid wrote the rows gathered here (PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    auto task_of = [&](uint64_t it, uint32_t& tile) -> uint4 {
        const uint64_t t = it / tiles;
        tile = static_cast<uint32_t>(it - t * tiles);
        return t < nrows ? rtask[t] : seg[t - nrows];
    };

    if (warp == kWarps) {
        // ---- producer: lane w feeds consumer warp w ----
        if (lane < kWarps) {
            const uint32_t w = lane;
            uint32_t s = 0, ph = 0;
            for (uint64_t it = static_cast<uint64_t>(blockIdx.x) * kWarps + w; it < items; it += stride) {
                uint32_t tile;
                const uint4 t = task_of(it, tile);
                const uint32_t k0 = t.y, k1 = t.z;
                // padding of a row's last group: its first source with weight 0
                // (a written row: 0 x activation = +0.0f)
                const uint32_t pad = k1 > k0 ? edges[k0].x : zero_row;
                for (uint32_t k = k0; k < k1; k += 4) {
                    uint2 e[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) e[j] = k + j < k1 ? edges[k + j] : make_uint2(pad, 0u);
                    const uint32_t i = w * kSub + s;
                    cta::producer_wait(&empty[i], ph ^ 1);
                    wts[i] = make_float4(__uint_as_float(e[0].y), __uint_as_float(e[1].y), __uint_as_float(e[2].y),
                                         __uint_as_float(e[3].y));
                    cta::expect_tx(&full[i], kStageBytes);
                    gather4(stage + static_cast<size_t>(i) * 4 * kTile, &tmA, &full[i],
                            static_cast<int32_t>(tile * kTile), static_cast<int32_t>(e[0].x),
                            static_cast<int32_t>(e[1].x), static_cast<int32_t>(e[2].x), static_cast<int32_t>(e[3].x));
                    if (++s == kSub) s = 0, ph ^= 1;
                }
            }
        }
    } else {
        // ---- consumer warp: lane owns columns 4 lane .. 4 lane + 3 of the tile ----
        uint32_t s = 0, ph = 0;
        for (uint64_t it = static_cast<uint64_t>(blockIdx.x) * kWarps + warp; it < items; it += stride) {
            uint32_t tile;
            const uint4 t = task_of(it, tile);
            const uint32_t k0 = t.y, k1 = t.z, aux = t.w;
            const uint64_t col = static_cast<uint64_t>(tile) * kTile + 4 * lane;
            float acc[4];
            if (aux & kAccLoad) load_cols_cg<4>(acc, accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col);
            else acc[0] = acc[1] = acc[2] = acc[3] = 0.0f;
            for (uint32_t g = 0; g < (k1 - k0 + 3) / 4; ++g) {
                const uint32_t i = warp * kSub + s;
                heavy::mbar_wait(&full[i], ph);
                const float4 w = wts[i];
                const float4* v = reinterpret_cast<const float4*>(stage + static_cast<size_t>(i) * 4 * kTile) + lane;
                const float4 v0 = v[0], v1 = v[kTile / 4], v2 = v[kTile / 2], v3 = v[3 * kTile / 4];
                const float wj[4] = {w.x, w.y, w.z, w.w};
                const float4 vj[4] = {v0, v1, v2, v3};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[0] = mac(acc[0], wj[j], vj[j].x);
                    acc[1] = mac(acc[1], wj[j], vj[j].y);
                    acc[2] = mac(acc[2], wj[j], vj[j].z);
                    acc[3] = mac(acc[3], wj[j], vj[j].w);
                }
                __syncwarp();
                if (lane == 0) heavy::mbar_arrive(&empty[i]);
                if (++s == kSub) s = 0, ph ^= 1;
            }
            if (aux & kAccStore) {
                store_cols<4>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col, acc);
            } else {
                sigmoid32_v<4>(acc);
                store_cols<4>(A + static_cast<uint64_t>(t.x) * ldA + col, acc);
                wc_note(t.x, static_cast<uint32_t>(col), 4);
            }
        }
    }
}
