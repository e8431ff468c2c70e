// win_rows.cuh -- K-rows-window: one dependency level of a wide batch whose
// rows all read from one narrow window of positions (config 2, a pruned MLP:
// every source of level l is a row of level l-1, 500 rows).
//
// k_rows gathers each (row, 128-column tile)'s ~50 source rows from L2 with
// per-lane registers in flight: 102 MB of gathers per config-2 level, ~0.45 of
// the L2 gather ceiling (profiles/r2_c2_l2.txt).  Here a block takes a
// 32-column tile and a chunk of the level's rows, first copies the whole
// source window for its tile into shared memory (coalesced 128-byte rows: on
// config 2 500 x 128 B = 64 KB), then gathers from shared memory: the L2
// traffic of a level drops from E x 128 B per tile to (window + edges) per
// block.  Rows and their order are k_rows' (rtask: {row, first edge, end
// edge}); each group of 8 lanes owns a row, lane 4 columns; the in-order
// FMUL/FADD chain of eval.cpp:20-21 per column, then sigmoid32.
// Included by kernels.cuh inside namespace asnn_b200.
#pragma once

namespace winrows {
constexpr int kTile = 32;         // columns per block
constexpr int kRowsPerBlock = 64; // 8 lanes per row -> 16 warps
constexpr int kThreads = kRowsPerBlock * 8;
}  // namespace winrows

// Shared memory: the window [win_n][kTile] floats, then each row's edges
// [kRowsPerBlock][cap] (cap >= the layout's largest in-degree), both filled
// before the gathers start -- the edge records' L2 round trips overlap the
// window's instead of preceding every batch of gathers.
__global__ void __launch_bounds__(winrows::kThreads, 2)
k_rows_win(const uint2* __restrict__ edges, float* __restrict__ A, uint32_t ldA, const uint4* __restrict__ rtask,
           uint32_t nrows, uint32_t win_lo, uint32_t win_n, uint32_t cap) {
    using namespace winrows;
    extern __shared__ __align__(16) float wr_smem[];  // [win_n][kTile] | [kRowsPerBlock][cap] uint2
    const uint32_t tiles = ldA / kTile;
    const uint32_t tile = blockIdx.x % tiles, chunk = blockIdx.x / tiles;
    const uint32_t tid = threadIdx.x;
    const uint32_t c0 = tile * kTile;
    uint2* es = reinterpret_cast<uint2*>(wr_smem + static_cast<size_t>(win_n) * kTile);
    const uint32_t r = chunk * kRowsPerBlock + tid / 8;
    const uint32_t slot = tid / 8, lane8 = tid & 7;
    uint4 t = make_uint4(0u, 0u, 0u, 0u);
    if (r < nrows) {
        t = rtask[r];
        // this row's edge records (written before this level: no PDL wait needed)
        // (eight loads in flight per lane before the first store)
        const uint32_t deg = t.z - t.y;
        for (uint32_t j = lane8; j < deg; j += 64) {
            uint2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (j + 8 * u < deg) v[u] = __ldg(edges + t.y + j + 8 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (j + 8 * u < deg) es[slot * cap + j + 8 * u] = v[u];
        }
    }
    // the previous level's grid wrote the window (PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // ---- the source window of this tile: win_n rows x 128 bytes ----
    {
        const float4* src = reinterpret_cast<const float4*>(A + static_cast<size_t>(win_lo) * ldA + c0);
        float4* dst = reinterpret_cast<float4*>(wr_smem);
        const uint32_t n4 = win_n * (kTile / 4), ld4 = ldA / 4;
        uint32_t i = tid;
        for (; i + 7 * kThreads < n4; i += 8 * kThreads) {  // eight loads in flight per thread
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t j = i + u * kThreads;
                v[u] = __ldcg(src + static_cast<size_t>(j / (kTile / 4)) * ld4 + j % (kTile / 4));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) dst[i + u * kThreads] = v[u];
        }
        float4 v[7];
        uint32_t m = 0;
#pragma unroll
        for (int u = 0; u < 7; ++u)
            if (i + u * kThreads < n4) {
                const uint32_t j = i + u * kThreads;
                v[u] = __ldcg(src + static_cast<size_t>(j / (kTile / 4)) * ld4 + j % (kTile / 4));
                m = u + 1;
            }
#pragma unroll
        for (int u = 0; u < 7; ++u)
            if (u < static_cast<int>(m)) dst[i + u * kThreads] = v[u];
        i += 7 * kThreads;
        for (; i < n4; i += kThreads) dst[i] = __ldcg(src + static_cast<size_t>(i / (kTile / 4)) * ld4 + i % (kTile / 4));
    }
    __syncthreads();
    // ---- rows: 8 lanes per row, 4 columns per lane ----
    if (r >= nrows) return;
    const uint32_t q = lane8 * 4;
    const float* ws = wr_smem + q;
    const uint2* er = es + slot * cap;
    const uint32_t deg = t.z - t.y;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    uint32_t k = 0;
    for (; k + 8 <= deg; k += 8) {
        uint2 e[8];
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) e[u] = er[k + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const float4*>(ws + (e[u].x - win_lo) * kTile);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float w = __uint_as_float(e[u].y);
            acc[0] = mac(acc[0], w, v[u].x);
            acc[1] = mac(acc[1], w, v[u].y);
            acc[2] = mac(acc[2], w, v[u].z);
            acc[3] = mac(acc[3], w, v[u].w);
        }
    }
    for (; k < deg; ++k) {
        const uint2 e = er[k];
        const float4 v = *reinterpret_cast<const float4*>(ws + (e.x - win_lo) * kTile);
        const float w = __uint_as_float(e.y);
        acc[0] = mac(acc[0], w, v.x);
        acc[1] = mac(acc[1], w, v.y);
        acc[2] = mac(acc[2], w, v.z);
        acc[3] = mac(acc[3], w, v.w);
    }
    sigmoid32_v<4>(acc);
    store_cols<4>(A + static_cast<size_t>(t.x) * ldA + c0 + q, acc);
    wc_note(t.x, c0 + q, 4);
}

// Per-level [min, max] source position over the level's scheduled rows
// (sched entries of level l: [lvl_off[l], lvl_off[l+1])), for the window test.
__global__ void k_level_windows(const uint4* __restrict__ rtask, const uint32_t* __restrict__ lvl_off,
                                uint32_t n_levels, uint32_t n, const uint2* __restrict__ edges,
                                uint32_t* __restrict__ wmin, uint32_t* __restrict__ wmax) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t a = 0, b = n_levels;  // level: lvl_off[a] <= i < lvl_off[a + 1]
    while (b - a > 1) {
        const uint32_t m = (a + b) / 2;
        if (lvl_off[m] <= i) a = m;
        else b = m;
    }
    const uint4 t = rtask[i];
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
    for (uint32_t k = t.y; k < t.z; ++k) {
        const uint32_t s = edges[k].x;
        lo = min(lo, s);
        hi = max(hi, s);
    }
    if (t.z > t.y) {
        atomicMin(&wmin[a], lo);
        atomicMax(&wmax[a], hi);
    }
}
