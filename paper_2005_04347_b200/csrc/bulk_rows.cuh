// bulk_rows.cuh -- K-rows-bulk: one dependency level of a wide batch (ldA a
// multiple of 512 columns, config 2) with every source row slice moved by the
// TMA engine as one contiguous bulk copy (cp.async.bulk, 2 KB = 512 columns
// of one row of A per edge) into a double-buffered shared-memory stage.
//
// Why: k_rows keeps its gathers in flight in registers (8 float4 per lane)
// and config 2's levels run at ~45% of the measured L2 gather ceiling
// (profiles/r2_c2_l2.txt); the gather4 tensor path (tma_rows.cuh) is bound by
// the gather4 issue rate.  Here one lane issues one plain bulk copy per edge:
// the bytes in flight are bounded by shared memory (2 stages x CHUNK edges x
// 2 KB per block, three blocks per SM at CHUNK = 16), not by registers.
//
// Block = 128 threads = one (row task or short segment, 512-column tile)
// item; thread c owns columns 4c..4c+3 of the tile.  Warp 0 issues chunk c+2
// of the item's edges into the stage chunk c used as soon as every thread has
// added chunk c.  Sums in stored order (eval.cpp:20-21), then sigmoid32 or the
// parked partial sum of a segment (accbuf, segments.cuh), exactly as k_rows.
// Included by kernels.cuh inside namespace asnn_b200, after cta.cuh.
#pragma once

namespace bulkrows {
constexpr uint32_t kTile = 512;           // columns per item
constexpr uint32_t kThreads = kTile / 4;  // four columns per thread
constexpr uint32_t kRowBytes = kTile * 4;
template <int CHUNK>
constexpr uint32_t smem_bytes() { return 2 * CHUNK * kRowBytes + 64; }
}  // namespace bulkrows

template <int CHUNK>
__global__ void __launch_bounds__(bulkrows::kThreads)
k_rows_bulk(const uint2* __restrict__ edges, float* __restrict__ A, uint32_t ldA,
            const uint4* __restrict__ rows, uint32_t n_rows, uint32_t tiles, const uint4* __restrict__ seg,
            uint32_t n_seg, float* __restrict__ accbuf) {
    using namespace bulkrows;
    extern __shared__ __align__(128) unsigned char br_smem[];
    float* stage = reinterpret_cast<float*>(br_smem);                                 // [2][CHUNK][kTile]
    uint64_t* full = reinterpret_cast<uint64_t*>(br_smem + 2 * CHUNK * kRowBytes);  // [2]
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t ni = blockIdx.x / tiles, tile = blockIdx.x - ni * tiles;
    if (ni >= n_seg + n_rows) return;  // uniform across the block
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const uint4 t = ni < n_seg ? __ldg(&seg[ni]) : __ldg(&rows[ni - n_seg]);
    const uint32_t node = t.x, beg = t.y, end = t.z, aux = t.w;
    if (tid == 0) {
        heavy::mbar_init(&full[0], 1);
        heavy::mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t col0 = tile * kTile;
    const uint32_t n_chunks = (end - beg + CHUNK - 1) / CHUNK;
    // warp 0: chunk c of the item's edges into stage c & 1
    auto issue = [&](uint32_t c) {
        if (tid >= 32 || c >= n_chunks) return;
        const uint32_t k0 = beg + c * CHUNK, n = min(static_cast<uint32_t>(CHUNK), end - k0);
        uint64_t* bar = &full[c & 1];
        if (lane == 0) cta::expect_tx(bar, n * kRowBytes);
        __syncwarp();
        for (uint32_t j = lane; j < n; j += 32) {
            const uint2 e = __ldg(&edges[k0 + j]);
            cta::bulk_g2s(stage + ((c & 1) * CHUNK + j) * kTile, A + static_cast<uint64_t>(e.x) * ldA + col0,
                          kRowBytes, bar);
        }
    };
    issue(0);
    issue(1);
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    const uint32_t col = col0 + tid * 4;
    if (aux & kAccLoad) {
        const float4 p = *reinterpret_cast<const float4*>(accbuf + static_cast<uint64_t>(aux & kSlotMask) * ldA + col);
        a0 = p.x, a1 = p.y, a2 = p.z, a3 = p.w;
    }
    for (uint32_t c = 0; c < n_chunks; ++c) {
        const uint32_t k0 = beg + c * CHUNK, n = min(static_cast<uint32_t>(CHUNK), end - k0);
        heavy::mbar_wait(&full[c & 1], (c >> 1) & 1);
        const float4* s = reinterpret_cast<const float4*>(stage + (c & 1) * CHUNK * kTile) + tid;
#pragma unroll 4
        for (uint32_t j = 0; j < n; ++j) {
            const float w = __uint_as_float(__ldg(&edges[k0 + j]).y);
            const float4 v = s[j * (kTile / 4)];
            a0 = mac(a0, w, v.x);
            a1 = mac(a1, w, v.y);
            a2 = mac(a2, w, v.z);
            a3 = mac(a3, w, v.w);
        }
        __syncthreads();  // stage c & 1 consumed
        issue(c + 2);
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
