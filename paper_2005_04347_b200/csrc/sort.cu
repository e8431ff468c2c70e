// sort.cu -- exclusive scan and stable LSD radix sort (see sort.cuh).
#include <string>
#include <utility>

#include "sort.cuh"

namespace asnn_b200 {

namespace {
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

// Block-wide exclusive scan of one value per thread (kScanThreads threads);
// returns the exclusive prefix, *total the block sum.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t s = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;  // inclusive
    }
    __syncthreads();
    const uint32_t before = wid ? warp_sums[wid - 1] : 0;
    *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before + x - v;
}
}  // namespace

__global__ void __launch_bounds__(kScanThreads)
k_scan_tiles(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n,
             uint32_t* __restrict__ tile_sums) {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    uint32_t total;
    uint32_t run = block_exclusive_scan(s, &total);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_sums(uint32_t* __restrict__ sums, uint32_t n_tiles, uint32_t* __restrict__ total_out) {
    uint32_t carry = 0;
    for (uint32_t b = 0; b < n_tiles; b += kScanThreads) {
        const uint32_t i = b + threadIdx.x;
        const uint32_t v = i < n_tiles ? sums[i] : 0;
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, &total);
        if (i < n_tiles) sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_add(uint32_t* __restrict__ out, uint64_t n, const uint32_t* __restrict__ tile_sums) {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    const uint32_t add = tile_sums[blockIdx.x];
    if (!add) return;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) out[base + i] += add;
}

int exclusive_scan(asnn_dev* dev, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* d_total,
                   cudaStream_t st) {
    if (n == 0) {
        if (d_total) {
            cudaError_t e = cudaMemsetAsync(d_total, 0, 4, st);
            if (e != cudaSuccess) return cuda_fail(dev, e, "scan memset");
        }
        return ASNN_OK;
    }
    const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    DevBuf<uint32_t> sums;
    cudaError_t e = sums.alloc(tiles);
    if (e != cudaSuccess) return cuda_fail(dev, e, "scan alloc");
    k_scan_tiles<<<static_cast<uint32_t>(tiles), kScanThreads, 0, st>>>(in, out, n, sums.p);
    k_scan_sums<<<1, kScanThreads, 0, st>>>(sums.p, static_cast<uint32_t>(tiles), d_total);
    k_scan_add<<<static_cast<uint32_t>(tiles), kScanThreads, 0, st>>>(out, n, sums.p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(dev, e, "scan launch");
    // keep `sums` alive until the kernels ran: stream-ordered free
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(dev, e, "scan sync");
    return ASNN_OK;
}

// ---- radix sort ---------------------------------------------------------------------
__global__ void __launch_bounds__(kSortThreads)
k_radix_hist(const uint32_t* __restrict__ keys, uint64_t n, int shift, uint32_t n_tiles,
             uint32_t* __restrict__ hist) {
    __shared__ uint32_t s[256];
    s[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile;
#pragma unroll 4
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = base + r * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&s[(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[static_cast<uint64_t>(threadIdx.x) * n_tiles + blockIdx.x] = s[threadIdx.x];
}

// Stable scatter: items are ranked in index order (round-major, then warp,
// then lane) inside the tile; tile bases come from the digit-major scan.
__global__ void __launch_bounds__(kSortThreads)
k_radix_scatter(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t n,
                int shift, const uint32_t* __restrict__ hist, uint32_t n_tiles,
                uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_cnt[kSortThreads / 32][256];
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    s_base[t] = hist[static_cast<uint64_t>(t) * n_tiles + blockIdx.x];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile;
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t first = base + static_cast<uint64_t>(r) * kSortThreads;
        if (first >= n) break;  // uniform across the block
#pragma unroll
        for (int k = 0; k < kSortThreads / 32; ++k) s_cnt[k][t] = 0;
        __syncthreads();
        const uint64_t i = first + t;
        const bool valid = i < n;
        const uint32_t key = valid ? keys[i] : 0u;
        const uint32_t d = (key >> shift) & 255u;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, valid ? d : 0x10000u + lane);
        const uint32_t rank = __popc(peers & lt_mask);
        if (valid && rank == 0) s_cnt[w][d] = __popc(peers);
        __syncthreads();
        uint32_t run = s_base[t];
#pragma unroll
        for (int k = 0; k < kSortThreads / 32; ++k) {
            const uint32_t c = s_cnt[k][t];
            s_cnt[k][t] = run;
            run += c;
        }
        s_base[t] = run;
        __syncthreads();
        if (valid) {
            const uint32_t pos = s_cnt[w][d] + rank;
            keys_out[pos] = key;
            if (vals) vals_out[pos] = vals[i];
        }
        __syncthreads();
    }
}

int radix_sort_pairs(asnn_dev* dev, uint32_t* keys, uint32_t* vals, uint64_t n, int key_bits,
                     SortBuffers& bufs, uint32_t** keys_out, uint32_t** vals_out, cudaStream_t st) {
    *keys_out = keys;
    *vals_out = vals;
    if (n <= 1 || key_bits <= 0) return ASNN_OK;
    if (n >= (1ull << 32)) return fail(dev, ASNN_E_INVALID, "radix sort of more than 2^32 items");
    const uint32_t tiles = static_cast<uint32_t>((n + kSortTile - 1) / kSortTile);
    cudaError_t e = bufs.k_alt.ensure(n);
    if (e == cudaSuccess && vals) e = bufs.v_alt.ensure(n);
    if (e == cudaSuccess) e = bufs.hist.ensure(static_cast<size_t>(tiles) * 256);
    if (e != cudaSuccess) return cuda_fail(dev, e, "radix sort alloc");
    uint32_t *ka = keys, *va = vals, *kb = bufs.k_alt.p, *vb = vals ? bufs.v_alt.p : nullptr;
    for (int shift = 0; shift < key_bits; shift += 8) {
        k_radix_hist<<<tiles, kSortThreads, 0, st>>>(ka, n, shift, tiles, bufs.hist.p);
        int rc = exclusive_scan(dev, bufs.hist.p, bufs.hist.p, static_cast<uint64_t>(tiles) * 256,
                                nullptr, st);
        if (rc) return rc;
        k_radix_scatter<<<tiles, kSortThreads, 0, st>>>(ka, va, n, shift, bufs.hist.p, tiles, kb, vb);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(dev, e, "radix sort launch");
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    *keys_out = ka;
    *vals_out = va;
    return ASNN_OK;
}

}  // namespace asnn_b200
