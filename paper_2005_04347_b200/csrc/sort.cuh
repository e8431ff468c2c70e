// sort.cuh -- device building blocks for preprocessing: exclusive scan and a
// stable LSD radix sort of (u32 key, u32 value) pairs, 8 bits per pass.
//
// Stability is what makes the device layout bit-exact: sorting node indices
// (already id-ordered) by level keeps ids ascending inside a level, which is
// the reference's (layer, id) order (layout.cpp:28-50); sorting edges by source
// id and then stably by target position gives each CSR row in ascending
// source-id order (layout.cpp:64-80).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.hpp"

namespace asnn_b200 {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;                        // per thread
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys per tile
constexpr int kScanThreads = 1024;

// ---- exclusive scan of u32 (in place allowed), u64 total ------------------
// Single-kernel decoupled scan is not needed at preprocessing scale: a tile
// pass writes per-tile sums, one block scans the sums, a third pass adds.
__global__ void k_scan_tiles(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                             uint64_t n, uint32_t* __restrict__ tile_sums);
__global__ void k_scan_sums(uint32_t* __restrict__ sums, uint32_t n_tiles, uint32_t* __restrict__ total);
__global__ void k_scan_add(uint32_t* __restrict__ out, uint64_t n, const uint32_t* __restrict__ tile_sums);

// out[i] = sum(in[0..i)), *d_total = sum(in); d_total device pointer (may be null).
int exclusive_scan(asnn_dev* dev, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* d_total,
                   cudaStream_t st);

// ---- radix sort ------------------------------------------------------------------
// Stable sort of n (key, value) pairs by key bits [0, key_bits).  Buffers are
// ping-ponged; on return *keys_out / *vals_out point at the sorted arrays
// (one of the inputs or the alternates).  values may be null (keys only).
struct SortBuffers {
    DevBuf<uint32_t> k_alt, v_alt, hist;
};
int radix_sort_pairs(asnn_dev* dev, uint32_t* keys, uint32_t* vals, uint64_t n, int key_bits,
                     SortBuffers& bufs, uint32_t** keys_out, uint32_t** vals_out, cudaStream_t st);

}  // namespace asnn_b200
