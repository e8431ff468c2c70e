// segments.cuh -- splitting heavy rows across levels (device preprocessing).
// Included by kernels.cuh inside namespace asnn_b200.
//
// A row's sum runs over its stored edges in ascending source id
// (layout.cpp:64-80) and cannot be reordered without changing its rounding.
// It can be *interrupted*, though: the first j edges can be summed as soon
// as their sources are final, the partial fp32 sum parked in accbuf, and the
// sum resumed later -- the same sequence of roundings.  Edge j's sources are
// final after level pm_j = max(level(src_0..j)), so the prefix up to j can
// run in the launch of level pm_j + 1 ("step").  When node ids follow the
// topological order (generated corpora, pruned MLPs, banded DAGs), pm grows
// slowly along a row and a heavy row's work spreads over many earlier
// levels instead of one long dependent chain in its own level.
//
// For every heavy row (in-degree above the heavy threshold) a warp walks the
// edges, computes pm with a warp max-scan, and cuts a segment before edge j
// when pm increases there, the segment so far holds >= min_len edges and its
// step is before the row's own level; the last segment runs in the row's
// level and applies sigmoid32.  Segment task = uint4 {row, first edge, end
// edge, aux} (common.cuh).  Pass 0 counts, pass 1 writes tasks and their
// sort keys (long << (lb + 16) | step << 16 | 0xFFFF - min(len, 0xFFFF)),
// so a stable radix sort groups them by (short/long, step), longest first.
#pragma once

struct SegArgs {
    const uint32_t* row_ptr;    // [P+1]
    const uint2* edges;         // {source position, weight}
    const uint32_t* lo;         // layer offsets of the network (positions), [nl + 1]
    uint32_t nl;                // layers
    const uint32_t* sched;      // level-major schedule (heavy rows first in each level)
    const uint32_t* hv_level;   // [n_heavy] level of heavy row h
    const uint32_t* hv_sched;   // [n_heavy] index into sched of heavy row h
    uint32_t n_heavy;
    uint32_t min_len;           // shortest interrupted segment
    uint32_t long_len;          // segments above this go to k_heavy
    uint32_t lb;                // bits for the step in the sort key
    uint32_t* count;            // [n_heavy] segments per row (pass 0)
    const uint32_t* base;       // [n_heavy] exclusive scan of count (pass 1)
    uint4* tasks;               // [total] (pass 1)
    uint32_t* keys;             // [total] (pass 1)
    uint32_t* vals;             // [total] (pass 1)
    uint32_t* step_count;       // [2][nl + 1] (pass 1): short, long per step
};

__device__ __forceinline__ uint32_t layer_of_pos(const uint32_t* __restrict__ lo, uint32_t nl, uint32_t p) {
    uint32_t a = 0, b = nl;  // lo[a] <= p < lo[b]
    while (b - a > 1) {
        const uint32_t m = (a + b) / 2;
        if (__ldg(&lo[m]) <= p) a = m;
        else b = m;
    }
    return a;
}

template <int PASS>
__global__ void k_segments(SegArgs s) {
    const uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const uint32_t lane = threadIdx.x & 31;
    if (h >= s.n_heavy) return;  // warp-uniform
    const uint32_t lr = s.hv_level[h];
    const uint32_t row = s.sched[s.hv_sched[h]];
    const uint32_t b = s.row_ptr[row], e = s.row_ptr[row + 1];
    uint32_t nseg = 0;
    uint32_t out = PASS ? s.base[h] : 0;
    auto emit = [&](uint32_t a, uint32_t z, uint32_t step, bool final_seg) {
        if (PASS && lane == 0) {
            const uint32_t aux = (a != b ? kAccLoad : 0u) | (final_seg ? 0u : kAccStore) | h;
            const uint32_t len = z - a;
            const uint32_t lng = len > s.long_len ? 1u : 0u;
            s.tasks[out] = make_uint4(row, a, z, aux);
            s.keys[out] = (lng << (s.lb + 16)) | (step << 16) | (0xFFFFu - min(len, 0xFFFFu));
            s.vals[out] = out;
            atomicAdd(&s.step_count[lng * (s.nl + 1) + step], 1u);
        }
        ++out;
        ++nseg;
    };
    uint32_t pm = 0, cur = b;
    for (uint32_t base = b; base < e; base += 32) {
        const uint32_t j = base + lane;
        uint32_t x = j < e ? layer_of_pos(s.lo, s.nl, s.edges[j].x) + 1 : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= static_cast<uint32_t>(o)) x = max(x, y);
        }
        x = max(x, pm);                                    // pm of edge j
        uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, x, 1); // pm of edge j-1
        if (lane == 0) prev = pm;
        uint32_t bal = __ballot_sync(0xFFFFFFFFu, j < e && x > prev);
        while (bal) {
            const uint32_t q = __ffs(bal) - 1;
            bal &= bal - 1;
            const uint32_t jb = base + q;
            const uint32_t step = __shfl_sync(0xFFFFFFFFu, prev, q);
            if (step >= 1 && step < lr && jb - cur >= s.min_len) {
                emit(cur, jb, step, false);
                cur = jb;
            }
        }
        pm = __shfl_sync(0xFFFFFFFFu, x, 31);
    }
    emit(cur, e, lr, true);
    if (!PASS && lane == 0) s.count[h] = nseg;
}

__global__ void k_gather_tasks(const uint4* __restrict__ in, const uint32_t* __restrict__ order, uint32_t n,
                               uint4* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[order[i]];
}

// Heavy rows of every level: hv_level[h], hv_sched[h] for h in [hv_prefix[l],
// hv_prefix[l+1]) = level l, sched index lvl_off[l] + (h - hv_prefix[l]).
__global__ void k_heavy_rows(const uint32_t* __restrict__ hv_prefix, const uint32_t* __restrict__ lvl_off,
                             uint32_t n_levels, uint32_t n_heavy, uint32_t* __restrict__ hv_level,
                             uint32_t* __restrict__ hv_sched) {
    const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= n_heavy) return;
    uint32_t a = 0, b = n_levels;  // hv_prefix[a] <= h < hv_prefix[b]
    while (b - a > 1) {
        const uint32_t m = (a + b) / 2;
        if (hv_prefix[m] <= h) a = m;
        else b = m;
    }
    hv_level[h] = a;
    hv_sched[h] = lvl_off[a] + (h - hv_prefix[a]);
}

// Whole-row task records in schedule order: rtask[i] = {sched[i], row_ptr of
// it, row_ptr of the next position, 0}.
__global__ void k_row_tasks(const uint32_t* __restrict__ sched, const uint32_t* __restrict__ row_ptr, uint32_t n,
                            uint4* __restrict__ rtask) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = sched[i];
    rtask[i] = make_uint4(p, row_ptr[p], row_ptr[p + 1], 0u);
}
