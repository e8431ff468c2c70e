// chain.cuh -- K-chain: the K-cta sweep for deep, narrow networks (config 3:
// 2000 layers of <= 26 rows, one batch column per CTA), rebuilt around the
// one thing that bounds it -- the dependent chain from layer l-1's values to
// layer l's values.  eval.cpp:64-77 semantics (per layer, every node's
// in-order fp32 sum then sigmoid32) with the same sequence of roundings.
//
// Each row's stored edges split at split[p] (k_splits with depth D): the
// prefix's sources all sit on layers <= l - D - 1, the tail starts at the
// first source on layer l - D or later (on config 3 the tail is one edge for
// 98% of rows, at most three).  Warp roles:
//  * F (two groups of NF warps, one item = (row, column) per lane; group f
//    finishes layers l = 1 + f (mod 2)): per layer, a named barrier with the
//    other group (layer l-1 final), the tail's source loads, two
//    multiply-adds, sigmoid32, one store and a barrier arrival for the other
//    group -- the record prefetch, the mbarrier arrivals and the loop overhead
//    of one group run in the shadow of the other group's chain (ncu, one
//    group: ~680 cycles per layer of which ~300 are the data chain).  Each F
//    warp arrives on layer l's done mbarrier (release) once its items are final;
//  * P (NP groups of NF warps; group j owns layers m = 1 + j (mod NP)): waits
//    (suspended) until layer m - D - 1 is final, sums the prefix of layer m's
//    rows (8 source loads in flight per lane), and leaves per item a 32-byte
//    record {partial sum, destination + staging slot + group-end flag, first
//    two tail edges as (shared-memory offset, weight), tail length + flag,
//    index of the third} in a ring of
//    kRecBufs layer buffers, then arrives on the buffer's mbarrier.  D = NP - 1
//    gives each prefix D - 1 whole F steps plus the current one of slack;
//  * the producer warp stages GROUPS of consecutive layers (row pointers,
//    splits and edges of a group are contiguous in the level-sorted CSR: three
//    bulk copies per group).  Per-layer staging cost the producer ~200
//    instructions and ~1000 cycles per layer -- the bound of config 3
//    (ncu: P warps waiting on `full` in 50% of all samples); groups of ~1/6
//    of the ring divide that by the layers per group.  Groups are host-built
//    {first layer, lo, le} records (ensure_groups in engine.cu).
// F fetches layer l+1's record while layer l's tail loads are in flight, so
// the record round trip overlaps the chain.  The partial sum is the same
// fp32 value an uninterrupted loop would hold at the split (segments.cuh);
// padding a short tail with (zero row, weight 0) adds +0.0f to the final sum,
// which sigmoid32 cannot tell from the unpadded value (it only changes the
// sign of a zero sum, and sigmoid32(-0) == sigmoid32(+0)).
// Included by kernels.cuh inside namespace asnn_b200 after cta.cuh.
#pragma once

namespace chain {
constexpr uint32_t kRecBufs = 4;           // >= D + 1 (D <= 3): F holds layers l, l+1
constexpr uint32_t kNoTail = 0xFFFFFFFFu;  // record of an item past the layer's width
constexpr uint32_t kUnstaged = 1u << 30;   // rb.z flag: the tail's edges are in global memory
constexpr uint32_t kTailMask = kUnstaged - 1;
// ra.y = destination (shared-memory float index, < 2^20) | staging slot << 20
// | the layer is its staging group's last << 25
constexpr uint32_t kDstMask = (1u << 20) - 1;
constexpr uint32_t kGroupEnd = 1u << 25;
constexpr uint32_t kDoneBars = 8;          // >= D + 2: layer k's barrier is reused for k + kDoneBars

// Waits for a phase of an mbarrier, suspending in the hardware between tests
// (woken when the phase completes).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n}" ::"r"(heavy::smem_u32(b)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// Named barriers 2 + f between the finish groups: group 1-f arrives when its
// layer is final, group f syncs before the next.
__device__ __forceinline__ void f_sync(uint32_t id, uint32_t n_threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n_threads) : "memory");
}
__device__ __forceinline__ void f_arrive(uint32_t id, uint32_t n_threads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n_threads) : "memory");
}

// Shared-memory bytes past the staging ring: mbarriers + group metas, then
// the record ring (2 x uint4 per item per buffer) and its mbarriers, then the
// layer-done mbarriers.
__host__ __device__ constexpr uint32_t tail_bytes(uint32_t nf) {
    return cta::kMetaBytes + kRecBufs * nf * 32 * 32 + kRecBufs * 8 + kDoneBars * 8;
}

// Bytes one group of layers takes in the ring: 16-byte aligned bulk copies
// of row_ptr[r0a .. r1], split[r0a .. r1) and edges[e0a .. e1) (global rows
// r0 .. r1, edges e0 .. e1).
__host__ __device__ inline void group_bytes(uint32_t r0, uint32_t r1, uint32_t e0, uint32_t e1, uint32_t& rbytes,
                                            uint32_t& sbytes, uint32_t& ebytes) {
    const uint32_t r0a = r0 & ~3u, e0a = e0 & ~1u;
    rbytes = ((r1 - r0a + 1) * 4 + 15) & ~15u;
    sbytes = ((r1 - r0a) * 4 + 15) & ~15u;
    ebytes = ((e1 - e0a) * 8 + 15) & ~15u;
}

// The producer warp: stages groups 0..K-1 of network n in order.  meta[slot]
// = {l1, r0a, e0a, staged, rows_at, split_at, extent, edges_at} (ring indices
// in u32 / u32 / uint2 units).  A group whose bytes would need the release of
// the group just before it is read from global memory instead: F finishes
// that group's last layer only with the next group's first prefix, which
// needs that group staged.
__device__ __forceinline__ void produce_groups(const CtaNet& n, const uint4* __restrict__ grp, uint32_t K,
                                               const uint32_t* __restrict__ row_ptr,
                                               const uint32_t* __restrict__ split, const uint2* __restrict__ edges,
                                               unsigned char* ring, uint32_t ring_bytes, uint64_t* full,
                                               uint64_t* empty, uint32_t* meta, int write_all, uint32_t lane) {
    using namespace cta;
    uint32_t w = 0, used = 0, oldest = 0;  // oldest: first group whose release is not yet seen
    auto release_to = [&](uint32_t upto) {
        for (; oldest < upto; ++oldest) used -= meta[8 * (oldest % kSlots) + 6];
    };
    // window of group records: lane j holds grp[base + j] (records 0..K, K = sentinel)
    uint32_t base = 0;
    uint4 rc = grp[min(base + lane, K)], rn = grp[min(base + 31 + lane, K)];
    const bool leader = lane == 0;
    for (uint32_t k = 0; k < K; ++k) {
        if (k - base == 31) {
            base += 31;
            rc = rn;
            rn = grp[min(base + 31 + lane, K)];
        }
        const uint32_t i0 = k - base;
        const uint32_t l1 = __shfl_sync(0xFFFFFFFFu, rc.x, i0 + 1);
        const uint32_t r0 = n.pos_base + __shfl_sync(0xFFFFFFFFu, rc.y, i0);
        const uint32_t r1 = n.pos_base + __shfl_sync(0xFFFFFFFFu, rc.y, i0 + 1);
        const uint32_t e0 = __shfl_sync(0xFFFFFFFFu, rc.z, i0), e1 = __shfl_sync(0xFFFFFFFFu, rc.z, i0 + 1);
        const uint32_t m = k % kSlots, u = k / kSlots;
        uint32_t rbytes, sbytes, ebytes;
        group_bytes(r0, r1, e0, e1, rbytes, sbytes, ebytes);
        const uint32_t r0a = r0 & ~3u, e0a = e0 & ~1u;
        const uint32_t size = rbytes + sbytes + ebytes;
        if (u > 0) {  // slot m's previous group (k - kSlots) and all before it are released
            producer_wait(&empty[m], (u - 1) & 1);
            release_to(k - kSlots + 1);
        }
        bool staged = size <= ring_bytes && !(write_all & 2);
        uint32_t at = 0, extent = 0;
        if (staged) {
            for (;;) {
                if (used == 0) w = 0;
                const bool wrap = w + size > ring_bytes;
                const uint32_t need = wrap ? ring_bytes - w + size : size;
                if (need <= ring_bytes - used) {
                    at = wrap ? 0u : w;
                    extent = need;
                    w = at + size;
                    used += need;
                    break;
                }
                if (oldest + 1 >= k) {  // only the previous group holds the space
                    staged = false;
                    break;
                }
                producer_wait(&empty[oldest % kSlots], (oldest / kSlots) & 1);
                release_to(oldest + 1);
            }
        }
        if (leader) {
            uint32_t* mm = meta + 8 * m;
            mm[0] = l1;
            mm[1] = r0a;
            mm[2] = e0a;
            mm[3] = staged ? 1u : 0u;
            mm[4] = at / 4;
            mm[5] = (at + rbytes) / 4;
            mm[6] = extent;
            mm[7] = (at + rbytes + sbytes) / 8;
            if (staged) {
                expect_tx(&full[m], size);
                bulk_g2s(ring + at, row_ptr + r0a, rbytes, &full[m]);
                bulk_g2s(ring + at + rbytes, split + r0a, sbytes, &full[m]);
                if (ebytes) bulk_g2s(ring + at + rbytes + sbytes, edges + e0a, ebytes, &full[m]);
            } else {
                heavy::mbar_arrive(&full[m]);
            }
        }
        __syncwarp();  // the extent in meta is read by every lane's release_to
    }
}
}  // namespace chain

template <int NF, int NP, bool GUARD>
__global__ void __launch_bounds__(32 * (NF * (2 + NP) + 1))
k_chain(const CtaNet* __restrict__ nets, const uint32_t* __restrict__ lo_cat, const uint4* __restrict__ grp,
        const uint32_t* __restrict__ grp_off, const uint32_t* __restrict__ lg_cat,
        const uint32_t* __restrict__ row_ptr, const uint2* __restrict__ edges, const uint4* __restrict__ sinfo,
        const uint4* __restrict__ oinfo, const float* __restrict__ x, uint32_t n_vec, float* __restrict__ A,
        uint32_t ldA, uint32_t C, uint32_t max_pos, uint32_t ring_bytes, int write_all, float* __restrict__ out,
        const uint32_t* __restrict__ split) {
    using namespace cta;
    using chain::kRecBufs;
    using chain::kNoTail;
    constexpr uint32_t D = NP - 1;
    constexpr uint32_t I = NF * 32;  // items of one layer
    static_assert(NP >= 2 && D + 1 <= kRecBufs, "record ring too small for the prefix depth");
    extern __shared__ __align__(128) unsigned char cta_smem[];
    const CtaNet n = nets[blockIdx.y];
    const uint32_t c0 = blockIdx.x * C;
    float* As = reinterpret_cast<float*>(cta_smem);  // [max_pos + 1][C], row max_pos = zeros
    const uint32_t zero_slot = max_pos;
    const size_t as_floats = (static_cast<size_t>(zero_slot + 1) * C + 3) & ~size_t(3);
    unsigned char* ring = reinterpret_cast<unsigned char*>(As + as_floats);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + ring_bytes);
    uint64_t* empty = full + kSlots;
    uint32_t* meta = reinterpret_cast<uint32_t*>(empty + kSlots);
    uint4* recA = reinterpret_cast<uint4*>(meta + 8 * kSlots);  // [kRecBufs][I]
    uint4* recB = recA + kRecBufs * I;                          // [kRecBufs][I]
    // rec_bar[b]: record buffer b filled (one arrival per P warp of the group);
    // done_bar[(k - 1) % kDoneBars]: layer k final (one arrival per F warp)
    uint64_t* rec_bar = reinterpret_cast<uint64_t*>(recB + kRecBufs * I);
    uint64_t* done_bar = rec_bar + kRecBufs;
    const uint4* ngrp = grp + grp_off[blockIdx.y];
    const uint32_t n_groups = grp_off[blockIdx.y + 1] - grp_off[blockIdx.y] - 1;  // + the sentinel
    const uint32_t* lo = lo_cat + n.lo_base;
    const uint32_t* lg = lg_cat + n.lo_base;

    const uint32_t Tc = 32 * NF * (2 + NP);  // consumer threads
    const uint32_t tid = threadIdx.x;
    const uint32_t warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (uint32_t s = 0; s < kSlots; ++s) {
            heavy::mbar_init(&full[s], 1);
            heavy::mbar_init(&empty[s], NF);
        }
        for (uint32_t b = 0; b < kRecBufs; ++b) heavy::mbar_init(&rec_bar[b], NF);
        for (uint32_t b = 0; b < chain::kDoneBars; ++b) heavy::mbar_init(&done_bar[b], NF);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint2* ring_u2 = reinterpret_cast<const uint2*>(ring);
    const uint32_t* ring_u32 = reinterpret_cast<const uint32_t*>(ring);
    // shared-memory offset of source `pos`, column q (GUARD: no position -> zero row)
    auto off = [&](uint32_t pos, uint32_t q) -> uint32_t {
        const uint32_t p = pos - n.pos_base;
        return (GUARD && p >= n.n_pos ? zero_slot : p) * C + q;
    };

    if (tid >= Tc) {
        chain::produce_groups(n, ngrp, n_groups, row_ptr, split, edges, ring, ring_bytes, full, empty, meta,
                              write_all, lane);
    } else {
        for (uint32_t c = tid; c < C; c += Tc) As[zero_slot * C + c] = 0.0f;
        // sensors (eval.cpp:17), as K-cta
        for (uint32_t i = tid; i < n.n_sensors * C; i += Tc) {
            const uint32_t c = i / n.n_sensors, s = i - c * n.n_sensors;
            const uint32_t k = sinfo[n.sens_prefix + s].w;
            const uint32_t col = c0 + c;
            float xv = 0.0f;
            if (col < n_vec && k != kUnassigned)
                xv = x[static_cast<uint64_t>(n_vec) * n.in_prefix + static_cast<uint64_t>(col) * n.n_in + k];
            As[static_cast<size_t>(s) * C + c] = sigmoid32(xv);
            wc_note(n.pos_base + s, col, 1);
        }
        consumer_barrier(Tc);

        if (warp >= 2 * NF) {
            // ---- P group j: prefixes of layers m = 1 + j, 1 + j + NP, ... ----
            const uint32_t j = warp / NF - 2, w = warp % NF;
            const uint32_t it = w * 32 + lane;
            const uint32_t i = it / C, q = it - i * C;
            // layer m's bounds and group, loaded one layer of this group ahead
            uint32_t m = 1 + j;
            uint32_t a_n = 0, b_n = 0, g_n = 0;
            if (m < n.n_layers) a_n = lo[m], b_n = lo[m + 1], g_n = lg[m];
            for (; m < n.n_layers; m += NP) {
                const uint32_t a = a_n, b = b_n, g = g_n;
                if (m + NP < n.n_layers) a_n = lo[m + NP], b_n = lo[m + NP + 1], g_n = lg[m + NP];
                // group g's staging (F releases it only after finishing layer m)
                chain::mbar_wait_sleep(&full[g % kSlots], (g / kSlots) & 1);
                const uint32_t* mm = meta + 8 * (g % kSlots);
                const uint32_t l1 = mm[0], r0a = mm[1], e0a = mm[2];
                const bool st = mm[3] != 0;
                const uint32_t rows_at = mm[4], split_at = mm[5], edges_at = mm[7];
                // sources on layers <= m - D - 1 are final (layer 0: the
                // sensor barrier); the record buffer (m - 1) % kRecBufs was
                // last read by F at layer m - kRecBufs <= m - D - 1.  Layer k's
                // barrier was last completed for k - kDoneBars, which F
                // finished before this group's previous layer could start.
                if (m > D + 1) {
                    const uint32_t k = m - D - 2;  // layer k + 1 (>= 1) done: phase k / kDoneBars
                    chain::mbar_wait_sleep(&done_bar[k % chain::kDoneBars], (k / chain::kDoneBars) & 1);
                }
                const uint32_t zo = zero_slot * C + q;
                // every item carries the staging slot and group end (F's lane 0 releases)
                const uint32_t tag = (g % kSlots) << 20 | (m + 1 == l1 ? chain::kGroupEnd : 0u);
                uint4 ra = make_uint4(0u, tag, zo, 0u), rb = make_uint4(zo, 0u, kNoTail, 0u);
                if (i < b - a) {
                    const uint32_t r = n.pos_base + a + i;
                    uint32_t k, ks, ke;
                    if (st) {
                        k = ring_u32[rows_at + r - r0a];
                        ke = ring_u32[rows_at + r + 1 - r0a];
                        ks = ring_u32[split_at + r - r0a];
                    } else {
                        k = row_ptr[r], ke = row_ptr[r + 1], ks = split[r];
                    }
                    // absolute edge index -> the staged copy (or global memory)
                    const uint2* Ep = st ? ring_u2 + edges_at - e0a : edges;
                    float acc = 0.0f;
                    for (; k + 8 <= ks; k += 8) {
                        uint2 ed[8];
                        float av[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) ed[u] = Ep[k + u];
#pragma unroll
                        for (int u = 0; u < 8; ++u) av[u] = As[off(ed[u].x, q)];
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc = mac(acc, __uint_as_float(ed[u].y), av[u]);
                    }
                    for (; k < ks; ++k) {
                        const uint2 ed = Ep[k];
                        acc = mac(acc, __uint_as_float(ed.y), As[off(ed.x, q)]);
                    }
                    ra.x = __float_as_uint(acc);
                    ra.y |= (a + i) * C + q;
                    if (ke > ks) {
                        const uint2 e0 = Ep[ks];
                        ra.z = off(e0.x, q);
                        ra.w = e0.y;
                    }
                    if (ke > ks + 1) {
                        const uint2 e1 = Ep[ks + 1];
                        rb.x = off(e1.x, q);
                        rb.y = e1.y;
                    }
                    // F reads edges beyond the second from ring_u2 (staged,
                    // index relative to the ring) or edges (absolute)
                    rb.z = (ke - ks) | (st ? 0u : chain::kUnstaged);
                    rb.w = st ? edges_at + ks + 2 - e0a : ks + 2;
                }
                recA[((m - 1) % kRecBufs) * I + it] = ra;
                recB[((m - 1) % kRecBufs) * I + it] = rb;
                __syncwarp();
                if (lane == 0) heavy::mbar_arrive(&rec_bar[(m - 1) % kRecBufs]);
            }
        } else {
            // ---- F group f: finish layers l = 1 + f, 3 + f, ... ----
            const uint32_t f = warp / NF, it = (warp % NF) * 32 + lane;
            const uint32_t q = it % C;
            constexpr uint32_t kPair = 2 * 32 * NF;  // both finish groups
            // record buffer (m - 1) % kRecBufs, its ((m - 1) / kRecBufs)-th fill
            auto wait_rec = [&](uint32_t m, uint4& ra, uint4& rb) {
                heavy::mbar_wait(&rec_bar[(m - 1) % kRecBufs], ((m - 1) / kRecBufs) & 1);
                ra = recA[((m - 1) % kRecBufs) * I + it];
                rb = recB[((m - 1) % kRecBufs) * I + it];
            };
            uint4 ra = make_uint4(0u, 0u, 0u, 0u), rb = make_uint4(0u, 0u, kNoTail, 0u);
            uint32_t l = 1 + f;
            if (l < n.n_layers) wait_rec(l, ra, rb);
            for (; l < n.n_layers; l += 2) {
                // layer l-1 final (the other group; layer 0: the sensor barrier)
                if (l > 1) chain::f_sync(2 + f, kPair);
                const float v0 = As[ra.z], v1 = As[rb.x];
                const uint32_t flags = rb.z;
                if (flags != kNoTail) {
                    const uint32_t nt = flags & chain::kTailMask;
                    float acc = __uint_as_float(ra.x);
                    acc = mac(acc, __uint_as_float(ra.w), v0);
                    acc = mac(acc, __uint_as_float(rb.y), v1);
                    if (nt > 2) {  // longer tails (and whole rows of layers <= D)
                        const uint2* Eb = (flags & chain::kUnstaged) ? edges : ring_u2;
                        const uint32_t ke = rb.w - 2 + nt;
                        for (uint32_t k = rb.w; k < ke; ++k) {
                            const uint2 ed = Eb[k];
                            acc = mac(acc, __uint_as_float(ed.y), As[off(ed.x, q)]);
                        }
                    }
                    As[ra.y & chain::kDstMask] = sigmoid32(acc);
                    wc_note(n.pos_base + (ra.y & chain::kDstMask) / C, c0 + q, 1);
                }
                __syncwarp();
                if (l + 1 < n.n_layers) chain::f_arrive(2 + (1 - f), kPair);  // layer l final
                if (lane == 0) {
                    heavy::mbar_arrive(&done_bar[(l - 1) % chain::kDoneBars]);
                    if (ra.y & chain::kGroupEnd) heavy::mbar_arrive(&empty[(ra.y >> 20) & (kSlots - 1)]);
                }
                if (l + 2 < n.n_layers) wait_rec(l + 2, ra, rb);
            }
        }
    }
    __syncthreads();
    write_back(n, As, C, A, ldA, c0, n_vec, oinfo, out, write_all, tid, blockDim.x);
}
