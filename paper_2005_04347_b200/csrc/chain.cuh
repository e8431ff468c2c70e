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
//    record {partial sum, destination, first two tail edges as (shared-memory
//    address, weight), tail length + staging slot + flags, index of the
//    third} in a ring of
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
// record ring of a prefix depth D: a power of two >= D + 1 (P writes layer m's
// buffer only after layer m - D - 1 is final; F holds at most layers m-D..m-1)
__host__ __device__ constexpr uint32_t rec_bufs(uint32_t d) { return d < 4 ? 4u : d < 8 ? 8u : 16u; }
// Record tail word rb.z: tail length (< 2^16: a row's in-degree is below the
// network's positions) | staging slot << 16 | group end | unstaged tail.
constexpr uint32_t kTailMask = 0xFFFFu;
constexpr uint32_t kGroupEnd = 1u << 21;  // the layer is its staging group's last
constexpr uint32_t kUnstaged = 1u << 22;  // the tail's edges beyond the second are in global memory
constexpr uint32_t kVal0 = 1u << 23;      // WIN: ra.z holds the first tail source's value (not an address)
constexpr uint32_t kVal1 = 1u << 24;      // WIN: rb.x holds the second's
// Staging plan records (ensure_groups): per group {r0a, e0a, ebytes, wait+1},
// {at | kPlanStaged, rbytes, sbytes, 0}; per layer {a, b, group | kPlanGroupEnd,
// edges_at}, {r0a, e0a, rows_at | kPlanStaged, split_at}.
constexpr uint32_t kPlanStaged = 1u << 31;
constexpr uint32_t kPlanGroupEnd = 1u << 31;
constexpr uint32_t kDoneBars = 16;         // >= D + 2: layer k's barrier is reused for k + kDoneBars

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
// (non-.aligned forms: no warp-convergence fence is emitted around them)
__device__ __forceinline__ void f_sync(uint32_t id, uint32_t n_threads) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n_threads) : "memory");
}
__device__ __forceinline__ void f_arrive(uint32_t id, uint32_t n_threads) {
    asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(n_threads) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
// sigmoid32's 2^(i/32) table from a shared-memory copy (16-byte entries)
struct ExpTabShared {
    uint32_t base;
    __device__ __forceinline__ ulonglong2 operator()(uint32_t i) const {
        ulonglong2 v;
        asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(base + i * 16));
        return v;
    }
};

// Shared-memory bytes past the staging ring: mbarriers + group metas, then
// the record ring (2 x uint4 per item per buffer) and its mbarriers, then the
// layer-done mbarriers.
__host__ __device__ constexpr uint32_t tail_bytes(uint32_t nf, uint32_t np) {
    return cta::kMetaBytes + rec_bufs(np - 1) * (nf * 32 * 32 + 8) + kDoneBars * 8;
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

// The producer (lane 0 of the last warp) executes the host-built plan of
// network n's K groups: wait for the release of the group the plan names
// (the bytes it overwrites, or its mbarrier slot's previous group), then
// three bulk copies (or a plain arrival: the group is read from global
// memory).  ~40 instructions per group instead of the ~200 of the dynamic
// ring bookkeeping.
__device__ __forceinline__ void produce_plan(const uint4* __restrict__ plan, uint32_t K,
                                             const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ split,
                                             const uint2* __restrict__ edges, unsigned char* ring, uint64_t* full,
                                             uint64_t* empty) {
    using namespace cta;
    uint4 p0 = K ? plan[0] : make_uint4(0u, 0u, 0u, 0u), p1 = K ? plan[1] : p0;
    for (uint32_t k = 0; k < K; ++k) {
        const uint4 c0 = p0, c1 = p1;
        if (k + 1 < K) p0 = plan[2 * k + 2], p1 = plan[2 * k + 3];  // next group's plan in flight
        if (c0.w) {
            const uint32_t x = c0.w - 1;
            producer_wait(&empty[x % kSlots], (x / kSlots) & 1);
        }
        uint64_t* fb = &full[k % kSlots];
        if (c1.x & kPlanStaged) {
            const uint32_t at = c1.x & ~kPlanStaged, rbytes = c1.y, sbytes = c1.z, ebytes = c0.z;
            expect_tx(fb, rbytes + sbytes + ebytes);
            bulk_g2s(ring + at, row_ptr + c0.x, rbytes, fb);
            bulk_g2s(ring + at + rbytes, split + c0.x, sbytes, fb);
            if (ebytes) bulk_g2s(ring + at + rbytes + sbytes, edges + c0.y, ebytes, fb);
        } else {
            heavy::mbar_arrive(fb);
        }
    }
}
}  // namespace chain

// WIN (the full slice would need more than one wave of CTAs, config 3): the
// CTA keeps only a ring of the newest W positions in shared memory (slot =
// local position & win_mask) and every activation is written through to A.
// The prefix warps read their sources -- all final, D steps old -- from A (L2;
// they have D steps of slack), and resolve the inline tail edges whose
// sources are already final into values; the finish warps read only sources
// of the last D layers, from the ring.  Two CTAs per SM: one wave.
template <int NF, int NP, bool GUARD, bool WIN>
__global__ void __launch_bounds__(32 * (NF * (2 + NP) + 1), WIN ? 2 : 1)
k_chain(const CtaNet* __restrict__ nets, const uint32_t* __restrict__ unused, const uint4* __restrict__ grp,
        const uint32_t* __restrict__ grp_off, const uint4* __restrict__ lplan,
        const uint32_t* __restrict__ row_ptr, const uint2* __restrict__ edges, const uint4* __restrict__ sinfo,
        const uint4* __restrict__ oinfo, const float* __restrict__ x, uint32_t n_vec, float* __restrict__ A,
        uint32_t ldA, uint32_t C, uint32_t max_pos, uint32_t ring_bytes, int write_all, float* __restrict__ out,
        const uint32_t* __restrict__ split, uint32_t win_mask) {
    using namespace cta;
    constexpr uint32_t D = NP - 1;
    constexpr uint32_t kRecBufs = chain::rec_bufs(D);
    constexpr uint32_t I = NF * 32;  // items of one layer
    static_assert(NP >= 2 && D + 1 <= kRecBufs, "record ring too small for the prefix depth");
    extern __shared__ __align__(128) unsigned char cta_smem[];
    const CtaNet n = nets[blockIdx.y];
    const uint32_t c0 = blockIdx.x * C;
    float* As = reinterpret_cast<float*>(cta_smem);  // [max_pos + 1][C], row max_pos = zeros (WIN: [W][C] ring)
    const uint32_t zero_slot = WIN ? 0u : max_pos;
    const size_t as_floats = ((static_cast<size_t>(WIN ? win_mask + 1 : zero_slot + 1)) * C + 3) & ~size_t(3);
    float* Ag = A + c0;  // WIN: the written-through activations, row stride ldA
    unsigned char* ring = reinterpret_cast<unsigned char*>(As + as_floats);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + ring_bytes);
    uint64_t* empty = full + kSlots;
    uint32_t* meta = reinterpret_cast<uint32_t*>(empty + kSlots);  // unused (plan in global memory)
    uint4* recA = reinterpret_cast<uint4*>(meta + 8 * kSlots);  // [kRecBufs][I]
    uint4* recB = recA + kRecBufs * I;                          // [kRecBufs][I]
    // rec_bar[b]: record buffer b filled (one arrival per P warp of the group);
    // done_bar[(k - 1) % kDoneBars]: layer k final (one arrival per F warp)
    uint64_t* rec_bar = reinterpret_cast<uint64_t*>(recB + kRecBufs * I);
    uint64_t* done_bar = rec_bar + kRecBufs;
    (void)unused;
    const uint4* gplan = grp + 2 * static_cast<size_t>(grp_off[blockIdx.y]);
    const uint32_t n_groups = grp_off[blockIdx.y + 1] - grp_off[blockIdx.y];
    const uint4* lp = lplan + 2 * static_cast<size_t>(n.lo_base);  // layer l: lp[2l], lp[2l + 1]

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
    // records carry 32-bit shared-memory addresses (F's loads and stores need
    // no address arithmetic); the meta area (unused by the plan-driven
    // producer) holds the sigmoid table copy and a scratch word for the
    // stores of items past a layer's width
    const uint32_t as_sh = heavy::smem_u32(As);
    const uint32_t tab_sh = heavy::smem_u32(meta), scratch_sh = tab_sh + 512;
    auto addr = [&](uint32_t pos, uint32_t q) -> uint32_t {
        if constexpr (WIN) return as_sh + 4 * (((pos - n.pos_base) & win_mask) * C + q);
        else return as_sh + 4 * off(pos, q);
    };
    // WIN: a final source's value from A (absolute position; the zero row is zero)
    auto gval = [&](uint32_t pos, uint32_t q) -> float { return Ag[static_cast<size_t>(pos) * ldA + q]; };

    if (tid >= Tc) {
        if (tid == Tc) chain::produce_plan(gplan, n_groups, row_ptr, split, edges, ring, full, empty);
    } else {
        if constexpr (!WIN)
            for (uint32_t c = tid; c < C; c += Tc) As[zero_slot * C + c] = 0.0f;
        for (uint32_t i = tid; i < 64; i += Tc) reinterpret_cast<uint64_t*>(meta)[i] = kExp32Tab[i];
        // sensors (eval.cpp:17), as K-cta
        for (uint32_t i = tid; i < n.n_sensors * C; i += Tc) {
            const uint32_t c = i / n.n_sensors, s = i - c * n.n_sensors;
            const uint32_t k = sinfo[n.sens_prefix + s].w;
            const uint32_t col = c0 + c;
            float xv = 0.0f;
            if (col < n_vec && k != kUnassigned)
                xv = x[static_cast<uint64_t>(n_vec) * n.in_prefix + static_cast<uint64_t>(col) * n.n_in + k];
            const float sv = sigmoid32(xv);
            if constexpr (WIN) {
                Ag[static_cast<size_t>(n.pos_base + s) * ldA + c] = sv;
                As[static_cast<size_t>(s & win_mask) * C + c] = sv;
            } else {
                As[static_cast<size_t>(s) * C + c] = sv;
            }
            wc_note(n.pos_base + s, col, 1);
        }
        consumer_barrier(Tc);

        if (warp >= 2 * NF) {
            // ---- P group j: prefixes of layers m = 1 + j, 1 + j + NP, ... ----
            const uint32_t j = warp / NF - 2, w = warp % NF;
            const uint32_t it = w * 32 + lane;
            const uint32_t i = it / C, q = it - i * C;
            // layer m's plan, loaded one layer of this group ahead
            uint32_t m = 1 + j;
            uint4 pa_n = make_uint4(0u, 0u, 0u, 0u), pb_n = pa_n;
            // WIN: lo[m - D], the first position whose value may not be final
            // when this prefix runs (sources below it are read from A)
            uint32_t rec_n = 0;
            if (m < n.n_layers) {
                pa_n = lp[2 * m], pb_n = lp[2 * m + 1];
                if (WIN && m > D) rec_n = lp[2 * (m - D)].x;
            }
            for (; m < n.n_layers; m += NP) {
                const uint4 pa = pa_n, pb = pb_n;
                const uint32_t recent = rec_n;
                if (m + NP < n.n_layers) {
                    pa_n = lp[2 * (m + NP)], pb_n = lp[2 * (m + NP) + 1];
                    if (WIN && m + NP > D) rec_n = lp[2 * (m + NP - D)].x;
                }
                const uint32_t a = pa.x, b = pa.y, g = pa.z & ~chain::kPlanGroupEnd;
                const bool gend = (pa.z & chain::kPlanGroupEnd) != 0;
                const uint32_t edges_at = pa.w, r0a = pb.x, e0a = pb.y, split_at = pb.w;
                const bool st = (pb.z & chain::kPlanStaged) != 0;
                const uint32_t rows_at = pb.z & ~chain::kPlanStaged;
                // group g's staging (F releases it only after finishing layer m)
                chain::mbar_wait_sleep(&full[g % kSlots], (g / kSlots) & 1);
                // sources on layers <= m - D - 1 are final (layer 0: the
                // sensor barrier); the record buffer (m - 1) % kRecBufs was
                // last read by F at layer m - kRecBufs <= m - D - 1.  Layer k's
                // barrier was last completed for k - kDoneBars, which F
                // finished before this group's previous layer could start.
                if (m > D + 1) {
                    const uint32_t k = m - D - 2;  // layer k + 1 (>= 1) done: phase k / kDoneBars
                    chain::mbar_wait_sleep(&done_bar[k % chain::kDoneBars], (k / chain::kDoneBars) & 1);
                }
                // every item carries the staging slot and group end (F's lane 0
                // releases); an item past the width: sigmoid of +0 into scratch;
                // missing tail edges: the zero row (WIN: the value 0) with weight 0
                const uint32_t tag = (g % kSlots) << 16 | (gend ? chain::kGroupEnd : 0u) |
                                     (WIN ? chain::kVal0 | chain::kVal1 : 0u);
                const uint32_t zo = WIN ? 0u : as_sh + 4 * (zero_slot * C + q);
                uint4 ra = make_uint4(0u, scratch_sh, zo, 0u), rb = make_uint4(zo, 0u, tag, 0u);
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
                    // (the tail first: its final sources' loads overlap the prefix's)
                    ra.y = WIN ? as_sh + 4 * (((a + i) & win_mask) * C + q) : as_sh + 4 * ((a + i) * C + q);
                    uint32_t vflags = WIN ? chain::kVal0 | chain::kVal1 : 0u;
                    // WIN: a tail source below `recent` is final now -- its value
                    // goes into the record; the others are read from the ring
                    auto tail_src = [&](uint32_t pos, uint32_t vbit) -> uint32_t {
                        if constexpr (WIN) {
                            if (pos - n.pos_base >= recent && pos - n.pos_base < n.n_pos) {
                                vflags &= ~vbit;
                                return addr(pos, q);
                            }
                            return __float_as_uint(gval(pos, q));
                        } else {
                            return addr(pos, q);
                        }
                    };
                    if (ke > ks) {
                        const uint2 e0 = Ep[ks];
                        ra.z = tail_src(e0.x, chain::kVal0);
                        ra.w = e0.y;
                    }
                    if (ke > ks + 1) {
                        const uint2 e1 = Ep[ks + 1];
                        rb.x = tail_src(e1.x, chain::kVal1);
                        rb.y = e1.y;
                    }
                    // batches of 8 (the last one predicated): all of a batch's
                    // source loads in flight together -- under WIN they are L2
                    // round trips, which a one-edge remainder loop would serialise
                    float acc = 0.0f;
                    for (; k < ks; k += 8) {
                        const uint32_t nb = min(8u, ks - k);
                        uint2 ed[8];
                        float av[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (u < nb) ed[u] = Ep[k + u];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (u < nb) av[u] = WIN ? gval(ed[u].x, q) : As[off(ed[u].x, q)];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (u < nb) acc = mac(acc, __uint_as_float(ed[u].y), av[u]);
                    }
                    ra.x = __float_as_uint(acc);
                    // F reads edges beyond the second from ring_u2 (staged,
                    // index relative to the ring) or edges (absolute)
                    rb.z = ((tag & ~(chain::kVal0 | chain::kVal1)) | vflags) | (ke - ks) | (st ? 0u : chain::kUnstaged);
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
            uint4 ra = make_uint4(0u, 0u, 0u, 0u), rb = ra;
            uint32_t l = 1 + f;
            uint32_t lo_l = 0;  // WIN: lo[l], for the write-through position
            if (l < n.n_layers) {
                wait_rec(l, ra, rb);
                if (WIN) lo_l = lp[2 * l].x;
            }
            for (; l < n.n_layers; l += 2) {
                const uint32_t lo_next = WIN && l + 2 < n.n_layers ? lp[2 * (l + 2)].x : 0u;
                // layer l-1 final (the other group; layer 0: the sensor barrier)
                if (l > 1) chain::f_sync(2 + f, kPair);
                const uint32_t flags = rb.z, nt = flags & chain::kTailMask;
                float v0 = __uint_as_float(ra.z), v1 = __uint_as_float(rb.x);
                if (!WIN || !(flags & chain::kVal0)) v0 = chain::lds_f32(ra.z);
                if (!WIN || !(flags & chain::kVal1)) v1 = chain::lds_f32(rb.x);
                float acc = __uint_as_float(ra.x);
                acc = mac(acc, __uint_as_float(ra.w), v0);
                acc = mac(acc, __uint_as_float(rb.y), v1);
                if (nt > 2) {  // longer tails (and whole rows of layers <= D)
                    const uint2* Eb = (flags & chain::kUnstaged) ? edges : ring_u2;
                    const uint32_t ke = rb.w - 2 + nt;
                    // WIN: sources below lo[l - D] are final and may have left the ring
                    const uint32_t recent = WIN && l > D ? lp[2 * (l - D)].x : 0u;
                    for (uint32_t k = rb.w; k < ke; ++k) {
                        const uint2 ed = Eb[k];
                        float v;
                        if constexpr (WIN)
                            v = ed.x - n.pos_base >= recent && ed.x - n.pos_base < n.n_pos
                                    ? chain::lds_f32(addr(ed.x, q)) : gval(ed.x, q);
                        else
                            v = chain::lds_f32(addr(ed.x, q));
                        acc = mac(acc, __uint_as_float(ed.y), v);
                    }
                }
                const float y = sigmoid32(acc, chain::ExpTabShared{tab_sh});
                chain::sts_f32(ra.y, y);
                // WIN: the write-through precedes the handoff -- a prefix warp
                // that saw layer l+1 done (done_bar, released after the other
                // group's barrier.sync) must also see layer l in A
                const uint32_t pos_w = n.pos_base + lo_l + it / C;  // WIN: this item's position
                if constexpr (WIN)
                    if (ra.y != scratch_sh) Ag[static_cast<size_t>(pos_w) * ldA + q] = y;
                if (l + 1 < n.n_layers) chain::f_arrive(2 + (1 - f), kPair);  // layer l final
                lo_l = lo_next;
#ifdef ASNN_WRITE_COUNT
                if (ra.y != scratch_sh)
                    wc_note(WIN ? pos_w : n.pos_base + (ra.y - as_sh) / 4 / C, c0 + q, 1);
#endif
                __syncwarp();
                if (lane == 0) {
                    heavy::mbar_arrive(&done_bar[(l - 1) % chain::kDoneBars]);
                    if (flags & chain::kGroupEnd) heavy::mbar_arrive(&empty[(flags >> 16) & (kSlots - 1)]);
                }
                if (l + 2 < n.n_layers) wait_rec(l + 2, ra, rb);
            }
        }
    }
    __syncthreads();
    if constexpr (WIN) {
        // every activation is already in A: only the declared outputs (eval.cpp:82-87)
        if (out) {
            const uint32_t vcols = c0 < n_vec ? min(C, n_vec - c0) : 0u;
            for (uint32_t i = tid; i < n.n_out * vcols; i += blockDim.x) {
                const uint32_t c = i / n.n_out, j = i - c * n.n_out;
                const uint32_t pos = oinfo[n.out_prefix + j].x;
                out[static_cast<uint64_t>(n_vec) * n.out_prefix + static_cast<uint64_t>(c0 + c) * n.n_out + j] =
                    pos != kUnassigned ? Ag[static_cast<size_t>(pos) * ldA + c] : 0.0f;
            }
        }
    } else {
        write_back(n, As, C, A, ldA, c0, n_vec, oinfo, out, write_all, tid, blockDim.x);
    }
}
