// cta.cuh -- K-cta: the whole level sweep of one network for one slice of C
// batch columns inside ONE CTA.  The paper's Algorithm 3 (one block, a
// barrier per layer) done right:
//  * the slice's activations live in shared memory (gathers are LDS);
//  * a producer warp stages each layer's row pointers and {col, w} edges --
//    contiguous in the level-sorted CSR -- with two TMA bulk copies into a
//    ring of R slots (a power of two chosen to fill shared memory; mbarrier
//    complete_tx), up to R-1 layers ahead of the one computing; consumer
//    warps release slots through an "empty" mbarrier;
//  * the consumer warps' per-layer critical path is LDS + the in-order FADD
//    chain + the sigmoid + one named barrier among themselves;
//  * batch columns (and networks of a population) are independent, so CTAs
//    never synchronise with each other -- no grid barrier, no kernel boundary
//    per layer.
// Used for deep/narrow networks, small networks and populations whose
// per-slice activations fit in shared memory (C1, C3, C5).
// Included by kernels.cuh inside namespace asnn_b200 (uses heavy::, sigmoid32, mac).
#pragma once

struct CtaNet {
    uint32_t pos_base, n_pos, n_sensors, sens_prefix;
    uint32_t in_prefix, n_in, out_prefix, n_out;
    uint32_t lo_base, n_layers, pad0, pad1;
};

namespace cta {

__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     heavy::smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            heavy::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(heavy::smem_u32(bar))
        : "memory");
}
// The producer's waits for ring space: it runs ahead of the consumers, so it
// waits suspended in the hardware (try_wait with a suspend-time hint, woken
// when the phase completes) instead of spinning -- a spinning producer warp
// takes issue slots from the consumer warp sharing its SM sub-partition.  (A
// __nanosleep back-off oversleeps: on config 3 under K-chain it held the
// staging rate to one layer per ~1250 cycles.)
__device__ __forceinline__ void producer_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "PWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra PWAIT_%=;\n}" ::"r"(heavy::smem_u32(b)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void consumer_barrier(uint32_t n_threads) {
    asm volatile("bar.sync 1, %0;" ::"r"(n_threads) : "memory");
}

// One layer's items for one thread: item it = (node i, column group q).
// Rp / Ep point at the staged slot (shared memory) or at the global arrays.
// As holds the slice's activations with row stride ld; position p lives in
// row p - row_base (shared memory: the network's rows, row_base = pos_base;
// global/L2 mode: the whole A, row_base = 0, As already offset by c0).
//
// MODE 0: whole rows, sigmoid into As.  MODE 1 (pipelined finish): start at
// the row's split edge with the partial sum left in pre[] by MODE 2 one step
// earlier.  MODE 2 (pipelined prefix): sum the edges before the row's split
// (split[i] for the layer's row i: staged slice or global, absolute edge
// indices) and park the partial sum and the split in pre[] / pre_k[] for
// MODE 1.
// WIN (one network deeper than shared memory holds for one wave of CTAs):
// shared memory keeps a ring of the newest W positions' activations (slot =
// local position & mask, the zero row at slot W) and every activation is
// also written through to A; at the step that finishes layer l a source is
// read from the ring iff its local position >= lo = end(l) - W (not
// overwritten before or during the step), otherwise from A (written by this
// CTA at an earlier step, ordered by the layer barrier; L2-resident).
// The prefix group's out-of-ring sources are staged one step early: right
// after summing layer l+1's prefix at step l it issues cp.async copies of
// the A values layer l+2's prefix will need from outside the ring (positions
// < end(l+1) - W, final since step l-1) into stg, so at step l+1 they are
// shared-memory reads and the L2 round trip left the critical path.  stg
// (when non-null) holds, for Ep-relative edge index k, the staged value of
// column group q at stg[k << gshift | q].
struct Win {
    float* Ag;      // A + c0
    uint32_t ldA;
    uint32_t mask;  // W - 1
    int32_t lo;
    const float* stg;
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(heavy::smem_u32(dst)), "l"(src) : "memory");
}

// Stage layer [a, b)'s prefix sources (edges [Rp[i], Sp[i]) of each row)
// that lie outside the ring at the step that will consume them (local
// position < lo).  Same (row, column group) -> thread map as layer_items.
template <bool GUARD>
__device__ __forceinline__ void stage_prefix(const uint32_t* Rp, const uint32_t* Sp, const uint2* Ep, uint32_t eb,
                                             uint32_t a, uint32_t b, uint32_t gshift, uint32_t pos_base,
                                             uint32_t n_pos, int32_t lo, const float* Ag, uint32_t ldA, float* stg,
                                             uint32_t tid, uint32_t T) {
    const uint32_t groups_mask = (1u << gshift) - 1u;
    for (uint32_t it = tid; it < ((b - a) << gshift); it += T) {
        const uint32_t i = it >> gshift, q = it & groups_mask;
        const uint32_t k1 = Sp[i] - eb;
        for (uint32_t k = Rp[i] - eb; k < k1; ++k) {
            const uint32_t pos = Ep[k].x;
            const uint32_t p = pos - pos_base;
            if (GUARD && p >= n_pos) continue;
            if (static_cast<int32_t>(p) < lo) cp_async4(stg + (k << gshift) + q, Ag + static_cast<size_t>(pos) * ldA + q);
        }
    }
}

template <int V, bool GUARD, int MODE = 0, bool WIN = false>
__device__ __forceinline__ void layer_items(float* As, const uint32_t* Rp, const uint2* Ep, uint32_t e0,
                                            uint32_t a, uint32_t b, uint32_t ld, uint32_t gshift,
                                            uint32_t pos_base, uint32_t row_base, uint32_t n_pos,
                                            uint32_t zero_row, uint32_t tid, uint32_t T,
                                            float* pre = nullptr, uint32_t* pre_k = nullptr,
                                            const uint32_t* split = nullptr, Win win = {}) {
    static_assert(!WIN || V == 1, "the windowed variant runs one column per item");
    if constexpr (WIN && MODE == 2)
        if (win.stg) asm volatile("cp.async.wait_group 1;" ::: "memory");  // staged a step ago (not the newest group)
    const uint32_t groups_mask = (1u << gshift) - 1u;
    for (uint32_t it = tid; it < ((b - a) << gshift); it += T) {
        const uint32_t i = it >> gshift, q = it & groups_mask;
        uint32_t k, ke;
        if constexpr (MODE == 0) {
            k = Rp[i] - e0;
            ke = Rp[i + 1] - e0;
        } else if constexpr (MODE == 1) {
            k = pre_k[i] - e0;
            ke = Rp[i + 1] - e0;
        } else {
            k = Rp[i] - e0;
            const uint32_t sp = split[i];
            ke = sp - e0;
            if (q == 0) pre_k[i] = sp;
        }
        const float* Aq = As + q * V;
        // GUARD: some predecessor of this layout has no position (hand-built
        // layouts only); it reads the zero row
        auto row = [&](uint32_t pos) -> size_t {
            const uint32_t p = pos - row_base;
            if constexpr (GUARD) return static_cast<size_t>(p - (pos_base - row_base) < n_pos ? p : zero_row) * ld;
            else return static_cast<size_t>(p) * ld;
        };
        // the address of source `pos`, column group q (WIN: ring or A)
        auto src_of = [&](uint32_t pos, uint32_t k_cur) -> const float* {
            if constexpr (WIN) {
                const uint32_t p = pos - pos_base;
                if (GUARD && p >= n_pos) return Aq + static_cast<size_t>(zero_row) * ld;
                if (static_cast<int32_t>(p) >= win.lo) return Aq + static_cast<size_t>(p & win.mask) * ld;
                if (MODE == 2 && win.stg) return win.stg + (k_cur << gshift) + q;
                return win.Ag + static_cast<size_t>(pos) * win.ldA + q;
            } else {
                return Aq + row(pos);
            }
        };
        float acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = MODE == 1 ? pre[it * V + v] : 0.0f;
        // four edges' loads in flight, then their adds in stored order
        for (; k + 4 <= ke; k += 4) {
            uint2 ed[4];
            float av[4][V];
#pragma unroll
            for (int j = 0; j < 4; ++j) ed[j] = Ep[k + j];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float* src = src_of(ed[j].x, k + j);
                if constexpr (V == 4) {
                    const float4 t = *reinterpret_cast<const float4*>(src);
                    av[j][0] = t.x;
                    av[j][1] = t.y;
                    av[j][2] = t.z;
                    av[j][3] = t.w;
                } else {
#pragma unroll
                    for (int v = 0; v < V; ++v) av[j][v] = src[v];
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = mac(acc[v], __uint_as_float(ed[j].y), av[j][v]);
        }
        for (; k < ke; ++k) {
            const uint2 ed = Ep[k];
            const float* src = src_of(ed.x, k);
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = mac(acc[v], __uint_as_float(ed.y), src[v]);
        }
        if constexpr (MODE == 2) {
#pragma unroll
            for (int v = 0; v < V; ++v) pre[it * V + v] = acc[v];
            continue;
        }
        float* dst = As + static_cast<size_t>(WIN ? ((a + i) & win.mask) : pos_base - row_base + a + i) * ld + q * V;
        sigmoid32_v<V>(acc);
        if constexpr (WIN) win.Ag[static_cast<size_t>(pos_base + a + i) * win.ldA + q] = acc[0];
        wc_note(pos_base + a + i, blockIdx.x * ((groups_mask + 1) * V) + q * V, V);
        if constexpr (V == 4) {
            *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v) dst[v] = acc[v];
        }
    }
}
}  // namespace cta

#ifdef ASNN_CHAIN_PROF
static __device__ long long g_issue_clk[4096];
static __device__ long long g_trace[5][4096];  // issue, P full ready, P done, F done, producer space-wait start
#endif
namespace cta {
constexpr uint32_t kSlots = 32;
constexpr uint32_t kMetaBytes = kSlots * (8 + 8 + 32);

// The producer (one warp; lane 0 issues the copies): stages layers
// 1..n_layers-1 in order into the ring.  The layer bounds (lo, le) are read
// 32 layers at a time by the warp's lanes and broadcast with __shfl, the next
// window loaded one window ahead: a dependent L2 round trip per layer capped
// the staging rate at ~1 layer / 1000 cycles (config 3 under K-chain).  meta[m] = {a, b, e0, staged, row index, edge index, extent, split
// index} of the layer using slot m; the extent (its bytes plus the wasted tail
// when it wrapped) is what its release frees, so the live bytes are always
// [w - used, w) modulo the ring.  SPLIT: the layer's split[] slice is staged
// too.  keep: the newest layers whose release the producer never waits for
// (the consumers need them staged before they release the older ones) --
// such a layer is read from global memory instead.
template <bool SPLIT>
__device__ __forceinline__ void produce(const CtaNet& n, const uint32_t* __restrict__ lo_cat,
                                        const uint32_t* __restrict__ le_cat, const uint32_t* __restrict__ row_ptr,
                                        const uint32_t* __restrict__ split, const uint2* __restrict__ edges,
                                        unsigned char* ring, uint32_t ring_bytes, uint64_t* full, uint64_t* empty,
                                        uint32_t* meta, int write_all, uint32_t keep, uint32_t lane) {
#ifdef ASNN_CHAIN_PROF
#define PROD_T0(v) const long long v = clock64()
#define PROD_T1(v, acc) acc += clock64() - v
    long long w_slot = 0, w_space = 0, w_issue = 0, w_total = 0;
    const long long t_start = clock64();
#else
#define PROD_T0(v)
#define PROD_T1(v, acc)
#endif
    uint32_t n_space = 0, n_global = 0;
    (void)n_space, (void)n_global;
    const uint32_t* lo = lo_cat + n.lo_base;
    const uint32_t* le = le_cat + n.lo_base;
    uint32_t w = 0;       // next write offset in the ring
    uint32_t used = 0;    // bytes of layers in flight (incl. wrap gaps)
    uint32_t oldest = 1;  // oldest layer whose release the producer has not seen
    auto release_to = [&](uint32_t upto) {  // layers < upto are released
        for (; oldest < upto; ++oldest) used -= meta[8 * ((oldest - 1) % kSlots) + 6];
    };
    // window [base, base + 32) of layer bounds in lanes (lo_c, le_c), the next
    // one (base + 31: windows overlap by one so l and l + 1 share one) in flight
    uint32_t base = 1, lo_c, le_c, lo_n, le_n;
    {
        const uint32_t i0 = min(base + lane, n.n_layers), i1 = min(base + 31 + lane, n.n_layers);
        lo_c = lo[i0], le_c = le[i0], lo_n = lo[i1], le_n = le[i1];
    }
    const bool leader = lane == 0;
    for (uint32_t l = 1; l < n.n_layers; ++l) {
        if (l - base == 31) {
            base += 31;
            lo_c = lo_n, le_c = le_n;
            const uint32_t i1 = min(base + 31 + lane, n.n_layers);
            lo_n = lo[i1], le_n = le[i1];
        }
        const uint32_t m = (l - 1) % kSlots, u = (l - 1) / kSlots;
        const uint32_t a = __shfl_sync(0xFFFFFFFFu, lo_c, l - base), b = __shfl_sync(0xFFFFFFFFu, lo_c, l - base + 1);
        const uint32_t e0 = __shfl_sync(0xFFFFFFFFu, le_c, l - base), e1 = __shfl_sync(0xFFFFFFFFu, le_c, l - base + 1);
        const uint32_t r0 = n.pos_base + a, r0a = r0 & ~3u;
        const uint32_t rbytes = ((b - a + 1 + (r0 - r0a)) * 4 + 15) & ~15u;
        // the layer's split[] slice too (same alignment as row_ptr)
        const uint32_t sbytes = SPLIT ? ((b - a + (r0 - r0a)) * 4 + 15) & ~15u : 0u;
        const uint32_t e0a = e0 & ~1u;
        const uint32_t ebytes = ((e1 - e0 + (e0 - e0a)) * 8 + 15) & ~15u;
        const uint32_t size = rbytes + sbytes + ebytes;
        if (u > 0) {  // slot m's previous layer (l - kSlots) and all before it are released
            PROD_T0(t0);
            producer_wait(&empty[m], (u - 1) & 1);
            PROD_T1(t0, w_slot);
            release_to(l - kSlots + 1);
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
                // pipelined consumers: layer l-1 is released only after the
                // step that also needs layer l (its prefix): never wait for
                // it -- layer l is then read from global memory instead
                if (keep && oldest + keep >= l) {
                    staged = false;
                    break;
                }
                PROD_T0(t1);
#ifdef ASNN_CHAIN_PROF
                if (blockIdx.x == 0 && blockIdx.y == 0 && l < 4096 && leader) g_trace[4][l] = oldest;
#endif
                producer_wait(&empty[(oldest - 1) % kSlots], ((oldest - 1) / kSlots) & 1);
                PROD_T1(t1, w_space);
                ++n_space;
                release_to(oldest + 1);
            }
        }
        if (leader) {
            uint32_t* mm = meta + 8 * m;
            mm[0] = a;
            mm[1] = b;
            mm[2] = e0;
            mm[3] = staged ? 1u : 0u;
            mm[4] = at / 4 + (r0 - r0a);
            mm[5] = (at + rbytes + sbytes) / 8 + (e0 - e0a);
            mm[6] = extent;
            mm[7] = (at + rbytes) / 4 + (r0 - r0a);
#ifdef ASNN_CHAIN_PROF
            if (blockIdx.x == 0 && blockIdx.y == 0 && l < 4096) g_issue_clk[l] = clock64();
#endif
            if (staged) {
                PROD_T0(t2);
                expect_tx(&full[m], size);
                bulk_g2s(ring + at, row_ptr + r0a, rbytes, &full[m]);
                if (sbytes) bulk_g2s(ring + at + rbytes, split + r0a, sbytes, &full[m]);
                if (ebytes) bulk_g2s(ring + at + rbytes + sbytes, edges + e0a, ebytes, &full[m]);
                PROD_T1(t2, w_issue);
            } else {
                heavy::mbar_arrive(&full[m]);
                ++n_global;
            }
        }
        __syncwarp();  // the extent in meta is read by every lane's release_to
    }
#ifdef ASNN_CHAIN_PROF
    if (blockIdx.x == 0 && blockIdx.y == 0 && leader)
        printf("producer: total %lld, slot waits %lld cycles, space waits %lld cycles (%u), issue %lld, unstaged layers %u, ring %u\n",
               clock64() - t_start, w_slot, w_space, n_space, w_issue, n_global, ring_bytes);
#endif
}
}  // namespace cta

namespace cta {
// Write back after the sweep: every row (state requested) or only the
// declared outputs, from the CTA's shared-memory rows As ([n_pos][C]).
__device__ __forceinline__ void write_back(const CtaNet& n, const float* As, uint32_t C, float* __restrict__ A,
                                           uint32_t ldA, uint32_t c0, uint32_t n_vec,
                                           const uint4* __restrict__ oinfo, float* __restrict__ out,
                                           int write_all, uint32_t tid, uint32_t T) {
    const uint32_t ncols = min(C, ldA - c0);
    if (write_all & 1) {
        for (uint32_t i = tid; i < n.n_pos * ncols; i += T) {
            const uint32_t p = i / ncols, c = i - p * ncols;
            A[static_cast<uint64_t>(n.pos_base + p) * ldA + c0 + c] = As[p * C + c];
        }
    } else if (out) {
        // read_outputs (eval.cpp:82-87) straight from shared memory into the
        // caller's [net][vector][output] buffer (device or mapped host memory):
        // no output gather launch, and the writes of finished CTAs overlap the
        // sweeps of the others
        const uint32_t vcols = c0 < n_vec ? min(C, n_vec - c0) : 0u;
        for (uint32_t i = tid; i < n.n_out * vcols; i += T) {
            const uint32_t c = i / n.n_out, j = i - c * n.n_out;
            const uint32_t pos = oinfo[n.out_prefix + j].x;
            out[static_cast<uint64_t>(n_vec) * n.out_prefix + static_cast<uint64_t>(c0 + c) * n.n_out + j] =
                pos != kUnassigned ? As[(pos - n.pos_base) * C + c] : 0.0f;
        }
    } else {
        for (uint32_t i = tid; i < n.n_out * ncols; i += T) {
            const uint32_t j = i / ncols, c = i - j * ncols;
            const uint32_t pos = oinfo[n.out_prefix + j].x;
            if (pos != kUnassigned)
                A[static_cast<uint64_t>(pos) * ldA + c0 + c] = As[(pos - n.pos_base) * C + c];
        }
    }
}
}  // namespace cta

// Block = consumer warps + 1 producer warp (the last).  Shared memory:
// [As[(max_pos+1)*C, 16-B rounded; row max_pos is zeros] unless GLOBAL] |
// ring[ring_bytes] | full[kSlots], empty[kSlots] u64 | meta[kSlots][8] u32.
// The ring is byte-granular: layer l's row pointers and edges (16-byte
// aligned bulk copies) are packed at the producer's write offset, wrapping to
// 0 when they do not fit before the end, so as many layers are in flight as
// their sizes allow (up to kSlots) -- small layers no longer pay for a slot
// sized by the largest one.  Layers larger than the ring (or every layer in
// debug mode 2) are read from global memory.  Layer l uses mbarrier pair
// (l-1) % kSlots for its ((l-1) / kSlots)-th time.

//
// PIPE (latency-bound layers: at most two warps of items): the consumers form
// two groups.  At step l the finish group completes layer l (the edges from
// each row's split on, whose sources include level l-1, then sigmoid32) while
// the prefix group sums layer l+1's rows up to their split (sources at levels
// <= l-1, final since step l-1) -- half of each layer's dependent work moves
// off the critical path.  The fp32 sum of a row is the same sequence of
// roundings (segments.cuh); split[] comes from k_splits.
template <int V, bool GUARD, bool GLOBAL, bool PIPE = false, bool WIN = false>
__global__ void __launch_bounds__(544)
k_cta(const CtaNet* __restrict__ nets, const uint32_t* __restrict__ lo_cat,
      const uint32_t* __restrict__ le_cat, const uint32_t* __restrict__ row_ptr,
      const uint2* __restrict__ edges, const uint4* __restrict__ sinfo,
      const uint4* __restrict__ oinfo, const float* __restrict__ x, uint32_t n_vec,
      float* __restrict__ A, uint32_t ldA, uint32_t C, uint32_t max_pos, uint32_t ring_bytes,
      int write_all, float* __restrict__ out, const uint32_t* __restrict__ split, uint32_t max_items,
      uint32_t win_mask, uint32_t stg_edges) {
    using namespace cta;
    extern __shared__ __align__(128) unsigned char cta_smem[];
    const CtaNet n = nets[blockIdx.y];
    const uint32_t c0 = blockIdx.x * C;
    // activations: shared-memory rows of this network (row max_pos is the
    // zero row for predecessors without a position), or A itself
    float* As = GLOBAL ? A + c0 : reinterpret_cast<float*>(cta_smem);
    const uint32_t ld = GLOBAL ? ldA : C;
    const uint32_t row_base = GLOBAL ? 0u : n.pos_base;
    // WIN: the ring of the newest W = win_mask + 1 positions, the zero row at slot W
    const uint32_t zero_slot = WIN ? win_mask + 1 : max_pos;
    const size_t as_floats = GLOBAL ? 0 : ((static_cast<size_t>(zero_slot + 1) * C + 3) & ~size_t(3));
    const Win win0{A + c0, ldA, win_mask, 0};
    unsigned char* ring = reinterpret_cast<unsigned char*>(reinterpret_cast<float*>(cta_smem) + as_floats);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + ring_bytes);
    uint64_t* empty = full + kSlots;
    uint32_t* meta = reinterpret_cast<uint32_t*>(empty + kSlots);
    // PIPE: two parity buffers of partial sums [max_items * V] and splits [max_items]
    float* pre = reinterpret_cast<float*>(meta + 8 * kSlots);
    uint32_t* pre_k = reinterpret_cast<uint32_t*>(pre + 2 * max_items * V);
    // WIN + PIPE: two parity buffers of staged prefix sources [stg_edges * C]
    float* stg_buf = reinterpret_cast<float*>(pre_k + 2 * max_items);

    const uint32_t groups = C / V;  // column groups per row (a power of two)
    const uint32_t gshift = __ffs(groups) - 1;
    const uint32_t Tc = blockDim.x - 32;  // consumer threads
    const uint32_t tid = threadIdx.x;

    if (tid == 0) {
        for (uint32_t s = 0; s < kSlots; ++s) {
            heavy::mbar_init(&full[s], 1);
            heavy::mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= Tc) {
        cta::produce<PIPE>(n, lo_cat, le_cat, row_ptr, split, edges, ring, ring_bytes, full, empty, meta,
                           write_all, PIPE ? (WIN && stg_edges ? 2u : 1u) : 0u, tid - Tc);
    } else {
        if constexpr (!GLOBAL)
            for (uint32_t c = tid; c < C; c += Tc) As[zero_slot * C + c] = 0.0f;
        // sensors: eval.cpp:17 (sigmoided input values), overlapping the staging.
        // One (column, sensor) per thread, sensor fastest: a column's inputs
        // are contiguous in x ([vector][input]), so the reads coalesce (they
        // may cross the host link when x is mapped host memory).
        for (uint32_t i = tid; i < n.n_sensors * C; i += Tc) {
            const uint32_t c = i / n.n_sensors, s = i - c * n.n_sensors;
            const uint32_t k = sinfo[n.sens_prefix + s].w;
            const uint32_t col = c0 + c;
            float xv = 0.0f;
            if (col < n_vec && k != kUnassigned)
                xv = x[static_cast<uint64_t>(n_vec) * n.in_prefix + static_cast<uint64_t>(col) * n.n_in + k];
            const float sv = sigmoid32(xv);
            if constexpr (WIN) {
                A[static_cast<uint64_t>(n.pos_base + s) * ldA + col] = sv;
                if (s + win_mask + 1 >= n.n_sensors) As[static_cast<size_t>(s & win_mask) * ld + c] = sv;
            } else {
                As[static_cast<size_t>(n.pos_base - row_base + s) * ld + c] = sv;
            }
            wc_note(n.pos_base + s, col, 1);
        }
        consumer_barrier(Tc);
        const uint32_t* ring_u32 = reinterpret_cast<const uint32_t*>(ring);
        const uint2* ring_u2 = reinterpret_cast<const uint2*>(ring);
        if constexpr (PIPE) {
            const uint32_t Th = Tc / 2;
            const bool fin = tid < Th;
            const uint32_t gtid = fin ? tid : tid - Th;
            for (uint32_t l = 0; l < n.n_layers; ++l) {
                // finish layer l (l >= 1) | prefix of layer l+1
                const uint32_t ll = fin ? l : l + 1;
                if ((fin && l >= 1) || (!fin && ll < n.n_layers)) {
                    const uint32_t m = (ll - 1) % kSlots;
                    heavy::mbar_wait(&full[m], ((ll - 1) / kSlots) & 1);
                    const uint32_t* mm = meta + 8 * m;
                    const uint32_t a = mm[0], b = mm[1], e0 = mm[2];
                    const uint32_t* Rp = mm[3] ? ring_u32 + mm[4] : row_ptr + n.pos_base + a;
                    const uint32_t* Sp = mm[3] ? ring_u32 + mm[7] : split + n.pos_base + a;
                    const uint2* Ep = mm[3] ? ring_u2 + mm[5] : edges;
                    const uint32_t eb = mm[3] ? e0 : 0u;
                    float* pb = pre + (ll & 1) * max_items * V;
                    uint32_t* pk = pre_k + (ll & 1) * max_items;
                    // this step's ring boundary: the end of layer l (= b of the
                    // finish group's layer, a of the prefix group's)
                    Win win = win0;
                    win.lo = static_cast<int32_t>(fin ? b : a) - static_cast<int32_t>(win_mask + 1);
                    if (fin) {
                        layer_items<V, GUARD, 1, WIN>(As, Rp, Ep, eb, a, b, ld, gshift, n.pos_base, row_base,
                                                      n.n_pos, zero_slot, gtid, Th, pb, pk, Sp, win);
                    } else {
                        // stage layer ll+1's out-of-ring prefix sources for the next
                        // step first: their L2 round trip overlaps this step's work
                        if constexpr (WIN)
                            if (stg_edges && ll + 1 < n.n_layers) {
                                const uint32_t m2 = ll % kSlots;
                                heavy::mbar_wait(&full[m2], (ll / kSlots) & 1);
                                const uint32_t* m2m = meta + 8 * m2;
                                const uint32_t a2 = m2m[0], b2 = m2m[1], e02 = m2m[2];
                                const uint32_t* Rp2 = m2m[3] ? ring_u32 + m2m[4] : row_ptr + n.pos_base + a2;
                                const uint32_t* Sp2 = m2m[3] ? ring_u32 + m2m[7] : split + n.pos_base + a2;
                                const uint2* Ep2 = m2m[3] ? ring_u2 + m2m[5] : edges;
                                const uint32_t eb2 = m2m[3] ? e02 : 0u;
                                float* st2 = stg_buf + ((ll + 1) & 1) * stg_edges * C -
                                             (static_cast<size_t>(e02 - eb2) << gshift);
                                stage_prefix<GUARD>(Rp2, Sp2, Ep2, eb2, a2, b2, gshift, n.pos_base, n.n_pos,
                                                    static_cast<int32_t>(b) - static_cast<int32_t>(win_mask + 1),
                                                    win0.Ag, ldA, st2, gtid, Th);
                            }
                        // one group per step, empty or not: wait_group 1 below then
                        // always means "everything staged before this step"
                        if constexpr (WIN)
                            if (stg_edges) asm volatile("cp.async.commit_group;" ::: "memory");
                        if constexpr (WIN)
                            if (stg_edges) win.stg = stg_buf + (ll & 1) * stg_edges * C - (static_cast<size_t>(e0 - eb) << gshift);
                        layer_items<V, GUARD, 2, WIN>(As, Rp, Ep, eb, a, b, ld, gshift, n.pos_base, row_base,
                                                      n.n_pos, zero_slot, gtid, Th, pb, pk, Sp, win);
                    }
                }
                consumer_barrier(Tc);  // layer l final, prefix of l+1 parked
                if (tid == 0 && l >= 1) heavy::mbar_arrive(&empty[(l - 1) % kSlots]);
            }
        } else
        for (uint32_t l = 1; l < n.n_layers; ++l) {
            const uint32_t m = (l - 1) % kSlots;
            heavy::mbar_wait(&full[m], ((l - 1) / kSlots) & 1);
            const uint32_t* mm = meta + 8 * m;
            const uint32_t a = mm[0], b = mm[1], e0 = mm[2];
            Win win = win0;
            win.lo = static_cast<int32_t>(b) - static_cast<int32_t>(win_mask + 1);
            if (mm[3])
                layer_items<V, GUARD, 0, WIN>(As, ring_u32 + mm[4], ring_u2 + mm[5], e0, a, b, ld, gshift,
                                              n.pos_base, row_base, n.n_pos, zero_slot, tid, Tc, nullptr,
                                              nullptr, nullptr, win);
            else
                layer_items<V, GUARD, 0, WIN>(As, row_ptr + n.pos_base + a, edges, 0, a, b, ld, gshift,
                                              n.pos_base, row_base, n.n_pos, zero_slot, tid, Tc, nullptr,
                                              nullptr, nullptr, win);
            consumer_barrier(Tc);  // layer l visible to every consumer
            if (tid == 0) heavy::mbar_arrive(&empty[m]);
        }
    }
    if constexpr (GLOBAL || WIN) return;  // the activations are already in A
    __syncthreads();

    cta::write_back(n, As, C, A, ldA, c0, n_vec, oinfo, out, write_all, tid, blockDim.x);
}

// split[p] for every non-sensor position p of network blockIdx.y: the first
// stored edge (ascending source id) whose source is on a layer >= level(p) -
// D, as an absolute edge index; the edges before it have all their sources on
// layers <= level(p) - D - 1 (K-cta's pipelined consumers use D = 1, K-chain
// D = its prefix groups - 1).  Sources outside the network (the zero row)
// count as layer 0.
__global__ void k_splits(const CtaNet* __restrict__ nets, const uint32_t* __restrict__ lo_cat,
                         const uint32_t* __restrict__ row_ptr, const uint2* __restrict__ edges,
                         uint32_t* __restrict__ split, uint32_t D) {
    const CtaNet n = nets[blockIdx.y];
    const uint32_t lp = blockIdx.x * blockDim.x + threadIdx.x;
    if (lp >= n.n_pos || lp < n.n_sensors) return;
    const uint32_t* lo = lo_cat + n.lo_base;
    auto layer_of = [&](uint32_t q) {  // lo[a] <= q < lo[a + 1]
        uint32_t a = 0, b = n.n_layers;
        while (b - a > 1) {
            const uint32_t m = (a + b) / 2;
            if (lo[m] <= q) a = m;
            else b = m;
        }
        return a;
    };
    const uint32_t p = n.pos_base + lp;
    const uint32_t lv = layer_of(lp);
    const uint32_t e1 = row_ptr[p + 1];
    uint32_t k = row_ptr[p];
    for (; k < e1; ++k) {
        const uint32_t src = edges[k].x;
        const uint32_t ls = src - n.pos_base < n.n_pos ? layer_of(src - n.pos_base) : 0u;
        if (ls + D >= lv) break;
    }
    split[p] = k;
}
