// serve.cuh -- K-serve: the batch-1 latency path.  One persistent CTA keeps a
// small network resident in shared memory (row pointers, edges with local
// source indices, activations) and answers activations through page-locked,
// mapped host memory.  No kernel launch, graph replay, copy or stream
// synchronisation per activation: on config 1 those fixed costs (~15 us)
// were most of the per-vector time (profiles/r1_bench_csv).
//
// Flagged 8-byte records in both directions (each value travels with the
// request's sequence number in one 8-byte store, which PCIe delivers whole):
//  * host -> device: in[0] = {n_vec | stop << 31, seq}, in[1 + k] = {x_k, seq}
//    for all max_vec x n_inputs slots; device threads poll their own record,
//    so the doorbell and the inputs cost one PCIe round trip together;
//  * device -> host: out[j] = {y_j, seq}; the host polls the records it
//    needs -- no system fence and no separate completion flag (a
//    __threadfence_system before a done flag cost ~3.4 us per request).
// The sweep is eval.cpp:64-77 (per layer, every row's in-order fp32 sum then
// sigmoid32, the layer barrier a __syncthreads) and read_outputs
// (eval.cpp:82-87).
// Included by kernels.cuh inside namespace asnn_b200.
#pragma once

// Device phase stamps of the last request (clock64 deltas; page-locked,
// mapped): inputs seen -> sensors -> layers -> outputs issued.
struct ServeCtl {
    long long t_sens, t_layers, t_out, t_wait, t_dbg0, t_dbg1, t_dbg2, t_dbg3;
};
constexpr uint32_t kServeStop = 1u << 31;

namespace serve {
__device__ __forceinline__ uint2 ld_rec(const uint2* p) {
    uint2 v;
    asm volatile("ld.relaxed.sys.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rec(uint2* p, uint32_t a, uint32_t b) {
    asm volatile("st.relaxed.sys.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}

// Shared-memory layout for a network of P positions (incl. sensors), E
// stored edges, S sensors, O outputs, L layers and ld columns.
__host__ __device__ inline uint32_t smem_bytes(uint32_t P, uint64_t E, uint32_t S, uint32_t O, uint32_t L,
                                               uint32_t ld) {
    uint64_t b = 8 * E                                   // edges {local src, w}
                 + 4ull * (P + 1) * ld                   // activations (+ zero row)
                 + 4ull * (P + 1) + 4ull * (L + 1)       // row pointers, layer offsets
                 + 4ull * (S + O) + 64;
    if (ld == 1) b += 8 * (E + 6ull * P) + 12ull * P + 32;  // batch-1 rows: padded edges, row info, partial sums
    return b > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(b);
}
}  // namespace serve

// One CTA, blockDim.x threads; ld = the largest batch a request may carry.
template <bool GUARD>
__global__ void __launch_bounds__(512)
k_serve(const CtaNet* __restrict__ nets, const uint32_t* __restrict__ lo_cat, const uint32_t* __restrict__ row_ptr,
        const uint2* __restrict__ edges, const uint4* __restrict__ sinfo, const uint4* __restrict__ oinfo,
        ServeCtl* ctl, const uint2* in_rec, uint2* out_rec, uint32_t ld) {
    extern __shared__ __align__(16) unsigned char sv_smem[];
    const CtaNet n = nets[0];
    const uint32_t P = n.n_pos, L = n.n_layers, S = n.n_sensors, O = n.n_out;
    const uint32_t e_base = row_ptr[n.pos_base];
    const uint32_t E = row_ptr[n.pos_base + P] - e_base;
    uint2* ed = reinterpret_cast<uint2*>(sv_smem);
    float* As = reinterpret_cast<float*>(ed + E);                 // [P + 1][ld], row P = zeros
    uint32_t* rp = reinterpret_cast<uint32_t*>(As + static_cast<size_t>(P + 1) * ld);  // [P + 1] local
    uint32_t* lo = rp + P + 1;                                    // [L + 1]
    uint32_t* sk = lo + L + 1;                                    // [S] input index of sensor s
    uint32_t* op = sk + S;                                        // [O] local position of output j
    // batch-1 rows (ld == 1), split like K-chain (chain.cuh) at depth 1: the
    // prefix (edges before the first source on layer l-1: sources final one
    // step early) and the rest, each padded to a multiple of 4 with {zero
    // row, 0.0} (+0.0f appended to a partial or final sum changes at most the
    // sign of a zero, which sigmoid32 ignores), as {shared address of the
    // source, weight}; row info {first padded edge, prefix batches | rest
    // batches << 16}; pre[r] the parked prefix sum
    uint2* ri = reinterpret_cast<uint2*>((reinterpret_cast<uintptr_t>(op + O) + 15) & ~uintptr_t(15));
    float* pre = reinterpret_cast<float*>(ri + (ld == 1 ? P : 0));
    uint2* e4 = reinterpret_cast<uint2*>((reinterpret_cast<uintptr_t>(pre + (ld == 1 ? P : 0)) + 15) & ~uintptr_t(15));
    __shared__ uint32_t sh_nvec;
    __shared__ uint32_t sh_scan[513];
    __shared__ float sh_x[512];                                   // this request's inputs
    __shared__ __align__(16) uint64_t sh_tab[64];                 // sigmoid32's 2^(i/32) table
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const uint32_t n_x = ld * n.n_in;  // input slots (<= 511, checked by the host)

    // ---- resident copy of the network (once) ----
    for (uint32_t k = tid; k < E; k += T) {
        const uint2 e = edges[e_base + k];
        const uint32_t p = e.x - n.pos_base;
        ed[k] = make_uint2(GUARD && p >= P ? P : p, e.y);
    }
    for (uint32_t i = tid; i <= P; i += T) rp[i] = row_ptr[n.pos_base + i] - e_base;
    for (uint32_t i = tid; i <= L; i += T) lo[i] = lo_cat[n.lo_base + i];
    for (uint32_t s = tid; s < S; s += T) sk[s] = sinfo[n.sens_prefix + s].w;
    for (uint32_t j = tid; j < O; j += T) {
        const uint32_t pos = oinfo[n.out_prefix + j].x;
        op[j] = pos == kUnassigned ? kUnassigned : pos - n.pos_base;
    }
    for (uint32_t c = tid; c < ld; c += T) As[static_cast<size_t>(P) * ld + c] = 0.0f;
    for (uint32_t i = tid; i < 64; i += T) sh_tab[i] = kExp32Tab[i];
    __syncthreads();
    const uint32_t as_sh = heavy::smem_u32(As);
    if (ld == 1) {
        // padded offsets: thread t scans rows [t*chunk, (t+1)*chunk), then a
        // serial scan of the T partial sums
        const uint32_t chunk = (P + T - 1) / T, r0 = min(P, tid * chunk), r1 = min(P, r0 + chunk);
        // split of row r: edges before the first source at or after lo[level(r) - 1]
        auto split_of = [&](uint32_t r) -> uint32_t {
            uint32_t a = 0, b = L;  // level: lo[a] <= r < lo[a + 1]
            while (b - a > 1) {
                const uint32_t m = (a + b) / 2;
                if (lo[m] <= r) a = m;
                else b = m;
            }
            const uint32_t thr = a >= 1 ? lo[a - 1] : 0u;
            uint32_t k = rp[r];
            while (k < rp[r + 1] && ed[k].x < thr) ++k;
            return k - rp[r];
        };
        uint32_t sum = 0;
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t sp = split_of(r), deg = rp[r + 1] - rp[r];
            sum += ((sp + 3) & ~3u) + ((deg - sp + 3) & ~3u);
        }
        sh_scan[tid] = sum;
        __syncthreads();
        if (tid == 0) {
            uint32_t acc = 0;
            for (uint32_t t = 0; t < T; ++t) {
                const uint32_t v = sh_scan[t];
                sh_scan[t] = acc;
                acc += v;
            }
        }
        __syncthreads();
        uint32_t at = sh_scan[tid];
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t k0 = rp[r], deg = rp[r + 1] - k0, sp = split_of(r);
            const uint32_t pp = (sp + 3) & ~3u, fp = (deg - sp + 3) & ~3u;
            ri[r] = make_uint2(at, pp / 4 | (fp / 4) << 16);
            pre[r] = 0.0f;
            for (uint32_t j = 0; j < pp; ++j)
                e4[at + j] = j < sp ? make_uint2(as_sh + 4 * ed[k0 + j].x, ed[k0 + j].y) : make_uint2(as_sh + 4 * P, 0u);
            for (uint32_t j = 0; j < fp; ++j)
                e4[at + pp + j] = sp + j < deg ? make_uint2(as_sh + 4 * ed[k0 + sp + j].x, ed[k0 + sp + j].y)
                                               : make_uint2(as_sh + 4 * P, 0u);
            at += pp + fp;
        }
        __syncthreads();
    }
    const chain::ExpTabShared tab{heavy::smem_u32(sh_tab)};

    uint32_t last = 0;
    for (;;) {
        // every thread polls its own input record (thread n_x the header);
        // the host bumps seq by one per request
        const uint32_t want = last + 1;
        const long long cw = clock64();
        for (uint32_t k = tid; k <= n_x; k += T) {
            uint2 r;
            do {
                r = serve::ld_rec(in_rec + (k == n_x ? 0 : 1 + k));
            } while (r.y != want);
            if (k == n_x) sh_nvec = r.x;
            else sh_x[k] = __uint_as_float(r.x);
        }
        __syncthreads();
        const uint32_t hdr = sh_nvec;
        if (hdr & kServeStop) break;
        last = want;
        const uint32_t nv = min(hdr, ld);
        const long long c0 = clock64();
        // sensors: eval.cpp:17 (sigmoided inputs), x = [vector][input] in host memory
        for (uint32_t i = tid; i < S * nv; i += T) {
            const uint32_t c = i / S, s = i - c * S;
            const uint32_t k = sk[s];
            const float xv = k != kUnassigned ? sh_x[c * n.n_in + k] : 0.0f;
            As[static_cast<size_t>(s) * ld + c] = sigmoid32(xv, tab);
        }
        __syncthreads();
        const long long c1 = clock64();
        if (ld == 1) {
            // step l: the first half of the threads finishes layer l from its
            // parked prefix sums, the second half sums layer l+1's prefixes
            // (sources final since step l-1); one barrier per step
            const uint32_t Th = T / 2;
            auto run = [&](float acc, const uint4* q, uint32_t nb) -> float {
#pragma unroll 4
                for (uint32_t bt = 0; bt < nb; ++bt) {
                    const uint4 p0 = q[2 * bt], p1 = q[2 * bt + 1];  // 4 x {source address, weight}
                    const float v0 = chain::lds_f32(p0.x), v1 = chain::lds_f32(p0.z);
                    const float v2 = chain::lds_f32(p1.x), v3 = chain::lds_f32(p1.z);
                    acc = mac(acc, __uint_as_float(p0.y), v0);
                    acc = mac(acc, __uint_as_float(p0.w), v1);
                    acc = mac(acc, __uint_as_float(p1.y), v2);
                    acc = mac(acc, __uint_as_float(p1.w), v3);
                }
                return acc;
            };
            for (uint32_t l = 1; l < L; ++l) {
                if (tid < Th) {
                    for (uint32_t r = lo[l] + tid; r < lo[l + 1]; r += Th) {
                        const uint2 info = ri[r];
                        const uint4* q = reinterpret_cast<const uint4*>(e4 + info.x) + 2 * (info.y & 0xFFFFu);
                        const float acc = run(pre[r], q, info.y >> 16);
                        chain::sts_f32(as_sh + 4 * r, sigmoid32(acc, tab));
                    }
                } else if (l + 1 < L) {
                    for (uint32_t r = lo[l + 1] + tid - Th; r < lo[l + 2]; r += Th) {
                        const uint2 info = ri[r];
                        pre[r] = run(0.0f, reinterpret_cast<const uint4*>(e4 + info.x), info.y & 0xFFFFu);
                    }
                }
                __syncthreads();
            }
        } else
        for (uint32_t l = 1; l < L; ++l) {
            const uint32_t a = lo[l], items = (lo[l + 1] - a) * nv;
            const long long d0 = clock64();
#ifdef ASNN_SERVE_TWICE
            for (int rep = 0; rep < 2; ++rep) {
            if (rep == 1) ctl->t_dbg3 = clock64() - d0;
#endif
#ifdef ASNN_SERVE_CAL
            if (tid == 0) {
                float f = __int_as_float(sh_nvec);
                const long long q0 = clock64();
#pragma unroll 1
                for (int u = 0; u < 100; ++u) f = __fadd_rn(f, 1e-7f);
                const long long q1 = clock64();
#pragma unroll
                for (int u = 0; u < 100; ++u) f = __fadd_rn(f, 1e-7f);
                const long long q2 = clock64();
                const uint32_t pp = f > 1e30f ? 1u : 0u;
                ctl->t_dbg3 = (q1 - q0) * 100000 + (q2 - q1) + (pp == 12345 ? 1 : 0);
            }
#endif
            for (uint32_t it = tid; it < items; it += T) {
                const uint32_t i = a + it / nv, c = it % nv;
                uint32_t k = rp[i];
                const uint32_t ke = rp[i + 1];
                float acc = 0.0f;
                // four edges' loads in flight, then their adds in stored order
                for (; k + 4 <= ke; k += 4) {
                    uint2 e[4];
                    float v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) e[u] = ed[k + u];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = As[static_cast<size_t>(e[u].x) * ld + c];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc = mac(acc, __uint_as_float(e[u].y), v[u]);
                }
                for (; k < ke; ++k) {
                    const uint2 e = ed[k];
                    acc = mac(acc, __uint_as_float(e.y), As[static_cast<size_t>(e.x) * ld + c]);
                }
#ifdef ASNN_SERVE_NOSIG
                As[static_cast<size_t>(i) * ld + c] = acc * 0.001f;
#else
                As[static_cast<size_t>(i) * ld + c] = sigmoid32(acc, tab);
#endif
            }
#ifdef ASNN_SERVE_TWICE
            }
#endif
            const long long d1 = clock64();
            __syncthreads();
            if (l == 3 && tid == 0) {
                ctl->t_dbg0 = d1 - d0, ctl->t_dbg1 = clock64() - d1, ctl->t_dbg2 = items;
#ifndef ASNN_SERVE_TWICE
                ctl->t_dbg3 = rp[a + 1] - rp[a];
#endif
            }
        }
        const long long c2 = clock64();
        // read_outputs (eval.cpp:82-87): flagged records [vector][output]
        for (uint32_t i = tid; i < O * nv; i += T) {
            const uint32_t c = i / O, j = i - c * O;
            const uint32_t p = op[j];
            const float y = p != kUnassigned ? As[static_cast<size_t>(p) * ld + c] : 0.0f;
            serve::st_rec(out_rec + i, __float_as_uint(y), last);
        }
        if (tid == 0) {
            const long long c3 = clock64();
            ctl->t_wait = c0 - cw, ctl->t_sens = c1 - c0, ctl->t_layers = c2 - c1, ctl->t_out = c3 - c2;
        }
    }
}
