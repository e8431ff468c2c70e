// gather_bw.cu -- ceiling of the C4 access pattern on this GPU (tool, not product).
//
// Config 4's sweep is dominated by uniformly random 256-byte row gathers
// (64 fp32 batch columns per source position) out of a 2.56 GB activation
// array.  This measures what DRAM delivers for that pattern, independent of
// the engine's kernels, so the roofline fraction can be read against both the
// copy bandwidth (MEASURED_PEAKS.json) and the random-row ceiling.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw tools/gather_bw.cu
//   ./gather_bw [rows=10000000] [row_bytes=256] [gathers=400000000]
//
// Modes:
//   0  raw: each 16-lane group gathers 8 independent random rows per step,
//      sums them (no dependency chain), writes one row per 64 gathers;
//   1  same with ld.global.nc.L1::no_allocate;
//   2  k_level-like: group = node of degree 50, edges {src,w} read from an
//      edge array, 8 gathers in flight, in-order FADD chain, one row written.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

__device__ __forceinline__ float4 ld_na(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

template <int MODE, int U>
__global__ void __launch_bounds__(256, 4)
k_raw(const float4* __restrict__ A, uint32_t row_f4, const uint32_t* __restrict__ idx,
      uint64_t n_groups, uint32_t per_group, float4* __restrict__ out) {
    const uint32_t lanes = row_f4;  // one float4 per lane per row
    const uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / lanes;
    const uint32_t lane = threadIdx.x % lanes;
    if (g >= n_groups) return;
    const uint32_t* ix = idx + g * per_group;
    float4 acc = make_float4(0, 0, 0, 0);
    for (uint32_t k = 0; k < per_group; k += U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t s = __ldg(ix + k + u);
            const float4* p = A + static_cast<uint64_t>(s) * row_f4 + lane;
            v[u] = MODE == 1 ? ld_na(p) : __ldg(p);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
    }
    out[g * lanes + lane] = acc;
}

int main(int argc, char** argv) {
    const uint64_t rows = argc > 1 ? strtoull(argv[1], 0, 10) : 10000000ull;
    const uint32_t row_bytes = argc > 2 ? atoi(argv[2]) : 256;
    const uint64_t gathers = argc > 3 ? strtoull(argv[3], 0, 10) : 400000000ull;
    const uint32_t row_f4 = row_bytes / 16;
    const uint32_t per_group = 64;
    const uint64_t n_groups = gathers / per_group;
    float4* A;
    uint32_t* idx;
    float4* out;
    CK(cudaMalloc(&A, rows * row_bytes));
    CK(cudaMalloc(&idx, n_groups * per_group * 4));
    CK(cudaMalloc(&out, n_groups * row_bytes));
    CK(cudaMemset(A, 0, rows * row_bytes));
    {
        std::vector<uint32_t> h(n_groups * per_group);
        uint64_t s = 0x9E3779B97F4A7C15ull;
        for (auto& x : h) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            x = static_cast<uint32_t>(s % rows);
        }
        CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const uint64_t threads = n_groups * row_f4;
    const uint32_t blocks = static_cast<uint32_t>((threads + 255) / 256);
    auto run = [&](const char* name, auto kern) {
        for (int i = 0; i < 2; ++i) kern<<<blocks, 256>>>(A, row_f4, idx, n_groups, per_group, out);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        const int reps = 5;
        for (int i = 0; i < reps; ++i) kern<<<blocks, 256>>>(A, row_f4, idx, n_groups, per_group, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= reps;
        const double bytes = static_cast<double>(gathers) * (row_bytes + 4) + n_groups * row_bytes;
        const double row_only = static_cast<double>(gathers) * row_bytes;
        printf("{\"mode\": \"%s\", \"rows\": %llu, \"row_bytes\": %u, \"gathers\": %llu, \"ms\": %.3f, "
               "\"gbs_total\": %.1f, \"gbs_rows\": %.1f}\n",
               name, (unsigned long long)rows, row_bytes, (unsigned long long)gathers, ms,
               bytes / ms / 1e6, row_only / ms / 1e6);
    };
    run("raw_u8", k_raw<0, 8>);
    run("raw_u16", k_raw<0, 16>);
    run("raw_u4", k_raw<0, 4>);
    run("noalloc_u8", k_raw<1, 8>);
    run("noalloc_u16", k_raw<1, 16>);
    return 0;
}
