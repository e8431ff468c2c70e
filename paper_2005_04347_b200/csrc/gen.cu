// gen.cu -- the bench corpora generated on the device.
//
// The reference's generate() (netgen.cpp:71-157) keeps a hash set of every
// pair and draws sequentially -- infeasible at 500M edges (netgen.cpp:87-88).
// The bench shapes (config 2's pruned MLP, config 4's banded power law) are
// counter-based instead: every node draws from its own SplitMix64 stream
// (gen_core.h), so one GPU thread per node reproduces the host generators
// (netgen.cpp) byte for byte, and the network never has to cross the host
// link: asnn_dev_gen_*_layout hand the device arrays straight to
// compute_required / segment / flatten (config 4: 495M edges generated and
// levelled in HBM instead of ~5 s of host generation + a 6 GB upload).
//
// Power law on the device:
//   1. mandatory successors (pl_succ) per non-output node; counting sort of
//      them by target (order inside a target is irrelevant: lists are sorted);
//   2. per target: raw source count (its successor-pickers + pl_draw's
//      emissions), exclusive scan, then the raw (source, target) pairs;
//   3. stable radix sort by source, then by target -> target-major, sources
//      ascending; adjacent duplicates dropped (the host's sort + unique);
//   4. per target: replay the source draws to reach the weight stream, then
//      one U[-1, 1] weight per kept source.
#include <cstring>
#include <vector>

#include "corpus.hpp"
#include "engine.hpp"
#include "gen_core.h"
#include "sort.cuh"

using namespace asnn_b200;

#define CKG(expr)                                                \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return cuda_fail(dev, _e, #expr); \
    } while (0)
#define RCG(expr)                 \
    do {                          \
        int _rc = (expr);         \
        if (_rc) return _rc;      \
    } while (0)

namespace {

constexpr uint32_t kGenThreads = 256;
inline uint32_t gblocks(uint64_t n) { return static_cast<uint32_t>((n + kGenThreads - 1) / kGenThreads); }

// ---- config 2 ------------------------------------------------------------------------
__global__ void k_mlp_count(uint64_t seed, uint32_t width, double p, uint32_t n, uint32_t* cnt) {
    const uint64_t t = width + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    cnt[t - width] = asnn_gen::mlp_draw(seed, width, p, static_cast<uint32_t>(t), [](uint32_t, float) {});
}

__global__ void k_mlp_fill(uint64_t seed, uint32_t width, double p, uint32_t n, const uint32_t* off,
                           uint32_t* src, uint32_t* dst, float* w) {
    const uint64_t t = width + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint32_t k = off[t - width];
    asnn_gen::mlp_draw(seed, width, p, static_cast<uint32_t>(t), [&](uint32_t s, float x) {
        src[k] = s;
        dst[k] = static_cast<uint32_t>(t);
        w[k] = x;
        ++k;
    });
}

// ---- config 4 ------------------------------------------------------------------------
__global__ void k_pl_succ(asnn_gen::PowerlawSpec spec, uint32_t n_src, uint32_t* succ, uint32_t* cnt) {
    const uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n_src) return;
    const uint32_t t = asnn_gen::pl_succ(spec, static_cast<uint32_t>(v));
    succ[v] = t;
    atomicAdd(&cnt[t], 1u);
}

__global__ void k_pl_succ_fill(uint32_t n_src, const uint32_t* succ, const uint32_t* off, uint32_t* cur,
                               uint32_t* pickers) {
    const uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n_src) return;
    const uint32_t t = succ[v];
    pickers[off[t] + atomicAdd(&cur[t], 1u)] = static_cast<uint32_t>(v);
}

// raw[t - first] = successor-pickers of t + pl_draw's emissions
__global__ void k_pl_count(asnn_gen::PowerlawSpec spec, uint32_t first, uint32_t n, const uint32_t* pcnt,
                           uint32_t* raw) {
    const uint64_t t = first + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint32_t c = pcnt[t];
    asnn_gen::pl_draw(spec, static_cast<uint32_t>(t), [&](uint32_t) { ++c; });
    raw[t - first] = c;
}

__global__ void k_pl_fill(asnn_gen::PowerlawSpec spec, uint32_t first, uint32_t n, const uint32_t* poff,
                          const uint32_t* pcnt, const uint32_t* pickers, const uint32_t* roff, uint32_t* src,
                          uint32_t* tgt) {
    const uint64_t t = first + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint32_t k = roff[t - first];
    for (uint32_t i = 0; i < pcnt[t]; ++i, ++k) {
        src[k] = pickers[poff[t] + i];
        tgt[k] = static_cast<uint32_t>(t);
    }
    asnn_gen::pl_draw(spec, static_cast<uint32_t>(t), [&](uint32_t s) {
        src[k] = s;
        tgt[k] = static_cast<uint32_t>(t);
        ++k;
    });
}

// keep[i] = first of a run of equal (target, source) pairs; per-target counts
__global__ void k_pl_mark(const uint32_t* tgt, const uint32_t* src, uint64_t n, uint32_t* keep, uint32_t* ucnt) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool k = i == 0 || tgt[i] != tgt[i - 1] || src[i] != src[i - 1];
    keep[i] = k;
    if (k) atomicAdd(&ucnt[tgt[i]], 1u);
}

__global__ void k_pl_compact(const uint32_t* tgt, const uint32_t* src, const uint32_t* keep, const uint32_t* pos,
                             uint64_t n, uint32_t* out_src, uint32_t* out_dst) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || !keep[i]) return;
    out_src[pos[i]] = src[i];
    out_dst[pos[i]] = tgt[i];
}

__global__ void k_pl_weights(asnn_gen::PowerlawSpec spec, uint32_t first, uint32_t n, const uint32_t* row,
                             const uint32_t* ucnt, float* w) {
    const uint64_t t = first + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    asnn_gen::Rng r = asnn_gen::pl_draw(spec, static_cast<uint32_t>(t), [](uint32_t) {});
    const uint32_t b = row[t];
    for (uint32_t i = 0; i < ucnt[t]; ++i) w[b + i] = r.uniform(-1.0f, 1.0f);
}

__global__ void k_iota(uint32_t* a, uint32_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) a[i] = static_cast<uint32_t>(i);
}

int bits_for(uint32_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

// A generated network resident on the device.
struct DevCorpus {
    DevBuf<uint32_t> nodes, src, dst;
    DevBuf<float> w;
    uint32_t N = 0;
    uint64_t E = 0;
    std::vector<uint32_t> inputs, outputs;
};

int gen_mlp(asnn_dev* dev, uint32_t layers, uint32_t width, double p, uint64_t seed, DevCorpus& c) {
    if (layers < 2 || width == 0 || !(p > 0.0 && p <= 1.0)) return fail(dev, ASNN_E_INVALID, "bad mlp spec");
    cudaStream_t st = dev->stream;
    const uint64_t n64 = static_cast<uint64_t>(layers) * width;
    if (n64 >= 0xFFFFFFFFull) return fail(dev, ASNN_E_INVALID, "too many nodes");
    const uint32_t n = static_cast<uint32_t>(n64), targets = n - width;
    DevBuf<uint32_t> cnt, off, total;
    CKG(cnt.alloc(targets));
    CKG(off.alloc(targets + 1));
    CKG(total.alloc(1));
    k_mlp_count<<<gblocks(targets), kGenThreads, 0, st>>>(seed, width, p, n, cnt.p);
    RCG(exclusive_scan(dev, cnt.p, off.p, targets, total.p, st));
    uint32_t E = 0;
    CKG(cudaMemcpyAsync(&E, total.p, 4, cudaMemcpyDeviceToHost, st));
    CKG(cudaStreamSynchronize(st));
    c.N = n;
    c.E = E;
    CKG(c.nodes.alloc(n));
    CKG(c.src.alloc(E));
    CKG(c.dst.alloc(E));
    CKG(c.w.alloc(E));
    k_iota<<<gblocks(n), kGenThreads, 0, st>>>(c.nodes.p, n);
    k_mlp_fill<<<gblocks(targets), kGenThreads, 0, st>>>(seed, width, p, n, off.p, c.src.p, c.dst.p, c.w.p);
    CKG(cudaGetLastError());
    for (uint32_t i = 0; i < width; ++i) c.inputs.push_back(i);
    for (uint32_t i = 0; i < width; ++i) c.outputs.push_back((layers - 1) * width + i);
    return ASNN_OK;
}

int gen_powerlaw(asnn_dev* dev, uint32_t n_nodes, uint32_t bands, uint32_t n_in, uint32_t n_out,
                 uint64_t target_edges, double alpha, uint64_t seed, DevCorpus& c) {
    if (bands < 3 || n_in == 0 || n_out == 0 || !(alpha > 1.0) || n_nodes < n_in + n_out + (bands - 2))
        return fail(dev, ASNN_E_INVALID, "bad power-law spec");
    cudaStream_t st = dev->stream;
    const std::vector<uint32_t> starts = powerlaw_band_starts(n_nodes, bands, n_in, n_out);
    DevBuf<uint32_t> d_starts;
    CKG(d_starts.alloc(starts.size()));
    CKG(cudaMemcpyAsync(d_starts.p, starts.data(), starts.size() * 4, cudaMemcpyHostToDevice, st));
    const asnn_gen::PowerlawSpec spec{d_starts.p, bands, powerlaw_xm(n_nodes, n_in, n_out, target_edges, alpha),
                                      alpha, seed};
    const uint32_t n_src = starts[bands - 1], first = n_in, targets = n_nodes - first;

    // 1. mandatory successors, grouped by target
    DevBuf<uint32_t> succ, pcnt, poff, cur, pickers, total;
    CKG(succ.alloc(n_src));
    CKG(pcnt.alloc(n_nodes + 1));
    CKG(poff.alloc(n_nodes + 1));
    CKG(cur.alloc(n_nodes));
    CKG(total.alloc(1));
    CKG(cudaMemsetAsync(pcnt.p, 0, (n_nodes + 1) * 4ull, st));
    CKG(cudaMemsetAsync(cur.p, 0, n_nodes * 4ull, st));
    k_pl_succ<<<gblocks(n_src), kGenThreads, 0, st>>>(spec, n_src, succ.p, pcnt.p);
    RCG(exclusive_scan(dev, pcnt.p, poff.p, n_nodes, total.p, st));
    CKG(pickers.alloc(n_src));
    k_pl_succ_fill<<<gblocks(n_src), kGenThreads, 0, st>>>(n_src, succ.p, poff.p, cur.p, pickers.p);
    succ.reset();
    cur.reset();

    // 2. raw (source, target) pairs
    DevBuf<uint32_t> raw, roff;
    CKG(raw.alloc(targets));
    CKG(roff.alloc(targets + 1));
    k_pl_count<<<gblocks(targets), kGenThreads, 0, st>>>(spec, first, n_nodes, pcnt.p, raw.p);
    RCG(exclusive_scan(dev, raw.p, roff.p, targets, total.p, st));
    uint32_t R = 0;
    CKG(cudaMemcpyAsync(&R, total.p, 4, cudaMemcpyDeviceToHost, st));
    CKG(cudaStreamSynchronize(st));
    DevBuf<uint32_t> rsrc, rtgt;
    CKG(rsrc.alloc(R + 1));
    CKG(rtgt.alloc(R + 1));
    k_pl_fill<<<gblocks(targets), kGenThreads, 0, st>>>(spec, first, n_nodes, poff.p, pcnt.p, pickers.p, roff.p,
                                                        rsrc.p, rtgt.p);
    CKG(cudaGetLastError());
    pickers.reset();
    raw.reset();
    roff.reset();

    // 3. target-major, sources ascending, duplicates dropped
    const int bits = bits_for(n_nodes);
    SortBuffers sb;
    uint32_t *k1, *v1;
    RCG(radix_sort_pairs(dev, rsrc.p, rtgt.p, R, bits, sb, &k1, &v1, st));  // by source
    uint32_t *k2, *v2;
    SortBuffers sb2;  // v1 / k1 may live in sb's alternates
    RCG(radix_sort_pairs(dev, v1, k1, R, bits, sb2, &k2, &v2, st));         // stably by target
    DevBuf<uint32_t> keep, kpos, ucnt;
    CKG(keep.alloc(R + 1));
    CKG(kpos.alloc(R + 1));
    CKG(ucnt.alloc(n_nodes + 1));
    CKG(cudaMemsetAsync(ucnt.p, 0, (n_nodes + 1) * 4ull, st));
    k_pl_mark<<<gblocks(R), kGenThreads, 0, st>>>(k2, v2, R, keep.p, ucnt.p);
    RCG(exclusive_scan(dev, keep.p, kpos.p, R, total.p, st));
    uint32_t E = 0;
    CKG(cudaMemcpyAsync(&E, total.p, 4, cudaMemcpyDeviceToHost, st));
    CKG(cudaStreamSynchronize(st));
    CKG(c.src.alloc(E + 1));
    CKG(c.dst.alloc(E + 1));
    k_pl_compact<<<gblocks(R), kGenThreads, 0, st>>>(k2, v2, keep.p, kpos.p, R, c.src.p, c.dst.p);
    CKG(cudaGetLastError());
    keep.reset();
    kpos.reset();
    rsrc.reset();
    rtgt.reset();
    sb.k_alt.reset();
    sb.v_alt.reset();
    sb2.k_alt.reset();
    sb2.v_alt.reset();

    // 4. weights: each target's stream after its source draws
    DevBuf<uint32_t> row;
    CKG(row.alloc(n_nodes + 1));
    RCG(exclusive_scan(dev, ucnt.p, row.p, n_nodes, total.p, st));
    CKG(c.w.alloc(E + 1));
    k_pl_weights<<<gblocks(targets), kGenThreads, 0, st>>>(spec, first, n_nodes, row.p, ucnt.p, c.w.p);
    CKG(c.nodes.alloc(n_nodes));
    k_iota<<<gblocks(n_nodes), kGenThreads, 0, st>>>(c.nodes.p, n_nodes);
    CKG(cudaGetLastError());
    CKG(cudaStreamSynchronize(st));  // d_starts / ucnt / row are freed on return
    c.N = n_nodes;
    c.E = E;
    for (uint32_t i = 0; i < n_in; ++i) c.inputs.push_back(i);
    for (uint32_t i = 0; i < n_out; ++i) c.outputs.push_back(starts[bands - 1] + i);
    return ASNN_OK;
}

int to_host(asnn_dev* dev, DevCorpus& c, asnn_corpus** out) {
    auto* h = new asnn_corpus;
    h->nodes.resize(c.N);
    h->src.resize(c.E);
    h->dst.resize(c.E);
    h->w.resize(c.E);
    h->inputs = c.inputs;
    h->outputs = c.outputs;
    cudaError_t e = cudaSuccess;
    if (c.N) e = download_host(dev, h->nodes.data(), c.nodes.p, c.N * 4ull, dev->stream);
    if (e == cudaSuccess && c.E) e = download_host(dev, h->src.data(), c.src.p, c.E * 4, dev->stream);
    if (e == cudaSuccess && c.E) e = download_host(dev, h->dst.data(), c.dst.p, c.E * 4, dev->stream);
    if (e == cudaSuccess && c.E) e = download_host(dev, h->w.data(), c.w.p, c.E * 4, dev->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(dev->stream);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(dev, e, "generator download");
    }
    *out = h;
    return ASNN_OK;
}

int to_layout(asnn_dev* dev, DevCorpus& c, asnn_dev_layout** out) {
    return build_device_network(dev, std::move(c.nodes), c.N, std::move(c.src), std::move(c.dst), std::move(c.w), c.E,
                                std::move(c.inputs), std::move(c.outputs), out);
}

struct Guard {
    std::lock_guard<std::recursive_mutex> lk;
    AllocStream on;
    explicit Guard(asnn_dev* d) : lk(d->mu), on(d->stream) {}
};

}  // namespace

extern "C" {

int asnn_dev_gen_mlp(asnn_dev* dev, uint32_t layers, uint32_t width, double p, uint64_t seed, asnn_corpus** out) {
    if (!dev || !out) return ASNN_E_INVALID;
    Guard g(dev);
    *out = nullptr;
    CKG(cudaSetDevice(dev->device));
    DevCorpus c;
    RCG(gen_mlp(dev, layers, width, p, seed, c));
    return to_host(dev, c, out);
}

int asnn_dev_gen_mlp_layout(asnn_dev* dev, uint32_t layers, uint32_t width, double p, uint64_t seed,
                            asnn_dev_layout** out) {
    if (!dev || !out) return ASNN_E_INVALID;
    Guard g(dev);
    *out = nullptr;
    CKG(cudaSetDevice(dev->device));
    DevCorpus c;
    RCG(gen_mlp(dev, layers, width, p, seed, c));
    return to_layout(dev, c, out);
}

int asnn_dev_gen_powerlaw(asnn_dev* dev, uint32_t n_nodes, uint32_t bands, uint32_t n_in, uint32_t n_out,
                          uint64_t target_edges, double alpha, uint64_t seed, asnn_corpus** out) {
    if (!dev || !out) return ASNN_E_INVALID;
    Guard g(dev);
    *out = nullptr;
    CKG(cudaSetDevice(dev->device));
    DevCorpus c;
    RCG(gen_powerlaw(dev, n_nodes, bands, n_in, n_out, target_edges, alpha, seed, c));
    return to_host(dev, c, out);
}

int asnn_dev_gen_powerlaw_layout(asnn_dev* dev, uint32_t n_nodes, uint32_t bands, uint32_t n_in, uint32_t n_out,
                                 uint64_t target_edges, double alpha, uint64_t seed, asnn_dev_layout** out) {
    if (!dev || !out) return ASNN_E_INVALID;
    Guard g(dev);
    *out = nullptr;
    CKG(cudaSetDevice(dev->device));
    DevCorpus c;
    RCG(gen_powerlaw(dev, n_nodes, bands, n_in, n_out, target_edges, alpha, seed, c));
    return to_layout(dev, c, out);
}

}  // extern "C"
