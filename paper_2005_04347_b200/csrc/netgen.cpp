// netgen.cpp -- deterministic synthetic ASNN corpora (host C++, not on the
// activation path).
//
//  * asnn_gen_reference: the reference's seeded generator restated so that
//    the same GenSpec gives a byte-identical network without the reference
//    checkout (netgen.cpp:21-157 of /root/reference/proj/src); pinned by
//    tests/test_corpus.py against oracle/_ref's asnn::generate.
//  * asnn_gen_mlp: config 2's "pruned MLP" shape.
//  * asnn_gen_powerlaw: config 4's banded power-law shape,
//    counter-based per node so it is identical for any thread count.
//
// Floating point here must match the reference's x86-64 build: no FMA
// contraction (compiled with -ffp-contract=off, no -march).
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <unordered_set>
#include <vector>

#include "asnn_dev.h"
#include "gen_core.h"

namespace {

// SplitMix64 (Vigna), the state transition of rng.hpp:10-38: same seed, same
// stream, on any platform.
struct SplitMix64 {
    std::uint64_t s;
    explicit SplitMix64(std::uint64_t seed) : s(seed) {}
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    std::uint64_t bounded(std::uint64_t n) {  // rejection sampling, unbiased
        const std::uint64_t threshold = (0 - n) % n;
        for (;;) {
            const std::uint64_t r = next();
            if (r >= threshold) return r % n;
        }
    }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    float uniform(float lo, float hi) {
        return static_cast<float>(lo + uniform01() * (static_cast<double>(hi) - lo));
    }
};

}  // namespace

#include "corpus.hpp"

namespace {

std::vector<std::uint32_t> band_starts(std::uint32_t in, std::uint32_t out, std::uint32_t hidden,
                                       std::uint32_t depth) {
    std::vector<std::uint32_t> starts{0, in};
    if (depth > 2) {
        const std::uint32_t bands = depth - 2;
        const std::uint32_t base = hidden / bands, rem = hidden % bands;
        for (std::uint32_t b = 0; b < bands; ++b) starts.push_back(starts.back() + base + (b < rem));
    }
    starts.push_back(starts.back() + out);
    return starts;
}

std::uint64_t capacity_of(const std::vector<std::uint32_t>& starts) {
    std::uint64_t cap = 0;
    for (std::size_t b = 1; b + 1 < starts.size(); ++b)
        cap += static_cast<std::uint64_t>(starts[b + 1] - starts[b]) * starts[b];
    return cap;
}

}  // namespace

// Pareto scale of config 4's extra-source count: expected mandatory edges are
// one predecessor per non-input plus one successor per non-output, the rest
// comes from the Pareto(alpha) draws (mean = xm * alpha / (alpha - 1)).
// Shared with gen.cu.
double powerlaw_xm(uint32_t n_nodes, uint32_t n_in, uint32_t n_out, uint64_t target_edges, double alpha) {
    const std::uint64_t non_inputs = n_nodes - n_in;
    const double mandatory = static_cast<double>(non_inputs) + (n_nodes - n_out);
    const double extra_mean = std::max(0.0, (static_cast<double>(target_edges) - mandatory) /
                                                 static_cast<double>(non_inputs));
    return extra_mean * (alpha - 1.0) / alpha;
}

std::vector<std::uint32_t> powerlaw_band_starts(uint32_t n_nodes, uint32_t bands, uint32_t n_in, uint32_t n_out) {
    return band_starts(n_in, n_out, n_nodes - n_in - n_out, bands);
}

namespace {

inline std::uint64_t pair_key(std::uint32_t s, std::uint32_t t) {
    return (static_cast<std::uint64_t>(s) << 32) | t;
}

}  // namespace

extern "C" {

uint64_t asnn_gen_max_connections(uint32_t in, uint32_t out, uint32_t hidden, uint32_t depth) {
    return capacity_of(band_starts(in, out, hidden, depth));
}

// Restates generate() (netgen.cpp:71-157): band layout, one mandatory
// predecessor from the adjacent band, then uniform unused forward pairs
// (dense: shuffled prefix of the free pairs; sparse: rejection sampling),
// finally sorted by (source, target).  The draw order of the SplitMix64
// stream is the reference's, so networks are byte-identical.
int asnn_gen_reference(uint32_t in, uint32_t out, uint32_t hidden, uint64_t conn, uint32_t depth,
                       float wmin, float wmax, uint64_t seed, asnn_corpus** result) {
    if (!result) return ASNN_E_INVALID;
    *result = nullptr;
    // check_feasible (netgen.cpp:29-53)
    if (in == 0 || out == 0 || depth < 2 || (depth == 2 && hidden > 0) ||
        (depth > 2 && hidden < depth - 2) || !(wmin <= wmax))
        return ASNN_E_INFEASIBLE;
    const auto starts = band_starts(in, out, hidden, depth);
    if (conn < static_cast<std::uint64_t>(hidden) + out || conn > capacity_of(starts))
        return ASNN_E_INFEASIBLE;

    auto* c = new asnn_corpus;
    const std::uint32_t node_count = starts.back();
    const std::uint32_t first = in;
    SplitMix64 rng(seed);
    auto band_of = [&starts](std::uint32_t id) {
        return static_cast<std::uint32_t>(std::upper_bound(starts.begin(), starts.end(), id) -
                                          starts.begin()) - 1;
    };
    std::vector<std::uint64_t> keys;  // (src << 32 | dst), weight kept alongside
    std::vector<float> weights;
    keys.reserve(conn);
    weights.reserve(conn);
    std::unordered_set<std::uint64_t> used;
    used.reserve(conn * 2);

    // netgen.cpp:95-102 -- mandatory predecessor from the adjacent band.
    for (std::uint32_t node = first; node < node_count; ++node) {
        const std::uint32_t band = band_of(node);
        const std::uint32_t lo = starts[band - 1], hi = starts[band];
        const std::uint32_t pred = lo + static_cast<std::uint32_t>(rng.bounded(hi - lo));
        used.insert(pair_key(pred, node));
        keys.push_back(pair_key(pred, node));
        weights.push_back(rng.uniform(wmin, wmax));
    }
    // netgen.cpp:104-113 -- cumulative forward-pair space per target.
    const std::uint64_t remaining = conn - keys.size();
    std::vector<std::uint64_t> cumulative(node_count - first + 1, 0);
    for (std::uint32_t node = first; node < node_count; ++node)
        cumulative[node - first + 1] = cumulative[node - first] + starts[band_of(node)];
    const std::uint64_t pair_space = cumulative.back();

    if (remaining * 2 > pair_space - keys.size()) {
        // netgen.cpp:115-128 -- dense: shuffle a prefix of the free pairs.
        std::vector<std::uint64_t> free_pairs;
        free_pairs.reserve(pair_space - keys.size());
        for (std::uint32_t node = first; node < node_count; ++node)
            for (std::uint32_t pred = 0; pred < starts[band_of(node)]; ++pred)
                if (!used.count(pair_key(pred, node))) free_pairs.push_back(pair_key(pred, node));
        for (std::uint64_t k = 0; k < remaining; ++k) {
            const std::uint64_t j = k + rng.bounded(free_pairs.size() - k);
            std::swap(free_pairs[k], free_pairs[j]);
            keys.push_back(free_pairs[k]);
            weights.push_back(rng.uniform(wmin, wmax));
        }
    } else {
        // netgen.cpp:129-141 -- sparse: rejection-sample the pair space.
        for (std::uint64_t k = 0; k < remaining;) {
            const std::uint64_t idx = rng.bounded(pair_space);
            const auto it = std::upper_bound(cumulative.begin(), cumulative.end(), idx);
            const std::uint32_t slot = static_cast<std::uint32_t>(it - cumulative.begin()) - 1;
            const std::uint32_t node = first + slot;
            const std::uint32_t pred = static_cast<std::uint32_t>(idx - cumulative[slot]);
            if (!used.insert(pair_key(pred, node)).second) continue;
            keys.push_back(pair_key(pred, node));
            weights.push_back(rng.uniform(wmin, wmax));
            ++k;
        }
    }
    // netgen.cpp:143-145 -- sort by (source, target); keys are unique.
    std::vector<std::uint32_t> order(keys.size());
    for (std::uint32_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(),
              [&keys](std::uint32_t a, std::uint32_t b) { return keys[a] < keys[b]; });
    c->src.resize(keys.size());
    c->dst.resize(keys.size());
    c->w.resize(keys.size());
    for (std::size_t i = 0; i < order.size(); ++i) {
        c->src[i] = static_cast<std::uint32_t>(keys[order[i]] >> 32);
        c->dst[i] = static_cast<std::uint32_t>(keys[order[i]] & 0xFFFFFFFFu);
        c->w[i] = weights[order[i]];
    }
    // netgen.cpp:147-156 -- dense ids, inputs = band 0, outputs = last band.
    c->nodes.resize(node_count);
    for (std::uint32_t i = 0; i < node_count; ++i) c->nodes[i] = i;
    c->inputs.resize(in);
    for (std::uint32_t i = 0; i < in; ++i) c->inputs[i] = i;
    c->outputs.resize(out);
    for (std::uint32_t i = 0; i < out; ++i) c->outputs[i] = starts[depth - 1] + i;
    *result = c;
    return ASNN_OK;
}

// Config 2: `layers` layers of `width` nodes, ids layer-major.
// Layer 0 = inputs, last layer = outputs; every node of layer l >= 1 links to
// each node of layer l-1 independently with probability p (at least one),
// weights U[-1, 1] (gen_core.h mlp_draw: one counter-seeded stream per
// target, so the device generator in gen.cu reproduces it byte for byte).
// Edges come out target-major, sources ascending.
int asnn_gen_mlp(uint32_t layers, uint32_t width, double p, uint64_t seed, asnn_corpus** result) {
    if (!result || layers < 2 || width == 0 || !(p > 0.0 && p <= 1.0)) return ASNN_E_INVALID;
    auto* c = new asnn_corpus;
    const std::uint32_t n = layers * width;
    c->nodes.resize(n);
    for (std::uint32_t i = 0; i < n; ++i) c->nodes[i] = i;
    for (std::uint32_t i = 0; i < width; ++i) c->inputs.push_back(i);
    for (std::uint32_t i = 0; i < width; ++i) c->outputs.push_back((layers - 1) * width + i);
    std::vector<std::uint64_t> row(n + 1, 0);
#pragma omp parallel for schedule(static)
    for (std::int64_t t = width; t < static_cast<std::int64_t>(n); ++t)
        row[t + 1] = asnn_gen::mlp_draw(seed, width, p, static_cast<std::uint32_t>(t), [](std::uint32_t, float) {});
    for (std::uint32_t t = 0; t < n; ++t) row[t + 1] += row[t];
    const std::uint64_t E = row[n];
    c->src.resize(E);
    c->dst.resize(E);
    c->w.resize(E);
#pragma omp parallel for schedule(static)
    for (std::int64_t t = width; t < static_cast<std::int64_t>(n); ++t) {
        std::uint64_t k = row[t];
        asnn_gen::mlp_draw(seed, width, p, static_cast<std::uint32_t>(t), [&](std::uint32_t s, float w) {
            c->src[k] = s;
            c->dst[k] = static_cast<std::uint32_t>(t);
            c->w[k] = w;
            ++k;
        });
    }
    *result = c;
    return ASNN_OK;
}

// Config 4: n_nodes ids in `bands` bands (band 0 = n_inputs
// inputs, bands 1..bands-2 hidden split evenly, last band = n_outputs
// outputs).  Node v of band b >= 1 gets
//   - one mandatory predecessor in band b-1 (pins its level to b),
//   - a Pareto(alpha) number of extra sources drawn uniformly without
//     replacement from all earlier bands [0, start(b)), scaled so that the
//     expected edge total is target_edges,
//   - every node of band b-1 that picked v as its mandatory successor (each
//     non-output node picks one in band b+1, so every node reaches an output
//     and is required).
// All randomness is a per-node SplitMix64 stream (gen_core.h pl_succ /
// pl_draw, shared with the device generator in gen.cu), so the result does
// not depend on the thread count or the processor.  Edges are target-major,
// sources ascending, weights U[-1, 1].
int asnn_gen_powerlaw(uint32_t n_nodes, uint32_t bands, uint32_t n_in, uint32_t n_out,
                      uint64_t target_edges, double alpha, uint64_t seed, asnn_corpus** result) {
    if (!result || bands < 3 || n_in == 0 || n_out == 0 || !(alpha > 1.0) ||
        n_nodes < n_in + n_out + (bands - 2))
        return ASNN_E_INVALID;
    const auto starts = band_starts(n_in, n_out, n_nodes - n_in - n_out, bands);
    const asnn_gen::PowerlawSpec spec{starts.data(), bands, powerlaw_xm(n_nodes, n_in, n_out, target_edges, alpha),
                                      alpha, seed};
    const std::uint32_t first = n_in;

    // Pass 1: mandatory successor of every non-output node.
    std::vector<std::uint32_t> msucc_count(n_nodes + 1, 0);
    std::vector<std::uint32_t> msucc(n_nodes, 0xFFFFFFFFu);
#pragma omp parallel for schedule(static)
    for (std::int64_t v = 0; v < static_cast<std::int64_t>(starts[bands - 1]); ++v)
        msucc[v] = asnn_gen::pl_succ(spec, static_cast<std::uint32_t>(v));
    for (std::uint32_t v = 0; v < starts[bands - 1]; ++v) msucc_count[msucc[v] + 1]++;
    for (std::uint32_t t = 0; t < n_nodes; ++t) msucc_count[t + 1] += msucc_count[t];
    std::vector<std::uint32_t> msucc_src(msucc_count[n_nodes]);
    {
        std::vector<std::uint32_t> cur(msucc_count.begin(), msucc_count.end() - 1);
        for (std::uint32_t v = 0; v < starts[bands - 1]; ++v) msucc_src[cur[msucc[v]]++] = v;
    }

    // Pass 2: per-target source lists (sizes first, then fill).
    auto draw_sources = [&](std::uint32_t t, std::vector<std::uint32_t>& out_src,
                            std::vector<float>* out_w) {
        out_src.clear();
        for (std::uint32_t i = msucc_count[t]; i < msucc_count[t + 1]; ++i) out_src.push_back(msucc_src[i]);
        asnn_gen::Rng r = asnn_gen::pl_draw(spec, t, [&](std::uint32_t s) { out_src.push_back(s); });
        std::sort(out_src.begin(), out_src.end());
        out_src.erase(std::unique(out_src.begin(), out_src.end()), out_src.end());
        if (out_w) {
            out_w->resize(out_src.size());
            for (auto& x : *out_w) x = r.uniform(-1.0f, 1.0f);
        }
    };
    std::vector<std::uint64_t> row(n_nodes + 1, 0);
#pragma omp parallel
    {
        std::vector<std::uint32_t> tmp;
#pragma omp for schedule(dynamic, 1024)
        for (std::int64_t t = first; t < static_cast<std::int64_t>(n_nodes); ++t) {
            draw_sources(static_cast<std::uint32_t>(t), tmp, nullptr);
            row[t + 1] = tmp.size();
        }
    }
    for (std::uint32_t t = 0; t < n_nodes; ++t) row[t + 1] += row[t];
    auto* c = new asnn_corpus;
    const std::uint64_t E = row[n_nodes];
    c->src.resize(E);
    c->dst.resize(E);
    c->w.resize(E);
#pragma omp parallel
    {
        std::vector<std::uint32_t> tmp;
        std::vector<float> tw;
#pragma omp for schedule(dynamic, 1024)
        for (std::int64_t t = first; t < static_cast<std::int64_t>(n_nodes); ++t) {
            draw_sources(static_cast<std::uint32_t>(t), tmp, &tw);
            const std::uint64_t b = row[t];
            std::memcpy(&c->src[b], tmp.data(), tmp.size() * 4);
            std::memcpy(&c->w[b], tw.data(), tw.size() * 4);
            std::fill(c->dst.begin() + b, c->dst.begin() + b + tmp.size(),
                      static_cast<std::uint32_t>(t));
        }
    }
    c->nodes.resize(n_nodes);
    for (std::uint32_t i = 0; i < n_nodes; ++i) c->nodes[i] = i;
    for (std::uint32_t i = 0; i < n_in; ++i) c->inputs.push_back(i);
    for (std::uint32_t i = 0; i < n_out; ++i) c->outputs.push_back(starts[bands - 1] + i);
    *result = c;
    return ASNN_OK;
}

int asnn_corpus_desc(const asnn_corpus* c, asnn_network_desc* d) {
    if (!c || !d) return ASNN_E_INVALID;
    d->n_nodes = static_cast<std::uint32_t>(c->nodes.size());
    d->nodes = c->nodes.data();
    d->n_inputs = static_cast<std::uint32_t>(c->inputs.size());
    d->inputs = c->inputs.data();
    d->n_outputs = static_cast<std::uint32_t>(c->outputs.size());
    d->outputs = c->outputs.data();
    d->n_connections = c->src.size();
    d->source = c->src.data();
    d->target = c->dst.data();
    d->weight = c->w.data();
    return ASNN_OK;
}

void asnn_corpus_free(asnn_corpus* c) { delete c; }

}  // extern "C"
