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

// Open-addressing set / map of non-zero 64-bit keys (linear probing, power-of-
// two capacity, never shrinks): the generator's only dynamic structures, sized
// by the connection count rather than by the forward-pair space.
struct KeyTable {
    std::vector<std::uint64_t> key;
    std::vector<std::uint64_t> val;
    std::uint64_t mask = 0;
    explicit KeyTable(std::uint64_t n, bool with_values) {
        std::uint64_t cap = 16;
        while (cap < 2 * n + 2) cap <<= 1;
        key.assign(cap, 0);
        if (with_values) val.assign(cap, 0);
        mask = cap - 1;
    }
    static std::uint64_t mix(std::uint64_t k) {
        k ^= k >> 33;
        k *= 0xFF51AFD7ED558CCDull;
        return k ^ (k >> 29);
    }
    // slot of k: holds k, or is the empty slot where k would go
    std::uint64_t find(std::uint64_t k) const {
        std::uint64_t i = mix(k) & mask;
        while (key[i] != 0 && key[i] != k) i = (i + 1) & mask;
        return i;
    }
    bool insert(std::uint64_t k) {  // false when already present
        const std::uint64_t i = find(k);
        if (key[i] == k) return false;
        key[i] = k;
        return true;
    }
};

// The forward-pair space of a banded network, by arithmetic on the bands:
// every target of band b >= 1 has the same source range [0, start(b)), so the
// space is piecewise regular -- pair index -> (source, target) is a search over
// the bands (<= depth entries) and a division, with no per-node table.
struct PairSpace {
    const std::vector<std::uint32_t>& starts;
    std::vector<std::uint64_t> off;  // off[b]: first pair index of band b (b >= 1)
    std::uint32_t drop;              // sources removed per target (0, or 1 = the mandatory one)
    PairSpace(const std::vector<std::uint32_t>& st, std::uint32_t d) : starts(st), off(st.size(), 0), drop(d) {
        for (std::size_t b = 1; b + 1 < st.size(); ++b)
            off[b + 1] = off[b] + static_cast<std::uint64_t>(st[b + 1] - st[b]) * (st[b] - drop);
    }
    std::uint64_t size() const { return off[starts.size() - 1]; }
    // index -> target node and source rank within the target's range
    void locate(std::uint64_t idx, std::uint32_t& node, std::uint32_t& rank) const {
        std::size_t b = 1;
        while (b + 2 < starts.size() && off[b + 1] <= idx) ++b;
        const std::uint64_t w = starts[b] - drop, r = idx - off[b];
        node = starts[b] + static_cast<std::uint32_t>(r / w);
        rank = static_cast<std::uint32_t>(r % w);
    }
};

}  // namespace

extern "C" {

uint64_t asnn_gen_max_connections(uint32_t in, uint32_t out, uint32_t hidden, uint32_t depth) {
    return capacity_of(band_starts(in, out, hidden, depth));
}

// Same networks as generate() (netgen.cpp:71-157), byte for byte: the
// SplitMix64 stream is consumed in the reference's order -- per non-input
// node ascending a mandatory source in the adjacent band and its weight, then
// the remaining connections as uniform unused forward pairs, then everything
// sorted by (source, target).
//
// The pair selection is reorganised so memory follows the connection count,
// not the pair space (config-scale specs have pair spaces of 10^11+):
//  * sparse requests (netgen.cpp:129-141): the drawn pair index is decoded by
//    band arithmetic (PairSpace) and deduplicated in a KeyTable;
//  * dense requests (netgen.cpp:115-128): the reference shuffles a
//    materialised list of the free pairs (target-major, sources ascending,
//    mandatory pairs left out) and takes its prefix.  The same draws drive a
//    virtual Fisher-Yates here: list entries are computed from their rank
//    (each target's free sources are its range minus its one mandatory
//    source), and only displaced ranks are stored.
int asnn_gen_reference(uint32_t in, uint32_t out, uint32_t hidden, uint64_t conn, uint32_t depth,
                       float wmin, float wmax, uint64_t seed, asnn_corpus** result) {
    if (!result) return ASNN_E_INVALID;
    *result = nullptr;
    // feasibility (netgen.cpp:29-53)
    if (in == 0 || out == 0 || depth < 2 || (depth == 2 && hidden > 0) ||
        (depth > 2 && hidden < depth - 2) || !(wmin <= wmax))
        return ASNN_E_INFEASIBLE;
    const auto starts = band_starts(in, out, hidden, depth);
    if (conn < static_cast<std::uint64_t>(hidden) + out || conn > capacity_of(starts))
        return ASNN_E_INFEASIBLE;

    const std::uint32_t n_nodes = starts.back();
    SplitMix64 rng(seed);
    struct Edge {
        std::uint64_t key;  // source << 32 | target (unique)
        float w;
    };
    std::vector<Edge> edges;
    edges.reserve(conn);
    auto key_of = [](std::uint32_t s, std::uint32_t t) { return (static_cast<std::uint64_t>(s) << 32) | t; };

    // mandatory sources, band by band (= node order)
    std::vector<std::uint32_t> mand(n_nodes, 0);
    for (std::size_t b = 1; b + 1 < starts.size(); ++b)
        for (std::uint32_t v = starts[b]; v < starts[b + 1]; ++v) {
            mand[v] = starts[b - 1] + static_cast<std::uint32_t>(rng.bounded(starts[b] - starts[b - 1]));
            const float w = rng.uniform(wmin, wmax);
            edges.push_back({key_of(mand[v], v), w});
        }
    const std::uint64_t n_mand = edges.size();
    const std::uint64_t remaining = conn - n_mand;
    const PairSpace all(starts, 0);

    if (remaining * 2 > all.size() - n_mand) {
        const PairSpace free_space(starts, 1);  // one mandatory source per target left out
        KeyTable moved(remaining, true);        // rank position -> displaced rank (+1)
        for (std::uint64_t k = 0; k < remaining; ++k) {
            const std::uint64_t j = k + rng.bounded(free_space.size() - k);
            auto at = [&moved](std::uint64_t pos) {
                const std::uint64_t i = moved.find(pos + 1);
                return moved.key[i] ? moved.val[i] - 1 : pos;
            };
            const std::uint64_t pick = at(j);
            const std::uint64_t i = moved.find(j + 1);
            moved.key[i] = j + 1;
            moved.val[i] = at(k) + 1;  // position k is never read again
            std::uint32_t v, r;
            free_space.locate(pick, v, r);
            const float w = rng.uniform(wmin, wmax);
            edges.push_back({key_of(r < mand[v] ? r : r + 1, v), w});
        }
    } else {
        KeyTable used(conn, false);
        for (std::uint64_t e = 0; e < n_mand; ++e) used.insert(edges[e].key);
        while (edges.size() < conn) {
            std::uint32_t v, s;
            all.locate(rng.bounded(all.size()), v, s);
            if (!used.insert(key_of(s, v))) continue;  // a duplicate consumes no weight draw
            const float w = rng.uniform(wmin, wmax);
            edges.push_back({key_of(s, v), w});
        }
    }
    std::sort(edges.begin(), edges.end(), [](const Edge& x, const Edge& y) { return x.key < y.key; });

    auto* c = new asnn_corpus;
    c->src.resize(edges.size());
    c->dst.resize(edges.size());
    c->w.resize(edges.size());
    for (std::size_t i = 0; i < edges.size(); ++i) {
        c->src[i] = static_cast<std::uint32_t>(edges[i].key >> 32);
        c->dst[i] = static_cast<std::uint32_t>(edges[i].key);
        c->w[i] = edges[i].w;
    }
    // dense ids; inputs = band 0, outputs = the last band (netgen.cpp:147-156)
    c->nodes.resize(n_nodes);
    for (std::uint32_t i = 0; i < n_nodes; ++i) c->nodes[i] = i;
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
