// tests/cpp/test_facade.cpp -- the C++ host API (include/asnn_b200.hpp) run
// through the reference's own test scenarios (proj/tests/test_segmentation.cpp,
// test_layout.cpp, test_eval.cpp), restated with a minimal CHECK harness (the
// reference's doctest.h is absent), plus seeded networks checked bitwise
// against the C oracle (oracle/asnn_oracle.c, linked as liboracle.so).
// Built by __graft_entry__.build(); run by tests/test_gpu_cpp.py on a GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "asnn_b200.hpp"

extern "C" {
int64_t orc_segment(uint32_t, const uint32_t*, uint32_t, const uint32_t*, uint64_t, const uint32_t*,
                    const uint32_t*, const uint8_t*, uint32_t*);
int orc_compute_required(uint32_t, const uint32_t*, uint32_t, const uint32_t*, uint64_t,
                         const uint32_t*, const uint32_t*, uint8_t*);
int orc_flatten(uint32_t, const uint32_t*, uint32_t, const uint32_t*, uint64_t, const uint32_t*,
                const uint32_t*, const float*, const uint32_t*, uint32_t, uint32_t*, uint32_t*,
                uint64_t*, uint32_t*, float*, uint32_t*, uint64_t*, uint32_t*);
int orc_eval_sequential(uint32_t, const uint32_t*, uint32_t, const uint64_t*, const uint32_t*,
                        const float*, uint32_t, const uint32_t*, uint32_t, const float*, uint32_t,
                        float*, float*);
}

using namespace asnn_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                           \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(cond)) {                                                        \
            ++g_fail;                                                         \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                  \
    do {                                          \
        bool thrown = false;                      \
        try {                                     \
            (void)(expr);                         \
        } catch (const T&) {                      \
            thrown = true;                        \
        } catch (...) {                           \
        }                                         \
        CHECK(thrown);                            \
    } while (0)

static Network fixture_two_in_one_out() { return make_network({0, 1}, {2}, {{0, 2, 0.5f}, {1, 2, -0.25f}}); }
static Network fixture_skip_connection() {
    return make_network({0}, {3}, {{0, 1, 1.0f}, {0, 2, 0.5f}, {1, 2, -1.0f}, {2, 3, 0.75f}, {0, 3, 0.25f}});
}
static Network fixture_pruned_node() { return make_network({0}, {2}, {{0, 2, 1.0f}, {0, 3, 1.0f}}); }

static LayeredLayout make_layout(const Network& n) { return flatten(n, segment(n, compute_required(n))); }

static void segmentation_cases() {  // test_segmentation.cpp:10-48
    auto a = segment(fixture_two_in_one_out(), compute_required(fixture_two_in_one_out()));
    CHECK(a.layers.size() == 2);
    CHECK((a.layers[0] == std::vector<NodeId>{0, 1}) && (a.layers[1] == std::vector<NodeId>{2}));
    CHECK(a.unassigned.empty() && depth(a) == 2);
    a = segment(fixture_skip_connection(), compute_required(fixture_skip_connection()));
    CHECK(a.layers.size() == 4 && a.layers[3] == std::vector<NodeId>{3});
    const Network p = fixture_pruned_node();
    a = segment(p, compute_required(p));
    CHECK(a.layers.size() == 2 && a.unassigned == std::vector<NodeId>{3});
    CHECK(unassigned_outputs(p, a).empty());
    CHECK(a.layer_of(0) == 0u && a.layer_of(2) == 1u && !a.layer_of(3) && !a.layer_of(99));
    CHECK(a.assigned_count() == 2);
    const Network u = make_network({0}, {2}, {{3, 2, 1.0f}}, {0});
    a = segment(u, compute_required(u));
    CHECK(unassigned_outputs(u, a) == std::vector<NodeId>{2});
    CHECK_THROWS_AS(flatten(u, a), UnassignedOutput);  // test_layout.cpp:41-47
}

static void layout_cases() {  // test_layout.cpp:18-72
    auto L = make_layout(fixture_two_in_one_out());
    CHECK(L.total_layers == 2 && (L.nodes_per_layer == std::vector<uint32_t>{2, 1}));
    CHECK(L.node_count() == 3 && L.nodes[2].id == 2);
    CHECK((L.nodes[2].in_nodes == std::vector<NodeId>{0, 1}));
    CHECK((L.nodes[2].in_weights == std::vector<float>{0.5f, -0.25f}));
    CHECK(L.dropped_connections == 0 && L.id_bound == 3);
    L = make_layout(fixture_skip_connection());
    CHECK((L.nodes[3].in_nodes == std::vector<NodeId>{0, 2}));
    CHECK((L.nodes[3].in_weights == std::vector<float>{0.25f, 0.75f}));
    L = make_layout(fixture_pruned_node());
    CHECK(L.node_count() == 2 && L.dropped_connections == 1 && L.id_bound == 4);
    L = make_layout(make_network({5, 30}, {90}, {{5, 90, 1.0f}, {30, 90, 1.0f}}));
    CHECK(L.id_bound == 91 && (L.nodes[2].in_nodes == std::vector<NodeId>{5, 30}));
    const auto two = make_layout(fixture_two_in_one_out());
    CHECK((layer_slice_bounds(two, 0) == std::pair<uint32_t, uint32_t>{0, 2}));
    CHECK((layer_slice_bounds(two, 1) == std::pair<uint32_t, uint32_t>{2, 1}));
    CHECK_THROWS_AS(layer_slice_bounds(two, 2), LayerOutOfRange);
    CHECK(max_layer_width(two) == 2 && max_layer_width(make_layout(fixture_skip_connection())) == 1);
}

static void eval_cases() {  // test_eval.cpp:22-107
    const auto L1 = make_layout(make_network({0}, {1}, {{0, 1, 1.0f}}));
    auto st = eval_parallel(L1, std::vector<float>{0.0f});
    CHECK(st.outputs[0] == 0.5f && std::fabs(st.outputs[1] - 0.9230835512325639) < 1e-6);
    const auto Lc = make_layout(make_network({0, 1}, {2}, {{0, 2, 1.0f}, {1, 2, -1.0f}}));
    for (float x : {0.0f, 0.7f, -1.3f}) CHECK(eval_parallel(Lc, std::vector<float>{x, x}).outputs[2] == 0.5f);
    const auto Ls = make_layout(fixture_two_in_one_out());
    st = eval_parallel(Ls, std::vector<float>{1.0f, -1.0f});
    CHECK(std::fabs(st.outputs[0] - 0.9931047268673539) < 1e-6 && st.inputs[0] == 1.0f && st.inputs[1] == -1.0f);
    const Network o = make_network({0, 1}, {4, 3}, {{0, 3, 1.0f}, {1, 4, 1.0f}, {0, 4, 0.5f}});
    st = eval_parallel(make_layout(o), std::vector<float>{0.2f, -0.9f});
    const auto outs = read_outputs(st, o);
    CHECK(outs.size() == 2 && outs[0] == st.outputs[4] && outs[1] == st.outputs[3]);
    CHECK_THROWS_AS(eval_parallel(Ls, std::vector<float>{1.0f}), InputArityMismatch);
    CHECK_THROWS_AS(eval_parallel(Ls, std::vector<float>{1.0f, 2.0f, 3.0f}), InputArityMismatch);
    ParallelConfig host;
    host.backend = ParallelConfig::Backend::HostParallel;
    CHECK_THROWS_AS(eval_parallel(Ls, std::vector<float>{0.0f, 0.0f}, host), BackendUnavailable);
    ParallelConfig hook;
    hook.node_hook = [](NodeId) {};
    CHECK_THROWS_AS(eval_parallel(Ls, std::vector<float>{0.0f, 0.0f}, hook), BackendUnavailable);
}

// Random DAGs over sparse ids vs the C oracle: levels, rows and activations bitwise.
static void random_vs_oracle() {
    std::mt19937_64 rng(2005);
    for (int trial = 0; trial < 40; ++trial) {
        const uint32_t n = 20 + rng() % 400;
        std::vector<NodeId> ids(n);
        for (uint32_t i = 0; i < n; ++i) ids[i] = i * 3 + static_cast<uint32_t>(rng() % 3);
        const uint32_t n_in = 1 + rng() % 6;
        std::vector<NodeId> inputs(ids.begin(), ids.begin() + n_in);
        std::vector<Connection> conns;
        for (uint32_t t = n_in; t < n; ++t) {
            const uint32_t k = 1 + rng() % 8;
            std::vector<uint32_t> srcs;
            for (uint32_t j = 0; j < k; ++j) srcs.push_back(rng() % t);
            std::sort(srcs.begin(), srcs.end());
            srcs.erase(std::unique(srcs.begin(), srcs.end()), srcs.end());
            for (uint32_t s : srcs)
                conns.push_back({ids[s], ids[t], std::uniform_real_distribution<float>(-1.5f, 1.5f)(rng)});
        }
        std::shuffle(conns.begin(), conns.end(), rng);
        std::vector<NodeId> outputs{ids[n - 1], ids[n - 2]};
        const Network net = make_network(inputs, outputs, conns);
        // oracle
        std::vector<uint32_t> src, dst;
        std::vector<float> w;
        for (const auto& c : net.connections) {
            src.push_back(c.source);
            dst.push_back(c.target);
            w.push_back(c.weight);
        }
        const uint32_t N = static_cast<uint32_t>(net.nodes.size());
        std::vector<uint8_t> req(N);
        orc_compute_required(N, net.nodes.data(), 2, outputs.data(), src.size(), src.data(), dst.data(), req.data());
        std::vector<uint32_t> level(N);
        const int64_t nl = orc_segment(N, net.nodes.data(), n_in, inputs.data(), src.size(), src.data(),
                                       dst.data(), req.data(), level.data());
        const auto a = segment(net, compute_required(net));
        CHECK(static_cast<int64_t>(a.layers.size()) == nl);
        bool levels_ok = true;
        for (uint32_t i = 0; i < N; ++i) {
            const auto l = a.layer_of(net.nodes[i]);
            levels_ok &= level[i] == ASNN_UNASSIGNED ? !l : (l && *l == level[i]);
        }
        CHECK(levels_ok);
        if (!unassigned_outputs(net, a).empty()) continue;
        std::vector<uint32_t> lo(nl + 1), nids(N), in(src.size());
        std::vector<uint64_t> rp(N + 1);
        std::vector<float> iw(src.size());
        uint32_t na = 0, idb = 0;
        uint64_t drop = 0;
        orc_flatten(N, net.nodes.data(), 2, outputs.data(), src.size(), src.data(), dst.data(), w.data(),
                    level.data(), static_cast<uint32_t>(nl), lo.data(), nids.data(), rp.data(), in.data(),
                    iw.data(), &na, &drop, &idb);
        const auto L = flatten(net, a);
        bool rows_ok = L.node_count() == na && L.dropped_connections == drop && L.id_bound == idb;
        for (uint32_t p = 0; rows_ok && p < na; ++p) {
            rows_ok &= L.nodes[p].id == nids[p];
            rows_ok &= L.nodes[p].in_nodes == std::vector<NodeId>(in.begin() + rp[p], in.begin() + rp[p + 1]);
            rows_ok &= std::memcmp(L.nodes[p].in_weights.data(), iw.data() + rp[p],
                                   (rp[p + 1] - rp[p]) * 4) == 0;
        }
        CHECK(rows_ok);
        std::vector<float> x(n_in);
        for (auto& v : x) v = std::uniform_real_distribution<float>(-2.0f, 2.0f)(rng);
        std::vector<float> si(idb), so(idb);
        orc_eval_sequential(na, nids.data(), lo[1], rp.data(), in.data(), iw.data(), n_in, inputs.data(), idb,
                            x.data(), n_in, si.data(), so.data());
        const auto st = eval_parallel(L, x);
        CHECK(std::memcmp(st.outputs.data(), so.data(), idb * 4) == 0);  // bitwise
        DeviceNetwork dn(net);
        const auto out = dn.activate(x, 1);
        CHECK(out.size() == 2 && out[0] == so[outputs[0]] && out[1] == so[outputs[1]]);
    }
}

// Multi-GPU through the facade (csrc/group.cu): a 2-device group over device 0
// (the copy-engine gather; one B200 in the test box) shards a batch and a
// population; results equal the single-device activation bit for bit.
static Network random_net(std::mt19937_64& rng, uint32_t n, uint32_t n_in, uint32_t n_out) {
    std::vector<Connection> conns;
    for (uint32_t t = n_in; t < n; ++t) {
        const uint32_t k = 1 + rng() % 6;
        for (uint32_t j = 0; j < k; ++j)
            conns.push_back({static_cast<NodeId>(rng() % t), t, std::uniform_real_distribution<float>(-1.5f, 1.5f)(rng)});
    }
    std::sort(conns.begin(), conns.end(), [](const Connection& a, const Connection& b) {
        return a.target != b.target ? a.target < b.target : a.source < b.source;
    });
    conns.erase(std::unique(conns.begin(), conns.end(),
                            [](const Connection& a, const Connection& b) {
                                return a.source == b.source && a.target == b.target;
                            }),
                conns.end());
    std::vector<NodeId> inputs(n_in), outputs;
    for (uint32_t i = 0; i < n_in; ++i) inputs[i] = i;
    for (uint32_t i = 0; i < n_out; ++i) outputs.push_back(n - 1 - i);
    return make_network(inputs, outputs, conns);
}

static void group_cases() {
    std::mt19937_64 rng(99);
    DeviceGroup grp({0, 0});
    CHECK(grp.gather() == "copy engines");
    const Network net = random_net(rng, 600, 5, 3);
    for (uint32_t B : {1u, 7u, 64u}) {
        std::vector<float> X(static_cast<size_t>(B) * 5);
        for (auto& v : X) v = std::uniform_real_distribution<float>(-2.0f, 2.0f)(rng);
        GroupNetwork gn(grp, net);
        DeviceNetwork dn(net);
        const auto a = gn.activate(X, B), b = dn.activate(X, B);
        CHECK(a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0);
    }
    std::vector<Network> pop;
    for (int k = 0; k < 9; ++k) pop.push_back(random_net(rng, 80 + k * 7, 4, 2));
    const uint32_t V = 5;
    std::vector<float> X;
    for (size_t k = 0; k < pop.size() * V * 4; ++k) X.push_back(std::uniform_real_distribution<float>(-2.0f, 2.0f)(rng));
    GroupNetwork gp(grp, pop);
    const auto all = gp.activate(X, V);
    CHECK(all.size() == pop.size() * V * 2);
    bool same = true;
    for (size_t k = 0; k < pop.size(); ++k) {
        DeviceNetwork dn(pop[k]);
        const auto o = dn.activate(std::span<const float>(X.data() + k * V * 4, V * 4), V);
        same &= std::memcmp(o.data(), all.data() + k * V * 2, o.size() * 4) == 0;
    }
    CHECK(same);
    CHECK_THROWS_AS(gp.activate(std::span<const float>(X.data(), X.size() - 1), V), InputArityMismatch);
}

// io.hpp through the facade: the test_io.cpp scenarios of the reference
// (round trip, comments / blank lines / CRLF, ParseError line numbers,
// ValidationError messages, IoError).
static void io_cases() {
    const std::string text =
        "# a comment\n\nasnn 1\r\ninputs 0 1\noutputs 3\nedge 0 2 0.5\n  edge\t1 2 -0.25\nedge 2 3 1e-3\n";
    const Network net = parse_network(text);
    CHECK(net.nodes == std::vector<NodeId>({0, 1, 2, 3}));
    CHECK(net.inputs == std::vector<NodeId>({0, 1}) && net.outputs == std::vector<NodeId>({3}));
    CHECK(net.connections.size() == 3 && net.connections[1].source == 1 && net.connections[1].weight == -0.25f);
    CHECK(net.connections[2].weight == 1e-3f);
    auto parse_line = [](const std::string& t) {
        try {
            parse_network(t);
        } catch (const ParseError& e) {
            return e.line;
        }
        return -1;
    };
    CHECK(parse_line("asnn 2\ninputs 0\noutputs 1\n") == 1);
    CHECK(parse_line("asnn 1\ninputs 0\noutputs 1\nedge 0 1 0.5\nedge 0 1 0.5\n") == 5);
    CHECK(parse_line("asnn 1\ninputs 0\noutputs 1\nedge 0 1 x\n") == 4);
    CHECK(parse_line("asnn 1\ninputs 0\n") == 3);  // truncated file
    bool validation = false;
    try {
        parse_network("asnn 1\ninputs 0\noutputs 2\nedge 0 1 1\nedge 1 2 1\nedge 2 1 1\n");
    } catch (const ValidationError& e) {
        validation = e.violations.size() == 1 && e.violations[0] == "cycle: 1->2->1->1";  // network.cpp:125-135 path format
    }
    CHECK(validation);
    const Network bad = make_network({0}, {2}, {{0, 1, 1.0f}, {1, 2, 1.0f}, {2, 1, 1.0f}, {1, 1, 0.5f}});
    const auto rep = validate(bad);
    CHECK(!rep.ok() && rep.violations.size() == 2 && rep.violations[0] == "self-loop at node 1");
    CHECK(validate(net).ok());
    const Network sparse = make_network({10}, {30}, {{10, 20, 1.0f}, {20, 30, 1.0f}});
    const Network dense = normalize(sparse);
    CHECK(dense.nodes == std::vector<NodeId>({0, 1, 2}) && dense.connections[1].source == 1 &&
          dense.connections[1].target == 2);
    bool io = false;
    try {
        read_network("/nonexistent/dir/net.asnn");
    } catch (const IoError&) {
        io = true;
    }
    CHECK(io);
}

int main() {
    try {
        io_cases();
        segmentation_cases();
        layout_cases();
        eval_cases();
        random_vs_oracle();
        group_cases();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "uncaught exception: %s\n", e.what());
        return 2;
    }
    std::printf("{\"checks\": %d, \"failures\": %d}\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
