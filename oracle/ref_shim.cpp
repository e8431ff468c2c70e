// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" surface over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libasnn_ref.so).  It lets the Python tests and the bench's
// reference arm drive the reference's own compute_required / segment /
// flatten / eval_sequential / eval_parallel / generate without a CLI
// (CLI11 and doctest are absent from the reference checkout).
// Nothing here re-implements reference logic: every entry point forwards to
// the reference function named in its comment and only converts containers.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <vector>

#include <charconv>
#include <string>
#include <string_view>

#include "asnn/errors.hpp"
#include "asnn/eval.hpp"
#include "asnn/io.hpp"
#include "asnn/layout.hpp"
#include "asnn/netgen.hpp"
#include "asnn/network.hpp"
#include "asnn/segmentation.hpp"

namespace {

struct RefHandle {
    asnn::Network net;
    asnn::RequiredSet required;
    asnn::LayerAssignment assignment;
    asnn::LayeredLayout layout;
    bool has_layout = false;
};

int map_exception() {
    try {
        throw;
    } catch (const asnn::InputArityMismatch&) {
        return 2;
    } catch (const asnn::UnassignedOutput&) {
        return 3;
    } catch (const asnn::LayerOutOfRange&) {
        return 4;
    } catch (const asnn::InfeasibleSpec&) {
        return 8;
    } catch (const asnn::BackendUnavailable&) {
        return 1;
    } catch (...) {
        return 5;
    }
}

}  // namespace

extern "C" {

// asnn::generate (netgen.cpp:71-157).  Returns a handle or nullptr (*err=8
// for InfeasibleSpec).
void* ref_generate(std::uint32_t in, std::uint32_t out, std::uint32_t hidden, std::uint64_t conn,
                   std::uint32_t depth, float wmin, float wmax, std::uint64_t seed, int* err) {
    try {
        asnn::GenSpec spec;
        spec.input_count = in;
        spec.output_count = out;
        spec.hidden_count = hidden;
        spec.connection_count = conn;
        spec.target_depth = depth;
        spec.weight_min = wmin;
        spec.weight_max = wmax;
        spec.seed = seed;
        auto h = std::make_unique<RefHandle>();
        h->net = asnn::generate(spec);
        *err = 0;
        return h.release();
    } catch (...) {
        *err = map_exception();
        return nullptr;
    }
}

// asnn::max_connections (netgen.cpp:63-69).
std::uint64_t ref_max_connections(std::uint32_t in, std::uint32_t out, std::uint32_t hidden,
                                  std::uint32_t depth) {
    asnn::GenSpec spec;
    spec.input_count = in;
    spec.output_count = out;
    spec.hidden_count = hidden;
    spec.target_depth = depth;
    return asnn::max_connections(spec);
}

// Wraps caller arrays into an asnn::Network verbatim (field by field, no
// make_network normalisation, so sparse or unsorted test inputs stay as given).
void* ref_network(std::uint32_t n_nodes, const std::uint32_t* nodes, std::uint32_t n_in,
                  const std::uint32_t* inputs, std::uint32_t n_out, const std::uint32_t* outputs,
                  std::uint64_t n_edges, const std::uint32_t* src, const std::uint32_t* dst,
                  const float* w) {
    auto h = std::make_unique<RefHandle>();
    h->net.nodes.assign(nodes, nodes + n_nodes);
    h->net.inputs.assign(inputs, inputs + n_in);
    h->net.outputs.assign(outputs, outputs + n_out);
    h->net.connections.resize(n_edges);
    for (std::uint64_t e = 0; e < n_edges; ++e) h->net.connections[e] = {src[e], dst[e], w[e]};
    return h.release();
}

void ref_free(void* hp) { delete static_cast<RefHandle*>(hp); }

// --- network getters ---------------------------------------------------------
std::uint32_t ref_net_n_nodes(void* hp) { return static_cast<RefHandle*>(hp)->net.nodes.size(); }
std::uint32_t ref_net_n_inputs(void* hp) { return static_cast<RefHandle*>(hp)->net.inputs.size(); }
std::uint32_t ref_net_n_outputs(void* hp) { return static_cast<RefHandle*>(hp)->net.outputs.size(); }
std::uint64_t ref_net_n_edges(void* hp) {
    return static_cast<RefHandle*>(hp)->net.connections.size();
}
void ref_net_copy(void* hp, std::uint32_t* nodes, std::uint32_t* inputs, std::uint32_t* outputs,
                  std::uint32_t* src, std::uint32_t* dst, float* w) {
    const auto& n = static_cast<RefHandle*>(hp)->net;
    std::memcpy(nodes, n.nodes.data(), n.nodes.size() * 4);
    std::memcpy(inputs, n.inputs.data(), n.inputs.size() * 4);
    std::memcpy(outputs, n.outputs.data(), n.outputs.size() * 4);
    for (std::size_t e = 0; e < n.connections.size(); ++e) {
        src[e] = n.connections[e].source;
        dst[e] = n.connections[e].target;
        w[e] = n.connections[e].weight;
    }
}

// asnn::validate (network.cpp:151-216): number of violations.
std::uint32_t ref_validate(void* hp) {
    return asnn::validate(static_cast<RefHandle*>(hp)->net).violations.size();
}

// validate (network.cpp:151-216): the messages joined by '\n' into buf.
std::uint32_t ref_validate_report(void* hp, char* buf, std::uint64_t cap) {
    const auto msgs = asnn::validate(static_cast<RefHandle*>(hp)->net).messages();
    std::string all;
    for (std::size_t i = 0; i < msgs.size(); ++i) all += (i ? "\n" : "") + msgs[i];
    const std::size_t m = std::min<std::size_t>(all.size(), cap - 1);
    std::memcpy(buf, all.data(), m);
    buf[m] = 0;
    return static_cast<std::uint32_t>(msgs.size());
}

// normalize (network.cpp:69-85) into a new handle.
void* ref_normalize(void* hp) {
    auto h = std::make_unique<RefHandle>();
    h->net = asnn::normalize(static_cast<RefHandle*>(hp)->net);
    return h.release();
}

// compute_required (network.cpp:222-255) + segment (segmentation.cpp:20-101)
// + flatten (layout.cpp:12-83).  Returns 0, or 3 when flatten throws
// UnassignedOutput (the assignment is still available).
int ref_preprocess(void* hp) {
    auto* h = static_cast<RefHandle*>(hp);
    try {
        h->required = asnn::compute_required(h->net);
        h->assignment = asnn::segment(h->net, h->required);
        h->layout = asnn::flatten(h->net, h->assignment);
        h->has_layout = true;
        return 0;
    } catch (...) {
        h->has_layout = false;
        return map_exception();
    }
}

// Timed variant for the CPU baseline (seconds per phase).
int ref_preprocess_timed(void* hp, double* t_required, double* t_segment, double* t_flatten) {
    auto* h = static_cast<RefHandle*>(hp);
    using clk = std::chrono::steady_clock;
    try {
        auto t0 = clk::now();
        h->required = asnn::compute_required(h->net);
        auto t1 = clk::now();
        h->assignment = asnn::segment(h->net, h->required);
        auto t2 = clk::now();
        h->layout = asnn::flatten(h->net, h->assignment);
        auto t3 = clk::now();
        *t_required = std::chrono::duration<double>(t1 - t0).count();
        *t_segment = std::chrono::duration<double>(t2 - t1).count();
        *t_flatten = std::chrono::duration<double>(t3 - t2).count();
        h->has_layout = true;
        return 0;
    } catch (...) {
        h->has_layout = false;
        return map_exception();
    }
}

std::uint32_t ref_required_count(void* hp) {
    return static_cast<RefHandle*>(hp)->required.members.size();
}
void ref_required_copy(void* hp, std::uint32_t* members) {
    const auto& m = static_cast<RefHandle*>(hp)->required.members;
    std::memcpy(members, m.data(), m.size() * 4);
}

// LayerAssignment (segmentation.hpp:14-21).
std::uint32_t ref_n_layers(void* hp) { return static_cast<RefHandle*>(hp)->assignment.layers.size(); }
std::uint32_t ref_assigned_count(void* hp) {
    return static_cast<RefHandle*>(hp)->assignment.assigned_count();
}
std::uint32_t ref_unassigned_count(void* hp) {
    return static_cast<RefHandle*>(hp)->assignment.unassigned.size();
}
// layer_sizes[n_layers], members[assigned] concatenated, unassigned[...]
void ref_assignment_copy(void* hp, std::uint32_t* layer_sizes, std::uint32_t* members,
                         std::uint32_t* unassigned) {
    const auto& a = static_cast<RefHandle*>(hp)->assignment;
    std::size_t k = 0;
    for (std::size_t l = 0; l < a.layers.size(); ++l) {
        layer_sizes[l] = a.layers[l].size();
        for (auto id : a.layers[l]) members[k++] = id;
    }
    std::memcpy(unassigned, a.unassigned.data(), a.unassigned.size() * 4);
}

// LayeredLayout (layout.hpp:27-37) as CSR.
std::uint32_t ref_layout_node_count(void* hp) {
    return static_cast<RefHandle*>(hp)->layout.node_count();
}
std::uint64_t ref_layout_edge_count(void* hp) {
    std::uint64_t n = 0;
    for (const auto& node : static_cast<RefHandle*>(hp)->layout.nodes) n += node.in_nodes.size();
    return n;
}
std::uint32_t ref_layout_total_layers(void* hp) {
    return static_cast<RefHandle*>(hp)->layout.total_layers;
}
std::uint32_t ref_layout_id_bound(void* hp) { return static_cast<RefHandle*>(hp)->layout.id_bound; }
std::uint64_t ref_layout_dropped(void* hp) {
    return static_cast<RefHandle*>(hp)->layout.dropped_connections;
}
void ref_layout_copy(void* hp, std::uint32_t* layer_offsets, std::uint32_t* node_ids,
                     std::uint32_t* node_layer, std::uint8_t* is_sensor, std::uint64_t* row_ptr,
                     std::uint32_t* in_nodes, float* in_weights, std::uint32_t* input_order) {
    const auto& L = static_cast<RefHandle*>(hp)->layout;
    std::memcpy(layer_offsets, L.layer_offsets.data(), L.layer_offsets.size() * 4);
    std::uint64_t k = 0;
    row_ptr[0] = 0;
    for (std::size_t p = 0; p < L.nodes.size(); ++p) {
        const auto& n = L.nodes[p];
        node_ids[p] = n.id;
        node_layer[p] = n.layer;
        is_sensor[p] = n.is_sensor ? 1 : 0;
        for (std::size_t i = 0; i < n.in_nodes.size(); ++i, ++k) {
            in_nodes[k] = n.in_nodes[i];
            in_weights[k] = n.in_weights[i];
        }
        row_ptr[p + 1] = k;
    }
    std::memcpy(input_order, L.input_order.data(), L.input_order.size() * 4);
}

// Builds an asnn::LayeredLayout directly from CSR arrays, for bench shapes
// whose reference preprocessing would take tens of minutes.
// Field meaning is exactly layout.hpp:13-37; the evaluators are untouched.
void* ref_layout_from_csr(std::uint32_t total_layers, const std::uint32_t* layer_offsets,
                          std::uint32_t node_count, const std::uint32_t* node_ids,
                          const std::uint64_t* row_ptr, const std::uint32_t* in_nodes,
                          const float* in_weights, std::uint32_t n_in,
                          const std::uint32_t* input_order, std::uint32_t id_bound) {
    auto h = std::make_unique<RefHandle>();
    auto& L = h->layout;
    L.total_layers = total_layers;
    L.layer_offsets.assign(layer_offsets, layer_offsets + total_layers + 1);
    L.nodes_per_layer.resize(total_layers);
    for (std::uint32_t l = 0; l < total_layers; ++l)
        L.nodes_per_layer[l] = layer_offsets[l + 1] - layer_offsets[l];
    L.nodes.resize(node_count);
    std::uint32_t layer = 0;
#pragma omp parallel for schedule(dynamic, 4096)
    for (std::int64_t p = 0; p < static_cast<std::int64_t>(node_count); ++p) {
        auto& n = L.nodes[p];
        n.id = node_ids[p];
        n.in_nodes.assign(in_nodes + row_ptr[p], in_nodes + row_ptr[p + 1]);
        n.in_weights.assign(in_weights + row_ptr[p], in_weights + row_ptr[p + 1]);
    }
    for (std::uint32_t p = 0; p < node_count; ++p) {
        while (layer + 1 < total_layers && p >= layer_offsets[layer + 1]) ++layer;
        L.nodes[p].layer = layer;
        L.nodes[p].is_sensor = (layer == 0);
    }
    L.input_order.assign(input_order, input_order + n_in);
    L.id_bound = id_bound;
    h->has_layout = true;
    return h.release();
}

// eval_sequential (eval.cpp:39-47).  state_in / state_out: id_bound floats.
int ref_eval_sequential(void* hp, const float* x, std::uint32_t n_x, float* state_in,
                        float* state_out) {
    auto* h = static_cast<RefHandle*>(hp);
    try {
        auto st = asnn::eval_sequential(h->layout, std::span<const float>(x, n_x));
        if (state_in) std::memcpy(state_in, st.inputs.data(), st.inputs.size() * 4);
        if (state_out) std::memcpy(state_out, st.outputs.data(), st.outputs.size() * 4);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// eval_parallel (eval.cpp:49-80).  backend: 0 HostParallel, 1 DeviceCompute.
int ref_eval_parallel(void* hp, const float* x, std::uint32_t n_x, std::uint32_t workers,
                      int backend, float* state_out) {
    auto* h = static_cast<RefHandle*>(hp);
    try {
        asnn::ParallelConfig cfg;
        cfg.workers = workers;
        cfg.backend = backend ? asnn::ParallelConfig::Backend::DeviceCompute
                              : asnn::ParallelConfig::Backend::HostParallel;
        auto st = asnn::eval_parallel(h->layout, std::span<const float>(x, n_x), cfg);
        if (state_out) std::memcpy(state_out, st.outputs.data(), st.outputs.size() * 4);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Batch of n_vec vectors X[n_vec][n_in] through the reference evaluators, the
// three CPU-baseline modes of BASELINE.md section 3:
//   mode 0: eval_sequential, one vector after another, 1 thread;
//   mode 1: eval_parallel (HostParallel, `workers` threads) per vector;
//   mode 2: `workers`-thread OpenMP loop over vectors of eval_sequential.
// Output values of the declared outputs go to OUT[n_vec][n_out] when given
// (read_outputs, eval.cpp:82-87, needs the network: pass out_ids).
// Returns wall seconds for the whole batch, or a negative error code.
double ref_eval_batch(void* hp, const float* X, std::uint32_t n_vec, int mode, std::uint32_t workers,
                      const std::uint32_t* out_ids, std::uint32_t n_out, float* OUT) {
    auto* h = static_cast<RefHandle*>(hp);
    const std::uint32_t n_in = h->layout.input_order.size();
    const int nthreads = workers ? static_cast<int>(workers) : omp_get_max_threads();
    int err = 0;
    const auto t0 = std::chrono::steady_clock::now();
    try {
        if (mode == 2) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
            for (std::int64_t v = 0; v < static_cast<std::int64_t>(n_vec); ++v) {
                auto st = asnn::eval_sequential(
                    h->layout, std::span<const float>(X + static_cast<std::size_t>(v) * n_in, n_in));
                if (OUT)
                    for (std::uint32_t j = 0; j < n_out; ++j)
                        OUT[static_cast<std::size_t>(v) * n_out + j] = st.outputs[out_ids[j]];
            }
        } else {
            asnn::ParallelConfig cfg;
            cfg.workers = static_cast<std::uint32_t>(nthreads);
            for (std::uint32_t v = 0; v < n_vec; ++v) {
                std::span<const float> xs(X + static_cast<std::size_t>(v) * n_in, n_in);
                auto st = mode == 0 ? asnn::eval_sequential(h->layout, xs)
                                    : asnn::eval_parallel(h->layout, xs, cfg);
                if (OUT)
                    for (std::uint32_t j = 0; j < n_out; ++j)
                        OUT[static_cast<std::size_t>(v) * n_out + j] = st.outputs[out_ids[j]];
            }
        }
    } catch (...) {
        err = map_exception();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (err) return -static_cast<double>(err);
    return std::chrono::duration<double>(t1 - t0).count();
}

int ref_max_threads() { return omp_get_max_threads(); }

// The reference LayeredLayout object of a handle (for integration/ tests).
const void* ref_layout_ptr(void* hp) { return &static_cast<RefHandle*>(hp)->layout; }

// sigmoid32 (network.hpp:54-59) over an array, for exhaustive exp checks.
// asnn::parse_network (io.cpp:83-156).  Returns a handle on success; on
// failure nullptr with *kind = 1 (ParseError, *line = its line) or 2
// (ValidationError) or 3 (other) and the exception's what() in err.
void* ref_parse(const char* text, std::uint64_t len, int* kind, int* line, char* err, std::uint64_t cap) {
    *kind = 0;
    *line = 0;
    if (cap) err[0] = 0;
    auto put = [&](const char* w) {
        if (!cap) return;
        std::strncpy(err, w, cap - 1);
        err[cap - 1] = 0;
    };
    try {
        auto h = std::make_unique<RefHandle>();
        h->net = asnn::parse_network(std::string_view(text, len));
        return h.release();
    } catch (const asnn::ParseError& e) {
        *kind = 1;
        *line = e.line;
        put(e.what());
    } catch (const asnn::ValidationError& e) {
        *kind = 2;
        put(e.what());
    } catch (const std::exception& e) {
        *kind = 3;
        put(e.what());
    }
    return nullptr;
}

// asnn::serialize_network (io.cpp:25-45) into out (cap bytes); returns the
// text size (call with cap = 0 for the size), or UINT64_MAX if it throws.
std::uint64_t ref_serialize(void* hp, char* out, std::uint64_t cap) {
    try {
        const std::string t = asnn::serialize_network(static_cast<RefHandle*>(hp)->net);
        if (cap >= t.size()) std::memcpy(out, t.data(), t.size());
        return t.size();
    } catch (...) {
        return ~0ull;
    }
}

// std::from_chars as parse_weight / parse_id use it (io.cpp:66-80): status 0
// = parsed the whole token, else 1 (error or partial consumption).
void ref_from_chars_f32(const char* buf, const std::uint64_t* off, std::uint64_t n, float* out,
                        std::uint8_t* status) {
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
        const char* b = buf + off[i];
        const char* e = buf + off[i + 1];
        float v = 0.0f;
        const auto r = std::from_chars(b, e, v);
        status[i] = (r.ec != std::errc{} || r.ptr != e) ? 1 : 0;
        out[i] = status[i] ? 0.0f : v;
    }
}

// asnn::format_double (io.cpp:19-23) into out (cap bytes, NUL-terminated).
void ref_format_double(double v, char* out, std::uint64_t cap) {
    const std::string t = asnn::format_double(v);
    std::strncpy(out, t.c_str(), cap - 1);
    out[cap - 1] = 0;
}

void ref_sigmoid32_many(const float* in, float* out, std::uint64_t n) {
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) out[i] = asnn::sigmoid32(in[i]);
}

}  // extern "C"
