// asnn_b200.hpp -- C++ host API of the B200 engine, mirroring the reference's
// public API (proj/include/asnn/{network,segmentation,layout,eval,errors}.hpp)
// name for name, with every computation on the GPU through include/asnn_dev.h.
//
//   make_network        network.cpp:39-55        (host: node set union)
//   compute_required    network.cpp:222-255      -> asnn_dev_compute_required
//   segment             segmentation.cpp:20-101  -> asnn_dev_segment
//   flatten             layout.cpp:12-83         -> asnn_dev_build_layout + download
//   eval_parallel       eval.cpp:49-80           -> asnn_eval_buf_stage + asnn_eval_buf_run (one call)
//   read_outputs, layer_slice_bounds, max_layer_width, depth, unassigned_outputs
//   parse_network       io.cpp:83-156 + validate -> asnn_dev_parse_network
//   read_network        io.cpp:167-173           -> asnn_dev_read_network
//   validate, normalize network.cpp:69-85,151-216 -> asnn_dev_validate / _normalize
//
// Types keep the reference's field names and meanings; exceptions mirror
// errors.hpp:9-55.  There is no host evaluator: ParallelConfig defaults to
// Backend::DeviceCompute and HostParallel throws BackendUnavailable.
// Header-only; link with -lasnn_b200.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "asnn_dev.h"

namespace asnn_b200 {

using NodeId = std::uint32_t;

// ---- errors.hpp:9-55 ----------------------------------------------------------
struct InputArityMismatch : std::runtime_error { using std::runtime_error::runtime_error; };
struct OutputUnreachable : std::runtime_error { using std::runtime_error::runtime_error; };
using UnassignedOutput = OutputUnreachable;
struct LayerOutOfRange : std::out_of_range { using std::out_of_range::out_of_range; };
struct BackendUnavailable : std::runtime_error { using std::runtime_error::runtime_error; };
struct InfeasibleSpec : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
// ParseError: what() = "line N: ...", line = N (errors.hpp:31-35).
struct ParseError : std::runtime_error {
    ParseError(int line_no, const std::string& what) : std::runtime_error(what), line(line_no) {}
    int line;
};
// ValidationError: what() = "invalid network\n  ..." (errors.hpp:37-53).
struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& what) : std::runtime_error(what) {
        std::size_t p = what.find("\n  ");
        while (p != std::string::npos) {
            const std::size_t q = what.find("\n  ", p + 3);
            violations.push_back(what.substr(p + 3, q == std::string::npos ? std::string::npos : q - p - 3));
            p = q;
        }
    }
    std::vector<std::string> violations;
};

// ---- network.hpp:12-32 ---------------------------------------------------------
struct Connection {
    NodeId source = 0;
    NodeId target = 0;
    float weight = 0.0f;
};

struct Network {
    std::vector<NodeId> nodes;  // sorted ascending, unique
    std::vector<NodeId> inputs;
    std::vector<NodeId> outputs;
    std::vector<Connection> connections;
};

inline Network make_network(std::vector<NodeId> inputs, std::vector<NodeId> outputs,
                            std::vector<Connection> connections, std::vector<NodeId> extra_nodes = {}) {
    Network net;
    net.nodes = std::move(extra_nodes);
    net.nodes.insert(net.nodes.end(), inputs.begin(), inputs.end());
    net.nodes.insert(net.nodes.end(), outputs.begin(), outputs.end());
    for (const auto& c : connections) {
        net.nodes.push_back(c.source);
        net.nodes.push_back(c.target);
    }
    std::sort(net.nodes.begin(), net.nodes.end());
    net.nodes.erase(std::unique(net.nodes.begin(), net.nodes.end()), net.nodes.end());
    net.inputs = std::move(inputs);
    net.outputs = std::move(outputs);
    net.connections = std::move(connections);
    return net;
}

struct RequiredSet {
    std::vector<NodeId> members;  // sorted ascending
    bool contains(NodeId id) const { return std::binary_search(members.begin(), members.end(), id); }
};

// ---- segmentation.hpp:14-21, layout.hpp:13-37, eval.hpp:14-27 --------------------
struct LayerAssignment {
    std::vector<std::vector<NodeId>> layers;
    std::vector<NodeId> unassigned;
    std::vector<std::pair<NodeId, std::uint32_t>> index;  // (id, layer), sorted by id

    std::optional<std::uint32_t> layer_of(NodeId id) const {
        auto it = std::lower_bound(index.begin(), index.end(), id,
                                   [](const auto& e, NodeId k) { return e.first < k; });
        if (it == index.end() || it->first != id) return std::nullopt;
        return it->second;
    }
    std::size_t assigned_count() const {
        std::size_t n = 0;
        for (const auto& l : layers) n += l.size();
        return n;
    }
};

struct FlatNode {
    NodeId id = 0;
    std::uint32_t layer = 0;
    bool is_sensor = false;
    std::vector<NodeId> in_nodes;
    std::vector<float> in_weights;
    std::uint32_t num_in() const { return static_cast<std::uint32_t>(in_nodes.size()); }
};

struct LayeredLayout {
    std::uint32_t total_layers = 0;
    std::vector<std::uint32_t> nodes_per_layer;
    std::vector<FlatNode> nodes;
    std::vector<std::uint32_t> layer_offsets;
    std::vector<NodeId> input_order;
    std::uint64_t dropped_connections = 0;
    std::uint32_t id_bound = 0;
    std::uint32_t node_count() const { return static_cast<std::uint32_t>(nodes.size()); }
};

struct ActivationState {
    std::vector<float> inputs;
    std::vector<float> outputs;
};

struct ParallelConfig {
    enum class Backend { HostParallel, DeviceCompute };
    std::uint32_t workers = 0;
    Backend backend = Backend::DeviceCompute;
    std::function<void(NodeId)> node_hook;
};

// ---- device plumbing ------------------------------------------------------------------
namespace detail {

[[noreturn]] inline void raise(int rc, const asnn_dev* dev) {
    const std::string msg = dev ? asnn_dev_last_error(dev) : "no CUDA device";
    switch (rc) {
        case ASNN_E_UNAVAILABLE: throw BackendUnavailable(msg.empty() ? "no CUDA device" : msg);
        case ASNN_E_ARITY: throw InputArityMismatch(msg);
        case ASNN_E_UNASSIGNED_OUTPUT: throw OutputUnreachable(msg);
        case ASNN_E_LAYER_RANGE: throw LayerOutOfRange(msg);
        case ASNN_E_INFEASIBLE: throw InfeasibleSpec(msg);
        case ASNN_E_INVALID: throw std::invalid_argument(msg);
        case ASNN_E_VALIDATION: throw ValidationError(msg);
        case ASNN_E_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}

inline asnn_dev* device(int index = 0) {
    static std::mutex mu;
    static std::vector<asnn_dev*> devs;
    std::lock_guard<std::mutex> lk(mu);
    if (devs.size() <= static_cast<std::size_t>(index)) devs.resize(index + 1, nullptr);
    if (!devs[index]) {
        asnn_dev* d = nullptr;
        const int rc = asnn_dev_open(index, &d);
        if (rc) raise(rc, nullptr);
        devs[index] = d;
    }
    return devs[index];
}

inline void check(int rc, const asnn_dev* dev) {
    if (rc) raise(rc, dev);
}

// SoA view of a Network for the C-ABI (connections are AoS in the reference).
struct NetView {
    std::vector<NodeId> src, dst;
    std::vector<float> w;
    asnn_network_desc d{};
    explicit NetView(const Network& n) {
        src.reserve(n.connections.size());
        dst.reserve(n.connections.size());
        w.reserve(n.connections.size());
        for (const auto& c : n.connections) {
            src.push_back(c.source);
            dst.push_back(c.target);
            w.push_back(c.weight);
        }
        d.n_nodes = static_cast<std::uint32_t>(n.nodes.size());
        d.nodes = n.nodes.data();
        d.n_inputs = static_cast<std::uint32_t>(n.inputs.size());
        d.inputs = n.inputs.data();
        d.n_outputs = static_cast<std::uint32_t>(n.outputs.size());
        d.outputs = n.outputs.data();
        d.n_connections = n.connections.size();
        d.source = src.data();
        d.target = dst.data();
        d.weight = w.data();
    }
};

}  // namespace detail

// ---- io.hpp:23-31: loading, parsed and validated on the device -------------------------
namespace detail {
inline Network network_from_corpus(asnn_corpus* c) {
    asnn_network_desc d{};
    asnn_corpus_desc(c, &d);
    Network net;
    net.nodes.assign(d.nodes, d.nodes + d.n_nodes);
    net.inputs.assign(d.inputs, d.inputs + d.n_inputs);
    net.outputs.assign(d.outputs, d.outputs + d.n_outputs);
    net.connections.resize(d.n_connections);
    for (std::uint64_t k = 0; k < d.n_connections; ++k)
        net.connections[k] = Connection{d.source[k], d.target[k], d.weight[k]};
    asnn_corpus_free(c);
    return net;
}
inline Network load(int rc, asnn_dev* dev, asnn_corpus* c, std::uint32_t line) {
    if (rc == ASNN_E_PARSE) throw ParseError(static_cast<int>(line), asnn_dev_last_error(dev));
    check(rc, dev);
    return network_from_corpus(c);
}
}  // namespace detail

inline Network parse_network(std::string_view text) {
    asnn_dev* dev = detail::device();
    asnn_corpus* c = nullptr;
    std::uint32_t line = 0;
    const int rc = asnn_dev_parse_network(dev, text.data(), text.size(), &c, &line);
    return detail::load(rc, dev, c, line);
}

// network.hpp:60-98: validate (all violations, the reference's order and
// wording) and normalize, both on the device.
struct ValidationReport {
    std::vector<std::string> violations;
    bool ok() const { return violations.empty(); }
    const std::vector<std::string>& messages() const { return violations; }
};

inline ValidationReport validate(const Network& net) {
    asnn_dev* dev = detail::device();
    detail::NetView v(net);
    std::uint32_t n = 0;
    std::string buf(1u << 20, '\0');
    detail::check(asnn_dev_validate(dev, &v.d, buf.data(), buf.size(), &n), dev);
    ValidationReport r;
    if (n) {
        std::string all(buf.c_str());
        std::size_t p = 0;
        for (;;) {
            const std::size_t q = all.find('\n', p);
            r.violations.push_back(all.substr(p, q == std::string::npos ? std::string::npos : q - p));
            if (q == std::string::npos) break;
            p = q + 1;
        }
    }
    return r;
}

inline Network normalize(const Network& net) {
    asnn_dev* dev = detail::device();
    detail::NetView v(net);
    asnn_corpus* c = nullptr;
    detail::check(asnn_dev_normalize(dev, &v.d, &c), dev);
    return detail::network_from_corpus(c);
}

inline Network read_network(const std::string& path) {
    asnn_dev* dev = detail::device();
    asnn_corpus* c = nullptr;
    std::uint32_t line = 0;
    const int rc = asnn_dev_read_network(dev, path.c_str(), &c, &line);
    return detail::load(rc, dev, c, line);
}

// ---- the path ---------------------------------------------------------------------------
inline RequiredSet compute_required(const Network& net) {
    asnn_dev* dev = detail::device();
    detail::NetView v(net);
    std::vector<std::uint8_t> mask(net.nodes.size());
    detail::check(asnn_dev_compute_required(dev, &v.d, mask.data()), dev);
    RequiredSet r;
    for (std::size_t i = 0; i < mask.size(); ++i)
        if (mask[i]) r.members.push_back(net.nodes[i]);
    return r;
}

inline LayerAssignment segment(const Network& net, const RequiredSet& required) {
    asnn_dev* dev = detail::device();
    detail::NetView v(net);
    std::vector<std::uint8_t> mask(net.nodes.size());
    for (std::size_t i = 0; i < net.nodes.size(); ++i) mask[i] = required.contains(net.nodes[i]);
    std::vector<std::uint32_t> level(net.nodes.size());
    std::uint32_t n_layers = 0;
    detail::check(asnn_dev_segment(dev, &v.d, mask.data(), level.data(), &n_layers), dev);
    LayerAssignment a;
    a.layers.resize(n_layers);
    for (std::size_t i = 0; i < net.nodes.size(); ++i) {  // nodes are id-sorted: layers stay sorted
        if (level[i] == ASNN_UNASSIGNED) a.unassigned.push_back(net.nodes[i]);
        else {
            a.layers[level[i]].push_back(net.nodes[i]);
            a.index.emplace_back(net.nodes[i], level[i]);
        }
    }
    return a;
}

inline std::size_t depth(const LayerAssignment& a) { return a.layers.size(); }

inline std::vector<NodeId> unassigned_outputs(const Network& net, const LayerAssignment& a) {
    std::vector<NodeId> missing;
    for (NodeId id : net.outputs)
        if (!a.layer_of(id)) missing.push_back(id);
    return missing;
}

// Device-resident layout (build once, activate many batches).
class DeviceNetwork {
public:
    explicit DeviceNetwork(const Network& net, int device = 0) : dev_(detail::device(device)) {
        detail::NetView v(net);
        detail::check(asnn_dev_build_layout(dev_, &v.d, &h_), dev_);
        detail::check(asnn_dev_layout_info(h_, &info_), dev_);
    }
    DeviceNetwork(const DeviceNetwork&) = delete;
    DeviceNetwork& operator=(const DeviceNetwork&) = delete;
    ~DeviceNetwork() { asnn_dev_free_layout(h_); }

    const asnn_layout_info& info() const { return info_; }

    // X: n_vec vectors of n_inputs floats; returns n_vec x n_outputs (read_outputs order).
    std::vector<float> activate(std::span<const float> X, std::uint32_t n_vec) {
        std::vector<float> out(static_cast<std::size_t>(n_vec) * info_.n_outputs);
        detail::check(asnn_dev_activate(h_, X.data(), n_vec, X.size(), out.data(), nullptr), dev_);
        return out;
    }

    LayeredLayout download() const {
        asnn_layout_info ni{};
        detail::check(asnn_dev_network_info(h_, 0, &ni), dev_);
        std::vector<std::uint32_t> lo(ni.total_layers + 1), ids(ni.node_count), in(ni.edge_count),
            io(ni.n_inputs);
        std::vector<std::uint64_t> rp(ni.node_count + 1);
        std::vector<float> w(ni.edge_count);
        detail::check(asnn_dev_layout_download(h_, 0, lo.data(), ids.data(), rp.data(), in.data(),
                                               w.data(), io.data()),
                      dev_);
        LayeredLayout L;
        L.total_layers = ni.total_layers;
        L.layer_offsets = lo;
        for (std::uint32_t l = 0; l < ni.total_layers; ++l) L.nodes_per_layer.push_back(lo[l + 1] - lo[l]);
        L.nodes.resize(ni.node_count);
        std::uint32_t layer = 0;
        for (std::uint32_t p = 0; p < ni.node_count; ++p) {
            while (layer + 1 < ni.total_layers && p >= lo[layer + 1]) ++layer;
            FlatNode& n = L.nodes[p];
            n.id = ids[p];
            n.layer = layer;
            n.is_sensor = layer == 0;
            n.in_nodes.assign(in.begin() + rp[p], in.begin() + rp[p + 1]);
            n.in_weights.assign(w.begin() + rp[p], w.begin() + rp[p + 1]);
        }
        L.input_order = io;
        L.dropped_connections = ni.dropped_connections;
        L.id_bound = ni.id_bound;
        return L;
    }

private:
    asnn_dev* dev_;
    asnn_dev_layout* h_ = nullptr;
    asnn_layout_info info_{};
};

// Multi-GPU (csrc/group.cu): one process driving several
// devices.  Batch sharding: a layout replica per device, each sweeps a
// contiguous slice of the vectors; population sharding: a contiguous slice of
// the networks per device.  The declared outputs are all-gathered on the
// devices (NCCL, or the copy engines when a device is listed twice).
class DeviceGroup {
public:
    explicit DeviceGroup(const std::vector<int>& devices) {
        const int rc = asnn_group_open(devices.data(), static_cast<std::uint32_t>(devices.size()), &g_);
        if (rc) detail::raise(rc, nullptr);
    }
    DeviceGroup(const DeviceGroup&) = delete;
    DeviceGroup& operator=(const DeviceGroup&) = delete;
    ~DeviceGroup() { asnn_group_close(g_); }
    asnn_group* handle() const { return g_; }
    // "single device", "nccl" or "copy engines"
    std::string gather() const {
        std::uint32_t n = 0, k = 0;
        asnn_group_info(g_, &n, &k);
        return k == 1 ? "nccl" : k == 2 ? "copy engines" : "single device";
    }
    void check(int rc) const {
        if (!rc) return;
        const std::string msg = asnn_group_last_error(g_);
        switch (rc) {
            case ASNN_E_ARITY: throw InputArityMismatch(msg);
            case ASNN_E_UNASSIGNED_OUTPUT: throw OutputUnreachable(msg);
            case ASNN_E_UNAVAILABLE: throw BackendUnavailable(msg);
            case ASNN_E_INVALID: throw std::invalid_argument(msg);
            default: throw DeviceError(msg);
        }
    }

private:
    asnn_group* g_ = nullptr;
};

class GroupNetwork {
public:
    // batch sharding of one network
    GroupNetwork(DeviceGroup& grp, const Network& net) : grp_(grp) {
        detail::NetView v(net);
        grp_.check(asnn_group_build_layout(grp_.handle(), &v.d, &h_));
        n_in_ = static_cast<std::uint32_t>(net.inputs.size());
        n_out_ = static_cast<std::uint32_t>(net.outputs.size());
    }
    // population sharding
    GroupNetwork(DeviceGroup& grp, const std::vector<Network>& nets) : grp_(grp), population_(true) {
        std::vector<detail::NetView> views;
        views.reserve(nets.size());
        std::vector<asnn_network_desc> d;
        for (const auto& n : nets) {
            views.emplace_back(n);
            d.push_back(views.back().d);
            n_in_ += static_cast<std::uint32_t>(n.inputs.size());
            n_out_ += static_cast<std::uint32_t>(n.outputs.size());
        }
        grp_.check(asnn_group_build_population(grp_.handle(), static_cast<std::uint32_t>(nets.size()),
                                               d.data(), &h_));
    }
    GroupNetwork(const GroupNetwork&) = delete;
    GroupNetwork& operator=(const GroupNetwork&) = delete;
    ~GroupNetwork() { asnn_group_free_layout(h_); }

    // X: n_vec vectors per network (networks concatenated for a population);
    // returns the declared outputs, [n_vec][n_outputs] per network.
    std::vector<float> activate(std::span<const float> X, std::uint32_t n_vec) {
        std::vector<float> out(static_cast<std::size_t>(n_vec) * n_out_);
        grp_.check(asnn_group_activate(h_, X.data(), n_vec, X.size(), out.data(), nullptr));
        return out;
    }

private:
    DeviceGroup& grp_;
    bool population_ = false;
    asnn_group_layout* h_ = nullptr;
    std::uint32_t n_in_ = 0, n_out_ = 0;
};

// layout.cpp:12-83.  The assignment must be segment()'s for this network
// (the device rebuilds it); UnassignedOutput when an output has no layer.
inline LayeredLayout flatten(const Network& net, const LayerAssignment& assignment) {
    if (auto missing = unassigned_outputs(net, assignment); !missing.empty()) {
        std::string msg = "unassigned output node(s):";
        for (NodeId id : missing) msg += ' ' + std::to_string(id);
        throw UnassignedOutput(msg);
    }
    return DeviceNetwork(net).download();
}

inline std::pair<std::uint32_t, std::uint32_t> layer_slice_bounds(const LayeredLayout& layout,
                                                                  std::uint32_t layer) {
    if (layer >= layout.total_layers)
        throw LayerOutOfRange("layer " + std::to_string(layer) + " out of range, total layers " +
                              std::to_string(layout.total_layers));
    return {layout.layer_offsets[layer], layout.nodes_per_layer[layer]};
}

inline std::uint32_t max_layer_width(const LayeredLayout& layout) {
    std::uint32_t w = 0;
    for (std::uint32_t c : layout.nodes_per_layer) w = std::max(w, c);
    return w;
}

// eval.cpp:49-80 with Backend::DeviceCompute: the layout is staged straight
// into a per-thread page-locked buffer and evaluated by one kernel on the
// id-indexed state (asnn_eval_buf, once.cu); nothing stays on the device.
inline ActivationState eval_parallel(const LayeredLayout& layout, std::span<const float> input_values,
                                     const ParallelConfig& cfg = {}) {
    if (cfg.backend != ParallelConfig::Backend::DeviceCompute)
        throw BackendUnavailable("this engine implements Backend::DeviceCompute only");
    if (cfg.node_hook) throw BackendUnavailable("node_hook cannot run per node on the device");
    if (input_values.size() != layout.input_order.size())
        throw InputArityMismatch("expected " + std::to_string(layout.input_order.size()) +
                                 " input values, got " + std::to_string(input_values.size()));
    asnn_dev* dev = detail::device();
    struct Buf {
        asnn_eval_buf* b = nullptr;
        ~Buf() { asnn_eval_buf_free(b); }
    };
    thread_local Buf buf;
    if (!buf.b) detail::check(asnn_eval_buf_create(dev, &buf.b), dev);
    ActivationState st;  // make_state (eval.cpp:29-33)
    st.inputs.assign(layout.id_bound, 0.0f);
    for (std::size_t i = 0; i < input_values.size(); ++i) st.inputs[layout.input_order[i]] = input_values[i];
    std::uint64_t edges = 0;
    for (const FlatNode& n : layout.nodes) edges += n.in_nodes.size();
    asnn_eval_dims dims{};
    dims.total_layers = layout.total_layers;
    dims.node_count = static_cast<std::uint32_t>(layout.nodes.size());
    dims.sensor_count = layout.total_layers ? layout.nodes_per_layer[0] : 0;
    dims.id_bound = layout.id_bound;
    dims.edge_count = edges;
    asnn_eval_stage s{};
    detail::check(asnn_eval_buf_stage(buf.b, &dims, &s), dev);
    std::copy(layout.layer_offsets.begin(), layout.layer_offsets.end(), s.layer_offsets);
    std::uint32_t at = 0;
    for (std::size_t k = 0; k < layout.nodes.size(); ++k) {
        const FlatNode& n = layout.nodes[k];
        s.node_ids[k] = n.id;
        s.row_ptr[k] = at;
        std::copy(n.in_nodes.begin(), n.in_nodes.end(), s.in_nodes + at);
        std::copy(n.in_weights.begin(), n.in_weights.end(), s.in_weights + at);
        at += static_cast<std::uint32_t>(n.in_nodes.size());
    }
    s.row_ptr[layout.nodes.size()] = at;
    for (std::uint32_t k = 0; k < dims.sensor_count; ++k) {
        const NodeId id = layout.nodes[k].id;
        s.sensor_inputs[k] = id < layout.id_bound ? st.inputs[id] : 0.0f;
    }
    st.outputs.resize(layout.id_bound);
    detail::check(asnn_eval_buf_run(buf.b, st.outputs.data()), dev);
    return st;
}

inline std::vector<float> read_outputs(const ActivationState& state, const Network& net) {
    std::vector<float> out;
    out.reserve(net.outputs.size());
    for (NodeId id : net.outputs) out.push_back(state.outputs[id]);
    return out;
}

}  // namespace asnn_b200
