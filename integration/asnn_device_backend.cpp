// integration/asnn_device_backend.cpp
//
// The reference-side binding a maintainer adds to /root/reference/proj to
// serve ParallelConfig::Backend::DeviceCompute (eval.hpp:20) with the B200
// engine.  It is compiled against the reference's own headers; the only
// change to the reference itself is the two-line branch at eval.cpp:51-52
// shown in INTEGRATION.md.  It converts the reference's LayeredLayout
// (layout.hpp:27-37) to the C-ABI's asnn_layout_desc, uploads it on every
// call (the reference mutates layouts in place between evaluations,
// asnn_main.cpp:264-278), activates one vector and maps status codes back to
// the reference's exception types (errors.hpp:9-55).
//
// Built here into oracle/_ref/libasnn_ref_dev.so (oracle/Makefile) so the GPU
// tests can run the reference's own evaluators and this backend side by side.
#include <cstdint>
#include <mutex>
#include <span>
#include <string>
#include <vector>

#include "asnn/errors.hpp"
#include "asnn/eval.hpp"
#include "asnn/layout.hpp"
#include "asnn_dev.h"

namespace asnn {

namespace {

[[noreturn]] void raise(int rc, asnn_dev* dev) {
    const std::string msg = dev ? asnn_dev_last_error(dev) : "device-compute backend unavailable";
    switch (rc) {
        case ASNN_E_ARITY: throw InputArityMismatch(msg);
        case ASNN_E_UNASSIGNED_OUTPUT: throw UnassignedOutput(msg);
        case ASNN_E_LAYER_RANGE: throw LayerOutOfRange(msg);
        case ASNN_E_UNAVAILABLE: throw BackendUnavailable(msg);
        default: throw std::runtime_error("asnn device backend: " + msg);
    }
}

// One device handle per process (device 0), opened on first use.
asnn_dev* device() {
    static std::once_flag once;
    static asnn_dev* dev = nullptr;
    static int rc = ASNN_OK;
    std::call_once(once, [] { rc = asnn_dev_open(0, &dev); });
    if (rc != ASNN_OK) raise(rc, nullptr);
    return dev;
}

}  // namespace

// eval_parallel(..., Backend::DeviceCompute): same contract as eval.cpp:49-80.
ActivationState eval_device(const LayeredLayout& layout, std::span<const float> input_values,
                            const ParallelConfig& cfg) {
    if (cfg.node_hook)
        throw BackendUnavailable("node_hook cannot run per node on the device-compute backend");
    if (input_values.size() != layout.input_order.size())  // eval.cpp:26-28
        throw InputArityMismatch("expected " + std::to_string(layout.input_order.size()) +
                                 " input values, got " + std::to_string(input_values.size()));
    asnn_dev* dev = device();

    // LayeredLayout -> CSR (layout.hpp:13-37)
    std::vector<std::uint32_t> ids(layout.nodes.size());
    std::vector<std::uint64_t> row_ptr(layout.nodes.size() + 1, 0);
    std::size_t edges = 0;
    for (const FlatNode& n : layout.nodes) edges += n.in_nodes.size();
    std::vector<std::uint32_t> in_nodes;
    std::vector<float> in_weights;
    in_nodes.reserve(edges);
    in_weights.reserve(edges);
    for (std::size_t k = 0; k < layout.nodes.size(); ++k) {
        const FlatNode& n = layout.nodes[k];
        ids[k] = n.id;
        in_nodes.insert(in_nodes.end(), n.in_nodes.begin(), n.in_nodes.end());
        in_weights.insert(in_weights.end(), n.in_weights.begin(), n.in_weights.end());
        row_ptr[k + 1] = in_nodes.size();
    }
    asnn_layout_desc d{};
    d.total_layers = layout.total_layers;
    d.layer_offsets = layout.layer_offsets.data();
    d.node_count = static_cast<std::uint32_t>(layout.nodes.size());
    d.node_ids = ids.data();
    d.row_ptr = row_ptr.data();
    d.in_nodes = in_nodes.data();
    d.in_weights = in_weights.data();
    d.n_inputs = static_cast<std::uint32_t>(layout.input_order.size());
    d.input_order = layout.input_order.data();
    d.id_bound = layout.id_bound;

    asnn_dev_layout* dl = nullptr;
    int rc = asnn_dev_upload_layout(dev, &d, &dl);
    if (rc) raise(rc, dev);
    ActivationState state;
    state.inputs.assign(layout.id_bound, 0.0f);  // make_state, eval.cpp:29-33
    for (std::size_t i = 0; i < input_values.size(); ++i)
        state.inputs[layout.input_order[i]] = input_values[i];
    state.outputs.assign(layout.id_bound, 0.0f);
    rc = asnn_dev_activate(dl, input_values.data(), 1, input_values.size(), nullptr,
                           state.outputs.data());
    asnn_dev_free_layout(dl);
    if (rc) raise(rc, dev);
    return state;
}

}  // namespace asnn

// ---- test hook (oracle/_ref/libasnn_ref_dev.so only) ---------------------------
// Runs eval_device on a reference LayeredLayout built by ref_shim.cpp.
extern "C" int ref_dev_eval(const asnn::LayeredLayout* layout, const float* x, std::uint32_t n_x,
                            float* state_out) {
    try {
        asnn::ParallelConfig cfg;
        cfg.backend = asnn::ParallelConfig::Backend::DeviceCompute;
        auto st = asnn::eval_device(*layout, std::span<const float>(x, n_x), cfg);
        std::copy(st.outputs.begin(), st.outputs.end(), state_out);
        return 0;
    } catch (const asnn::InputArityMismatch&) {
        return 2;
    } catch (const asnn::BackendUnavailable&) {
        return 1;
    } catch (...) {
        return 6;
    }
}
