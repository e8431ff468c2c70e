// integration/asnn_device_backend.cpp
//
// The reference-side binding a maintainer adds to /root/reference/proj to
// serve ParallelConfig::Backend::DeviceCompute (eval.hpp:20) with the B200
// engine.  It is compiled against the reference's own headers; the only
// change to the reference itself is the two-line branch at eval.cpp:51-52
// shown in INTEGRATION.md.  It converts the reference's LayeredLayout
// (layout.hpp:27-37) into the C-ABI's page-locked staging (asnn_eval_buf,
// once.cu) on every call (the reference mutates layouts in place between evaluations,
// asnn_main.cpp:264-278), activates one vector and maps status codes back to
// the reference's exception types (errors.hpp:9-55).
//
// Built here into oracle/_ref/libasnn_ref_dev.so (oracle/Makefile) so the GPU
// tests can run the reference's own evaluators and this backend side by side.
#include <chrono>
#include <omp.h>
#include <algorithm>
#include <cmath>
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

}  // namespace

// One device handle per process (device 0), opened on first use.
asnn_dev* device() {
    static std::once_flag once;
    static asnn_dev* dev = nullptr;
    static int rc = ASNN_OK;
    std::call_once(once, [] { rc = asnn_dev_open(0, &dev); });
    if (rc != ASNN_OK) raise(rc, nullptr);
    return dev;
}

// Phase clock of eval_device for tools/once_probe.py (off unless enabled by
// ref_dev_phase_clock): make_state, sizes, staging fill, device run.
namespace {
struct PhaseClock {
    bool on = false;
    double acc[4] = {0, 0, 0, 0};
    std::chrono::steady_clock::time_point t;
    void start() {
        if (on) t = std::chrono::steady_clock::now();
    }
    void lap(int i) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        acc[i] += std::chrono::duration<double, std::micro>(n - t).count();
        t = n;
    }
};
thread_local PhaseClock phase_clock;
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
    // one page-locked staging buffer per calling thread (once.cu): the
    // LayeredLayout's AoS nodes are written straight into it, no copy between
    struct Buf {
        asnn_eval_buf* b = nullptr;
        ~Buf() { asnn_eval_buf_free(b); }
    };
    thread_local Buf buf;
    if (!buf.b) {
        const int rc = asnn_eval_buf_create(dev, &buf.b);
        if (rc) raise(rc, dev);
    }
    const std::size_t N = layout.nodes.size();
    phase_clock.start();
    // make_state (eval.cpp:29-33)
    ActivationState state;
    state.inputs.assign(layout.id_bound, 0.0f);
    for (std::size_t i = 0; i < input_values.size(); ++i)
        state.inputs[layout.input_order[i]] = input_values[i];
    phase_clock.lap(0);
    asnn_eval_dims dims{};
    dims.total_layers = layout.total_layers;
    dims.node_count = static_cast<std::uint32_t>(N);
    dims.sensor_count = layout.total_layers ? layout.nodes_per_layer[0] : 0;
    dims.id_bound = layout.id_bound;
    // LayeredLayout -> CSR (layout.hpp:13-37).  Large layouts are converted by
    // all host threads: per-chunk edge totals, then each chunk writes its
    // row_ptr run and copies its nodes' predecessors.
    const std::int64_t n64 = static_cast<std::int64_t>(N);
    const int nt = N >= 4096 ? std::max(1, omp_get_max_threads()) : 1;
    std::vector<std::uint64_t> part(nt + 1, 0);
    auto chunk = [&](int i) { return n64 * i / nt; };
#pragma omp parallel num_threads(nt) if (nt > 1)
    {
        const int i = nt > 1 ? omp_get_thread_num() : 0;
        std::uint64_t e = 0;
        for (std::int64_t k = chunk(i); k < chunk(i + 1); ++k) e += layout.nodes[k].in_nodes.size();
        part[i + 1] = e;
    }
    for (int i = 0; i < nt; ++i) part[i + 1] += part[i];
    const std::uint64_t edges = part[nt];
    dims.edge_count = edges;
    asnn_eval_stage s{};
    phase_clock.lap(1);
    int rc = asnn_eval_buf_stage(buf.b, &dims, &s);
    if (rc) raise(rc, dev);
    std::copy(layout.layer_offsets.begin(), layout.layer_offsets.end(), s.layer_offsets);
#pragma omp parallel num_threads(nt) if (nt > 1)
    {
        const int i = nt > 1 ? omp_get_thread_num() : 0;
        auto at = static_cast<std::uint32_t>(part[i]);
        for (std::int64_t k = chunk(i); k < chunk(i + 1); ++k) {
            const FlatNode& n = layout.nodes[k];
            s.node_ids[k] = n.id;
            s.row_ptr[k] = at;
            std::copy(n.in_nodes.begin(), n.in_nodes.end(), s.in_nodes + at);
            std::copy(n.in_weights.begin(), n.in_weights.end(), s.in_weights + at);
            at += static_cast<std::uint32_t>(n.in_nodes.size());
        }
    }
    s.row_ptr[N] = static_cast<std::uint32_t>(edges);
    for (std::uint32_t k = 0; k < dims.sensor_count; ++k) {
        const NodeId id = layout.nodes[k].id;
        s.sensor_inputs[k] = id < layout.id_bound ? state.inputs[id] : 0.0f;
    }
    state.outputs.resize(layout.id_bound);
    phase_clock.lap(2);
    rc = asnn_eval_buf_run(buf.b, state.outputs.data());
    if (rc) raise(rc, dev);
    phase_clock.lap(3);
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

// Timing hooks for tools/bench_csv.py (the reference's bench protocol with
// device rows, bench.cpp:41-100): mean / sample stddev in microseconds of
// `reps` calls after `warmup`, timed inside C++ like the reference's own
// sequential / parallel rows.  "per call" = the drop-in eval_parallel
// (DeviceCompute): conversion + upload + activate + state back + free every
// call; "resident" = asnn_dev_activate on a layout uploaded once (state back).
namespace {
void stats_us(const std::vector<double>& s, double* mean, double* sd) {
    double m = 0;
    for (double v : s) m += v;
    m /= s.size();
    double q = 0;
    for (double v : s) q += (v - m) * (v - m);
    *mean = m;
    *sd = s.size() > 1 ? std::sqrt(q / (s.size() - 1)) : 0.0;
}
}  // namespace

extern "C" void ref_dev_phase_clock(int on, double* acc4) {
    if (acc4)
        for (int i = 0; i < 4; ++i) acc4[i] = asnn::phase_clock.acc[i];
    asnn::phase_clock = asnn::PhaseClock{};
    asnn::phase_clock.on = on != 0;
}

extern "C" int ref_dev_eval_timed(const asnn::LayeredLayout* layout, const float* x, std::uint32_t n_x,
                                  std::uint32_t warmup, std::uint32_t reps, double* mean_us, double* sd_us) {
    try {
        asnn::ParallelConfig cfg;
        cfg.backend = asnn::ParallelConfig::Backend::DeviceCompute;
        std::span<const float> xs(x, n_x);
        for (std::uint32_t i = 0; i < warmup; ++i) (void)asnn::eval_device(*layout, xs, cfg);
        std::vector<double> s;
        for (std::uint32_t i = 0; i < reps; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            auto st = asnn::eval_device(*layout, xs, cfg);
            s.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
        }
        stats_us(s, mean_us, sd_us);
        return 0;
    } catch (...) {
        return 6;
    }
}

extern "C" int ref_dev_resident_timed(const asnn::LayeredLayout* layout, const float* x, std::uint32_t n_x,
                                      std::uint32_t warmup, std::uint32_t reps, double* mean_us, double* sd_us) {
    asnn_dev* dev = asnn::device();
    std::vector<std::uint32_t> ids(layout->nodes.size()), in;
    std::vector<std::uint64_t> rp(layout->nodes.size() + 1, 0);
    std::vector<float> w;
    for (std::size_t k = 0; k < layout->nodes.size(); ++k) {
        ids[k] = layout->nodes[k].id;
        in.insert(in.end(), layout->nodes[k].in_nodes.begin(), layout->nodes[k].in_nodes.end());
        w.insert(w.end(), layout->nodes[k].in_weights.begin(), layout->nodes[k].in_weights.end());
        rp[k + 1] = in.size();
    }
    asnn_layout_desc d{};
    d.total_layers = layout->total_layers;
    d.layer_offsets = layout->layer_offsets.data();
    d.node_count = static_cast<std::uint32_t>(layout->nodes.size());
    d.node_ids = ids.data();
    d.row_ptr = rp.data();
    d.in_nodes = in.data();
    d.in_weights = w.data();
    d.n_inputs = static_cast<std::uint32_t>(layout->input_order.size());
    d.input_order = layout->input_order.data();
    d.id_bound = layout->id_bound;
    asnn_dev_layout* dl = nullptr;
    if (asnn_dev_upload_layout(dev, &d, &dl)) return 6;
    std::vector<float> state(layout->id_bound);
    int rc = 0;
    for (std::uint32_t i = 0; i < warmup + 2 && !rc; ++i)  // the 2nd call captures the sweep graph
        rc = asnn_dev_activate(dl, x, 1, n_x, nullptr, state.data());
    std::vector<double> s;
    for (std::uint32_t i = 0; i < reps && !rc; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        rc = asnn_dev_activate(dl, x, 1, n_x, nullptr, state.data());
        s.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    asnn_dev_free_layout(dl);
    if (rc) return rc;
    stats_us(s, mean_us, sd_us);
    return 0;
}

// Resident server row (tools/bench_csv.py "device_server"): the layout uploaded
// once and held by the persistent server kernel (asnn_dev_server_*), one
// vector per request, the declared outputs back (read_outputs, eval.cpp:82-87).
extern "C" int ref_dev_server_timed(const asnn::LayeredLayout* layout, const std::uint32_t* outputs,
                                    std::uint32_t n_out, const float* x, std::uint32_t n_x, std::uint32_t warmup,
                                    std::uint32_t reps, double* mean_us, double* sd_us) {
    asnn_dev* dev = asnn::device();
    std::vector<std::uint32_t> ids(layout->nodes.size()), in;
    std::vector<std::uint64_t> rp(layout->nodes.size() + 1, 0);
    std::vector<float> w;
    for (std::size_t k = 0; k < layout->nodes.size(); ++k) {
        ids[k] = layout->nodes[k].id;
        in.insert(in.end(), layout->nodes[k].in_nodes.begin(), layout->nodes[k].in_nodes.end());
        w.insert(w.end(), layout->nodes[k].in_weights.begin(), layout->nodes[k].in_weights.end());
        rp[k + 1] = in.size();
    }
    asnn_layout_desc d{};
    d.total_layers = layout->total_layers;
    d.layer_offsets = layout->layer_offsets.data();
    d.node_count = static_cast<std::uint32_t>(layout->nodes.size());
    d.node_ids = ids.data();
    d.row_ptr = rp.data();
    d.in_nodes = in.data();
    d.in_weights = w.data();
    d.n_inputs = static_cast<std::uint32_t>(layout->input_order.size());
    d.input_order = layout->input_order.data();
    d.n_outputs = n_out;
    d.outputs = outputs;
    d.id_bound = layout->id_bound;
    asnn_dev_layout* dl = nullptr;
    if (asnn_dev_upload_layout(dev, &d, &dl)) return 6;
    asnn_dev_server* srv = nullptr;
    int rc = asnn_dev_server_start(dl, 1, &srv);
    if (rc) {
        asnn_dev_free_layout(dl);
        return rc == ASNN_E_UNAVAILABLE ? 1 : 6;
    }
    std::vector<float> out(std::max<std::uint32_t>(1, n_out));
    for (std::uint32_t i = 0; i < warmup + 2 && !rc; ++i) rc = asnn_dev_server_activate(srv, x, 1, n_x, out.data());
    std::vector<double> s;
    for (std::uint32_t i = 0; i < reps && !rc; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        rc = asnn_dev_server_activate(srv, x, 1, n_x, out.data());
        s.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    asnn_dev_server_stop(srv);
    asnn_dev_free_layout(dl);
    if (rc) return 6;
    stats_us(s, mean_us, sd_us);
    return 0;
}
