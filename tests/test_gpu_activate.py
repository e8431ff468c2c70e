"""Parity of the device activation path (asnn_dev_upload_layout +
asnn_dev_activate, i.e. eval_parallel with Backend::DeviceCompute) against
the oracle and the reference-generated golden vectors.

Tolerance (BASELINE.json north_star): every value within 1e-5 relative of the
reference (denormal clamp values: 1e-5 absolute), plus the reference's own
`verify` criterion, absolute 1e-5 (asnn_main.cpp:281-284).  The kernels keep
the reference's summation order, so values are expected to be bitwise equal
except where CUDA's double exp and glibc's differ in the last bit (SURVEY.md
7.2-2); the bitwise-equal fraction is asserted >= 99.9%."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from conftest import bitwise_equal, rel_close

pytestmark = pytest.mark.gpu
DEV = A.ParallelConfig(backend=A.Backend.DeviceCompute)


@pytest.fixture(params=[1, 2, 3, 4, 5], ids=["layer-launches", "k_cta", "whole-rows", "k_cta-window",
                                              "k_chain-window"])
def sweep_mode(request):
    """Run a test under every sweep strategy: one launch per dependency level
    (heavy rows split into segments where eligible), the one-CTA-per-slice
    sweep (k_cta / k_chain), per-level launches of whole rows (k_rows/k_level +
    k_heavy), the windowed k_cta (a ring of the newest positions in shared
    memory, older sources from A) with its smallest ring, and the windowed
    k_chain (chain.cuh WIN, forced on single networks)."""
    dev = A.Device.get(0)
    dev.set_sweep_mode(request.param)
    yield request.param
    dev.set_sweep_mode(0)


def to_layout(d: dict, outputs=()) -> A.LayeredLayout:
    return A.LayeredLayout(d["total_layers"], d["layer_offsets"], d["node_ids"], d["row_ptr"],
                           d["in_nodes"], d["in_weights"], d["input_order"],
                           d["dropped_connections"], d["id_bound"], np.asarray(outputs, np.uint32))


def check_close(g: np.ndarray, r: np.ndarray, stats: dict):
    assert g.shape == r.shape
    ok = rel_close(g, r)
    assert ok.all(), f"{(~ok).sum()} values beyond 1e-5 relative; worst " \
                     f"{np.max(np.abs(g.astype(np.float64) - r)):.3g}"
    assert np.max(np.abs(g.astype(np.float64) - r.astype(np.float64))) <= 1e-5
    stats["n"] = stats.get("n", 0) + g.size
    stats["eq"] = stats.get("eq", 0) + int((g.view(np.uint32) == r.view(np.uint32)).sum())


# --- hand-traced fixtures (test_eval.cpp) ------------------------------------------
def test_single_edge(oracle):
    net = A.make_network([0], [1], [(0, 1, 1.0)])
    lay = to_layout(oracle.layout(net))
    st = A.eval_parallel(lay, [0.0], DEV)
    assert st.outputs[0] == np.float32(0.5)
    assert abs(float(st.outputs[1]) - 0.9230835512325639) < 1e-6


def test_zero_weights_force_half(oracle):
    rng = A.SplitMix64(51)
    spec = A.random_spec(rng, 40, 200)
    spec.weight_min = spec.weight_max = 0.0
    net = A.generate(spec)
    d = oracle.layout(net)
    st = A.eval_parallel(to_layout(d), np.full(len(net.inputs), 0.3, np.float32), DEV)
    non_sensor = d["node_ids"][d["layer_offsets"][1]:]
    assert np.all(st.outputs[non_sensor] == np.float32(0.5))


def test_cancellation_and_sensors(oracle):
    lay = to_layout(oracle.layout(A.make_network([0, 1], [2], [(0, 2, 1.0), (1, 2, -1.0)])))
    for x in (0.0, 0.7, -1.3):
        assert A.eval_parallel(lay, [x, x], DEV).outputs[2] == np.float32(0.5)
    lay = to_layout(oracle.layout(A.make_network([0, 1], [2], [(0, 2, 0.5), (1, 2, -0.25)])))
    st = A.eval_parallel(lay, [1.0, -1.0], DEV)
    assert abs(float(st.outputs[0]) - 0.9931047268673539) < 1e-6
    assert abs(float(st.outputs[1]) - 0.0068952731326461) < 1e-8
    assert st.inputs[0] == 1.0 and st.inputs[1] == -1.0


def test_skip_fixture_matches_oracle_bitwise(oracle):
    net = A.make_network([0], [3], [(0, 1, 1.0), (0, 2, 0.5), (1, 2, -1.0), (2, 3, 0.75),
                                    (0, 3, 0.25)])
    d = oracle.layout(net)
    st = A.eval_parallel(to_layout(d), [0.4], DEV)
    assert bitwise_equal(st.outputs, oracle.eval_batch(d, np.array([0.4], np.float32))[0])


def test_output_and_input_order(oracle):
    net = A.make_network([0, 1], [4, 3], [(0, 3, 1.0), (1, 4, 1.0), (0, 4, 0.5)])
    d = oracle.layout(net)
    st = A.eval_parallel(to_layout(d), [0.2, -0.9], DEV)
    outs = A.read_outputs(st, net)
    assert outs[0] == st.outputs[4] and outs[1] == st.outputs[3]
    # device-side read_outputs through the resident layout agrees
    dl = A.DeviceLayout.from_layout(to_layout(d, net.outputs))
    out, _ = dl.activate(np.array([[0.2, -0.9]], np.float32))
    assert bitwise_equal(out[0], outs)
    net = A.Network([0, 1, 2], [1, 0], [2], [0, 1], [2, 2], [1.0, 1.0])
    st = A.eval_parallel(to_layout(oracle.layout(net)), [0.9, 0.1], DEV)
    assert st.inputs[1] == np.float32(0.9) and st.inputs[0] == np.float32(0.1)
    assert st.outputs[1] == oracle.sigmoid32(np.float32(0.9))


def test_arity_and_pruned_and_sparse(oracle):
    lay = to_layout(oracle.layout(A.make_network([0, 1], [2], [(0, 2, 0.5), (1, 2, -0.25)])))
    with pytest.raises(A.InputArityMismatch):
        A.eval_parallel(lay, [1.0], DEV)
    with pytest.raises(A.InputArityMismatch):
        A.eval_parallel(lay, [1.0, 2.0, 3.0], DEV)
    lay = to_layout(oracle.layout(A.make_network([0], [2], [(0, 2, 1.0), (0, 3, 1.0)])))
    st = A.eval_parallel(lay, [0.9], DEV)
    assert st.outputs[3] == 0.0 and len(st.outputs) == 4      # pruned slot untouched
    d = oracle.layout(A.make_network([5, 30], [90], [(5, 90, 1.0), (30, 90, 1.0)]))
    st = A.eval_parallel(to_layout(d), [0.1, -0.2], DEV)
    assert len(st.outputs) == 91
    assert bitwise_equal(st.outputs, oracle.eval_batch(d, np.array([0.1, -0.2], np.float32))[0])


def test_layer_slice_and_width(oracle):
    d = oracle.layout(A.make_network([0, 1], [2], [(0, 2, 0.5), (1, 2, -0.25)]))
    dl = A.DeviceLayout.from_layout(to_layout(d))
    assert dl.layer_slice(0) == (0, 2) and dl.layer_slice(1) == (2, 1)
    with pytest.raises(A.LayerOutOfRange):
        dl.layer_slice(2)
    assert dl.info()["max_layer_width"] == 2


# --- the reference's verify corpus (golden op arrays from the reference) ----------------
def test_verify_corpus_against_reference_golden(oracle, verify_corpus, sweep_mode):
    stats = {}
    for case in verify_corpus:
        net = A.generate(case["spec"])
        d = oracle.layout(net)
        st = A.eval_parallel(to_layout(d), case["x"], DEV)
        check_close(st.outputs, case["op"], stats)
    assert stats["eq"] == stats["n"], stats          # bitwise


def test_adversarial_against_reference_golden(oracle, adversarial_nets, sweep_mode):
    stats = {}
    for case in adversarial_nets:
        if not case["flatten_ok"]:
            continue
        d = oracle.layout(case["net"])
        st = A.eval_parallel(to_layout(d), case["x"], DEV)
        check_close(st.outputs, case["op"], stats)
    assert stats["eq"] == stats["n"], stats          # bitwise


# --- batches: every padding / lane configuration -------------------------------------
@pytest.mark.parametrize("B", [1, 2, 3, 4, 5, 8, 16, 31, 64, 100, 128, 129, 256, 300, 1024])
def test_batch_widths(oracle, B, sweep_mode):
    rng = A.SplitMix64(1000 + B)
    spec = A.random_spec(rng, 2000, 20000)
    net = A.generate(spec)
    d = oracle.layout(net)
    X = np.array([[rng.uniform(-2, 2) for _ in net.inputs] for _ in range(B)], np.float32)
    dl = A.DeviceLayout.from_layout(to_layout(d, net.outputs))
    out, st = dl.activate(X, outputs=True, state=True)
    ref = oracle.eval_batch(d, X)
    stats = {}
    check_close(st, ref, stats)
    assert bitwise_equal(out, st[:, net.outputs])
    assert stats["eq"] == stats["n"], stats          # bitwise


def test_repeat_activation_is_deterministic(oracle, sweep_mode):
    rng = A.SplitMix64(77)
    net = A.generate(A.random_spec(rng, 5000, 20000))
    d = oracle.layout(net)
    dl = A.DeviceLayout.from_layout(to_layout(d, net.outputs))
    X = np.random.default_rng(3).uniform(-2, 2, (64, len(net.inputs))).astype(np.float32)
    a = dl.activate(X, state=True)[1]
    for _ in range(3):
        assert bitwise_equal(dl.activate(X, state=True)[1], a)


def test_inject_fault_is_seen(oracle):
    """asnn_main.cpp:264-278: the layout is mutated in place between two
    evaluations; the device backend must not serve a cached upload."""
    rng = A.SplitMix64(99)
    net = A.generate(A.random_spec(rng, 1000, 5000))
    d = oracle.layout(net)
    lay = to_layout(d)
    x = np.array([rng.uniform(-2, 2) for _ in net.inputs], np.float32)
    before = A.eval_parallel(lay, x, DEV).outputs.copy()
    k = int(np.argmax(np.abs(lay.in_weights)))
    lay.in_weights[k] *= -1.0
    after = A.eval_parallel(lay, x, DEV).outputs
    assert not bitwise_equal(before, after)
    d["in_weights"] = lay.in_weights
    stats = {}
    check_close(after, oracle.eval_batch(d, x)[0], stats)


def test_self_consistency(oracle, sweep_mode):
    """test_eval.cpp:109-134: every value recomputes exactly from the op array."""
    rng = A.SplitMix64(52)
    for _ in range(5):
        net = A.generate(A.random_spec(rng, 100, 3000))
        d = oracle.layout(net)
        x = np.array([rng.uniform(-3, 3) for _ in net.inputs], np.float32)
        st = A.eval_parallel(to_layout(d), x, DEV)
        vals = st.outputs[d["node_ids"]]
        assert np.all(vals > 0) and np.all(vals < 1)
        rec = oracle.recompute(d, x, st.outputs, np.arange(len(d["node_ids"])))
        assert np.array_equal(rec.view(np.uint32), vals.view(np.uint32))


# --- the streamed heavy-row kernel (k_heavy) ------------------------------------------
@pytest.mark.parametrize("B", [4, 8, 16, 32, 64, 100, 128, 256])
@pytest.mark.parametrize("thr", [16, 64])
def test_heavy_rows_bitwise(oracle, B, thr):
    """Power-law rows routed through the TMA-fed heavy kernel give the same
    values as the light kernel and the oracle (same summation order)."""
    net = A.generate_powerlaw(6000, 12, 32, 16, 150_000, 2.1, 11)
    d = oracle.layout(net)
    dl = A.DeviceLayout.from_network(net)
    X = np.random.default_rng(B).uniform(-2, 2, (B, len(net.inputs))).astype(np.float32)
    dev = A.Device.get(0)
    dev.set_sweep_mode(1)
    try:
        dev.set_heavy_threshold(thr)
        _, st_heavy = dl.activate(X, outputs=False, state=True)
        dev.set_heavy_threshold(None)
        _, st_light = dl.activate(X, outputs=False, state=True)
    finally:
        dev.set_heavy_threshold(512)
        dev.set_sweep_mode(0)
    assert bitwise_equal(st_heavy, st_light)
    stats = {}
    check_close(st_heavy, oracle.eval_batch(d, X), stats)
    assert stats["eq"] == stats["n"], stats          # bitwise


# --- hand-built layouts whose rows read ids without a position --------------------------
@pytest.mark.parametrize("B", [1, 4, 64, 256])
def test_predecessors_without_position(oracle, B, sweep_mode):
    """A LayeredLayout may list predecessors that have no position (pruned
    ids): eval_sequential reads their zero-initialised op slots
    (eval.cpp:20-21, make_state eval.cpp:25-35).  Every strategy must read
    0.0f for them (the never-written zero row) -- including K-cta's pipelined
    consumers, whose split treats such sources as layer 0."""
    rng = A.SplitMix64(404)
    net = A.generate(A.random_spec(rng, 500, 4000))
    dead = int(net.nodes.max()) + 7                       # a pruned node: never reaches an output
    net = A.Network(np.append(net.nodes, dead), net.inputs, net.outputs,
                    np.append(net.source, net.inputs[0]), np.append(net.target, dead),
                    np.append(net.weight, np.float32(0.5)))
    d = oracle.layout(net)
    assert dead not in set(d["node_ids"].tolist()) and d["id_bound"] > dead
    w = np.random.default_rng(B).random(len(d["in_nodes"]))
    d["in_nodes"] = d["in_nodes"].copy()
    d["in_nodes"][w < 0.05] = dead                        # 5% of the reads hit the zero slot
    X = np.random.default_rng(5).uniform(-2, 2, (B, len(d["input_order"]))).astype(np.float32)
    dl = A.DeviceLayout.from_layout(to_layout(d, net.outputs))
    _, st = dl.activate(X, outputs=True, state=True)
    assert bitwise_equal(st, oracle.eval_batch(d, X))


@pytest.mark.parametrize("sweep_mode", [0, 1, 2, 3, 4])
def test_zero_row_reused_across_narrowing_batches(oracle, sweep_mode):
    """One DeviceLayout reused with batch widths going down (256, 64, 4, 1):
    the zero row at the narrower pitch overlaps rows the wider sweep wrote
    and must read 0.0f again (eval.cpp:20-21 reads a zero-initialised slot)."""
    rng = A.SplitMix64(405)
    net = A.generate(A.random_spec(rng, 500, 4000))
    dead = int(net.nodes.max()) + 3
    net = A.Network(np.append(net.nodes, dead), net.inputs, net.outputs,
                    np.append(net.source, net.inputs[0]), np.append(net.target, dead),
                    np.append(net.weight, np.float32(0.5)))
    d = oracle.layout(net)
    d["in_nodes"] = d["in_nodes"].copy()
    d["in_nodes"][np.random.default_rng(7).random(len(d["in_nodes"])) < 0.05] = dead
    dl = A.DeviceLayout.from_layout(to_layout(d, net.outputs))
    A.Device.get(0).set_sweep_mode(sweep_mode)
    try:
        for B in (256, 64, 4, 1, 64, 2):
            X = np.random.default_rng(B).uniform(-2, 2, (B, len(d["input_order"]))).astype(np.float32)
            _, st = dl.activate(X, outputs=True, state=True)
            assert bitwise_equal(st, oracle.eval_batch(d, X)), B
    finally:
        A.Device.get(0).set_sweep_mode(0)


def test_upload_rejects_malformed_descriptors(oracle):
    """asnn_dev_upload_layout validates the CSR it is handed: row_ptr must
    start at 0 and never decrease, layer_offsets likewise (ASNN_E_INVALID,
    not out-of-bounds device reads)."""
    rng = A.SplitMix64(406)
    net = A.generate(A.random_spec(rng, 200, 1000))
    d = oracle.layout(net)
    for key, mutate in (("row_ptr", lambda a: a.__setitem__(3, a[4] + 5)),
                        ("row_ptr", lambda a: a.__setitem__(0, 1)),
                        ("layer_offsets", lambda a: a.__setitem__(1, a[2] + 1)),
                        ("layer_offsets", lambda a: a.__setitem__(0, 1))):
        bad = dict(d)
        bad[key] = d[key].copy()
        mutate(bad[key])
        with pytest.raises(ValueError):
            A.DeviceLayout.from_layout(to_layout(bad, net.outputs))
    A.DeviceLayout.from_layout(to_layout(d, net.outputs)).free()
