"""Parity of the one-call eval_parallel path (asnn_eval_buf / asnn_dev_eval_layout,
once.cu): a host layout staged in page-locked memory and evaluated by one kernel
with the reference's id-indexed state -- the per-call drop-in behind
eval.cpp:51-52.  Every kernel variant (zero-copy into shared memory, DMA + one
CTA, DMA + cooperative grid) is checked bitwise against the reference's golden
op arrays and the oracle (eval.cpp:16-23 restated in oracle/asnn_oracle.c)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from test_gpu_activate import to_layout

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["auto", "1", "2", "3", "4", "5", "6"],
                ids=["auto", "dma-cta", "dma-grid", "cta-plain", "grid-plain", "cluster", "cluster-ranges"])
def once_mode(request):
    old = os.environ.get("ASNN_ONCE_MODE")
    if request.param == "auto":
        os.environ.pop("ASNN_ONCE_MODE", None)
    else:
        os.environ["ASNN_ONCE_MODE"] = request.param
    yield request.param
    if old is None:
        os.environ.pop("ASNN_ONCE_MODE", None)
    else:
        os.environ["ASNN_ONCE_MODE"] = old


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_verify_corpus_against_reference_golden(oracle, verify_corpus, once_mode):
    for case in verify_corpus:
        d = oracle.layout(A.generate(case["spec"]))
        out = A.eval_once(to_layout(d), case["x"])
        assert np.array_equal(bits(out), bits(case["op"]))


def test_adversarial_against_reference_golden(oracle, adversarial_nets, once_mode):
    n = 0
    for case in adversarial_nets:
        if not case["flatten_ok"]:
            continue
        d = oracle.layout(case["net"])
        out = A.eval_once(to_layout(d), case["x"])
        assert np.array_equal(bits(out), bits(case["op"]))
        n += 1
    assert n > 100


@pytest.mark.parametrize("lo,hi", [(200, 1000), (2000, 20000), (12000, 120000), (200000, 400000)])
def test_random_specs_against_oracle(oracle, once_mode, lo, hi):
    rng = A.SplitMix64(lo * 7 + hi)
    for _ in range(3):
        spec = A.random_spec(rng, lo, hi)
        d = oracle.layout(A.generate(spec))
        lay = to_layout(d)
        x = np.array([np.float32((i % 13) * 0.17 - 1.0) for i in range(len(lay.input_order))], np.float32)
        ref = oracle.eval_batch(d, x[None, :])[0]
        assert np.array_equal(bits(A.eval_once(lay, x)), bits(ref))


def test_bench_corpus_shapes(oracle, once_mode):
    """The reference bench corpus (asnn_main.cpp make_corpus_spec): 8 inputs,
    2 outputs, hidden = connections / 10, depths 10 and 100."""
    for c, dpt in [(1000, 10), (10000, 10), (100000, 10), (10000, 100), (100000, 100)]:
        spec = A.corpus_spec(c, dpt, 8, 2, 42 + c + dpt)
        d = oracle.layout(A.generate(spec))
        lay = to_layout(d)
        x = np.full(len(lay.input_order), 0.5, np.float32)
        ref = oracle.eval_batch(d, x[None, :])[0]
        assert np.array_equal(bits(A.eval_once(lay, x)), bits(ref))


def test_variant_selection(oracle):
    os.environ.pop("ASNN_ONCE_MODE", None)
    buf = A.EvalBuffer()
    try:
        for c, dpt, want in [(1000, 10, 0), (10000, 10, 0), (100000, 10, 5), (1000000, 10, 2), (100000, 100, 6),
                             (20000, 100, 0)]:
            spec = A.corpus_spec(c, dpt, 8, 2, 7 + c)
            d = oracle.layout(A.generate(spec))
            lay = to_layout(d)
            x = np.linspace(-1, 1, len(lay.input_order)).astype(np.float32)
            buf.stage_layout(lay, x)
            out = buf.run()
            assert buf.mode == want, (c, buf.mode)
            assert np.array_equal(bits(out), bits(oracle.eval_batch(d, x[None, :])[0]))
    finally:
        buf.free()


def test_buffer_reuse_shrinking_and_growing(oracle, once_mode):
    """One staging buffer across layouts of different sizes: no stale state
    (ids past the new id_bound, edges of the previous layout) leaks in."""
    buf = A.EvalBuffer()
    try:
        for nodes, conns in [(20000, 200000), (300, 2000), (5000, 40000), (50, 100), (20000, 200000)]:
            spec = A.random_spec(A.SplitMix64(nodes + conns), nodes, conns)
            d = oracle.layout(A.generate(spec))
            lay = to_layout(d)
            x = np.full(len(lay.input_order), -0.25, np.float32)
            buf.stage_layout(lay, x)
            assert np.array_equal(bits(buf.run()), bits(oracle.eval_batch(d, x[None, :])[0]))
    finally:
        buf.free()


def test_heavy_rows_and_sparse_ids(oracle, once_mode):
    # one node with 6000 predecessors, ids with gaps (pruned nodes keep their ids)
    ins = list(range(0, 12000, 2))
    src = ins + [12001, 12001]
    edges = [(s, 12001, ((s * 37) % 101 - 50) / 50.0) for s in ins] + [(12001, 12003, 0.75),
                                                                       (ins[5], 12003, -0.5)]
    net = A.make_network(ins, [12003], edges)
    d = oracle.layout(net)
    lay = to_layout(d)
    x = np.linspace(-2, 2, len(ins)).astype(np.float32)
    assert np.array_equal(bits(A.eval_once(lay, x)), bits(oracle.eval_batch(d, x[None, :])[0]))
    del src


def test_duplicate_inputs_last_wins(oracle):
    net = A.make_network([0, 1, 0], [2], [(0, 2, 1.0), (1, 2, -1.0)])
    d = oracle.layout(net)
    lay = to_layout(d)
    x = np.array([0.3, 0.1, -0.7], np.float32)
    out = A.eval_once(lay, x)
    assert np.array_equal(bits(out), bits(oracle.eval_batch(d, x[None, :])[0]))
    st = A.eval_parallel(lay, x, A.ParallelConfig(backend=A.Backend.DeviceCompute))
    assert st.inputs[0] == np.float32(-0.7)
    assert np.array_equal(bits(st.outputs), bits(out))


def test_arity_and_malformed_layouts(oracle):
    net = A.make_network([0, 1], [3], [(0, 2, 0.5), (1, 2, 0.25), (2, 3, 1.0)])
    d = oracle.layout(net)
    lay = to_layout(d)
    with pytest.raises(A.InputArityMismatch):
        A.eval_once(lay, np.zeros(3, np.float32))
    # predecessor id outside the state
    bad = to_layout(d)
    bad.in_nodes = bad.in_nodes.copy()
    bad.in_nodes[-1] = 99
    with pytest.raises(ValueError, match="malformed"):
        A.eval_once(bad, np.zeros(2, np.float32))
    # node id outside the state
    bad = to_layout(d)
    bad.node_ids = bad.node_ids.copy()
    bad.node_ids[-1] = 1000
    with pytest.raises(ValueError, match="malformed"):
        A.eval_once(bad, np.zeros(2, np.float32))
    # row_ptr out of order
    bad = to_layout(d)
    bad.row_ptr = bad.row_ptr.copy()
    bad.row_ptr[3] = bad.row_ptr[4] + 1
    with pytest.raises(ValueError):
        A.eval_once(bad, np.zeros(2, np.float32))
    # layer table that does not cover the nodes
    bad = to_layout(d)
    bad.layer_offsets = bad.layer_offsets.copy()
    bad.layer_offsets[-1] -= 1
    with pytest.raises(ValueError):
        A.eval_once(bad, np.zeros(2, np.float32))
    # nodes but an empty state
    with pytest.raises(ValueError, match="malformed"):
        A.eval_once(A.LayeredLayout(1, [0, 1], [0], [0, 0], [], [], [], 0, 0), np.zeros(0, np.float32))
    # the handle still works afterwards
    x = np.array([0.5, -0.5], np.float32)
    assert np.array_equal(bits(A.eval_once(lay, x)), bits(oracle.eval_batch(d, x[None, :])[0]))


def test_empty_and_sensor_only():
    lay = A.LayeredLayout(1, [0, 2], [0, 1], [0, 0, 0], [], [], [0, 1], 0, 2)
    out = A.eval_once(lay, np.array([0.0, -200.0], np.float32))
    assert out[0] == np.float32(0.5)
    assert bits(out)[1] == 1  # sigmoid32(-200) = 0x1p-149, no flush to zero
    lay = A.LayeredLayout(0, [0], [], [0], [], [], [], 0, 0)
    assert A.eval_once(lay, np.zeros(0, np.float32)).size == 0


def test_concurrent_callers(oracle):
    """SPEC.md:331-332 on the one-call path: threads on one device handle, each
    with its own staging buffer (EvalBuffer) or the handle's (eval_once)."""
    import threading
    cases = []
    for i in range(6):
        spec = A.corpus_spec(2000 * (i + 1), 5 + 7 * i, 8, 2, 900 + i)
        d = oracle.layout(A.generate(spec))
        lay = to_layout(d)
        x = np.linspace(-1, 1, len(lay.input_order)).astype(np.float32) * (i + 1)
        cases.append((lay, x, oracle.eval_batch(d, x[None, :])[0]))
    errors = []

    def worker(k):
        try:
            buf = A.EvalBuffer() if k % 2 else None
            for r in range(20):
                lay, x, ref = cases[(k + r) % len(cases)]
                if buf is None:
                    out = A.eval_once(lay, x)
                else:
                    buf.stage_layout(lay, x)
                    out = buf.run()
                if not np.array_equal(bits(out), bits(ref)):
                    errors.append((k, r))
            if buf is not None:
                buf.free()
        except Exception as e:  # noqa: BLE001
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(6)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
