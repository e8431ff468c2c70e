"""The drop-in, end to end with the reference's own types: the reference's
compute_required / segment / flatten build a LayeredLayout, and
eval_parallel(..., Backend::DeviceCompute) is served by the maintainer's
binding in integration/asnn_device_backend.cpp (the two-line patch at
eval.cpp:51-52 of INTEGRATION.md) over the C-ABI.  Compared with the
reference's eval_sequential on the `verify` recipe (asnn_main.cpp:233-297)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from conftest import rel_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def refdev():
    from oracle.bind import RefDev, available_ref_dev
    if not available_ref_dev():
        pytest.skip("oracle/_ref/libasnn_ref_dev.so not built (reference checkout absent)")
    return RefDev()


def test_verify_recipe_through_reference_types(refdev):
    """The acceptance criterion (acceptance.cpp:72-85): 200
    trials of the verify recipe, 100..50,000 connections, seed 20260810."""
    master = A.SplitMix64(20260810)
    n_vals = n_eq = 0
    max_div = 0.0
    for trial in range(200):
        net_seed = master.next()
        rng = A.SplitMix64(net_seed)
        conn = 100 + rng.bounded(50000 - 100 + 1)
        depth = 3 + rng.bounded(2) if conn < 64 else 3 + rng.bounded(38)
        n_in = 1 + rng.bounded(8)
        n_out = 1 + rng.bounded(4)
        rn = refdev.generate(A.corpus_spec(conn, depth, n_in, n_out, net_seed))
        assert rn.preprocess() == 0
        x = np.array([rng.uniform(-2.0, 2.0) for _ in range(n_in)], np.float32)
        _, seq = rn.eval_sequential(x)
        rc, dev = refdev.eval_device(rn, x)
        assert rc == 0
        # asnn_main.cpp:280-291: absolute 1e-5 per node; plus 1e-5 relative
        max_div = max(max_div, float(np.max(np.abs(seq.astype(np.float64) - dev))))
        assert rel_close(dev, seq).all()
        n_vals += seq.size
        n_eq += int((seq.view(np.uint32) == dev.view(np.uint32)).sum())
    assert max_div <= 1e-5
    assert n_eq == n_vals          # bitwise


def test_arity_maps_to_reference_exception(refdev):
    rn = refdev.network(A.make_network([0, 1], [2], [(0, 2, 0.5), (1, 2, -0.25)]))
    assert rn.preprocess() == 0
    rc, _ = refdev.eval_device(rn, np.zeros(3, np.float32))
    assert rc == 2          # InputArityMismatch
    rc, out = refdev.eval_device(rn, np.array([1.0, -1.0], np.float32))
    assert rc == 0 and abs(float(out[0]) - 0.9931047268673539) < 1e-6


def test_reference_host_backends_untouched(refdev):
    """With the binding present, HostParallel still runs the reference's own
    OpenMP evaluator, bitwise equal to eval_sequential (test_eval.cpp:136-149)."""
    rng = A.SplitMix64(53)
    for _ in range(5):
        rn = refdev.generate(A.random_spec(rng, 100, 5000))
        assert rn.preprocess() == 0
        n_in = len(rn.layout()["input_order"])
        x = np.array([rng.uniform(-2, 2) for _ in range(n_in)], np.float32)
        _, seq = rn.eval_sequential(x)
        rc, par = rn.eval_parallel(x, workers=2, backend=0)
        assert rc == 0 and np.array_equal(seq.view(np.uint32), par.view(np.uint32))


def test_concurrent_callers_through_the_binding(refdev):
    """SPEC.md:331-332 through the drop-in: eval_parallel(DeviceCompute) from
    several host threads at once -- distinct layouts, and one immutable layout
    with distinct input vectors -- each result bitwise the reference's
    eval_sequential on the same call."""
    import threading
    rng = A.SplitMix64(331)
    nets = [refdev.generate(A.random_spec(rng, 2000, 20000)) for _ in range(4)]
    for rn in nets:
        assert rn.preprocess() == 0
    n_ins = [len(rn.layout()["input_order"]) for rn in nets]
    errors = []

    def worker(t, shared):
        try:
            r = np.random.default_rng(t)
            for it in range(25):
                k = 0 if shared else t
                rn = nets[k]
                x = r.uniform(-2, 2, n_ins[k]).astype(np.float32)
                rc, dev = refdev.eval_device(rn, x)
                _, seq = rn.eval_sequential(x)
                if rc != 0 or not np.array_equal(dev.view(np.uint32), seq.view(np.uint32)):
                    errors.append((t, it, rc))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((t, repr(e)))

    for shared in (False, True):
        th = [threading.Thread(target=worker, args=(t, shared)) for t in range(4)]
        for x in th:
            x.start()
        for x in th:
            x.join()
    assert errors == []
