"""Concurrent callers on the engine's C-ABI (every operation
is reentrant; safe on distinct layouts, and on one immutable layout with
distinct states).  Host threads call asnn_dev_activate at once (ctypes drops
the GIL for the call): distinct handles with distinct layouts, one handle
with distinct layouts, and one layout with distinct batches; every result is
bitwise the oracle's eval_sequential."""
from __future__ import annotations

import threading

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from conftest import bitwise_equal

pytestmark = pytest.mark.gpu


def _run(workers):
    errors = []

    def wrap(fn, t):
        try:
            fn(t)
        except Exception as e:
            errors.append((t, repr(e)))
    th = [threading.Thread(target=wrap, args=(fn, t)) for t, fn in enumerate(workers)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert errors == []


@pytest.fixture(scope="module")
def corpus(oracle):
    rng = A.SplitMix64(332)
    nets = [A.generate(A.random_spec(rng, 3000, 40000)) for _ in range(4)]
    return [(n, oracle.layout(n)) for n in nets]


def test_distinct_handles_distinct_layouts(oracle, corpus):
    import ctypes as C
    devs = [A.Device(0) for _ in corpus]      # one asnn_dev (stream) per thread
    dls = []
    for dev, (n, _) in zip(devs, corpus):
        h = C.c_void_p()
        d = n.desc()
        dev.check(dev.lib.asnn_dev_build_layout(dev.h, C.byref(d), C.byref(h)))
        dls.append(A.DeviceLayout(dev, h))

    def worker(t):
        n, d = corpus[t]
        r = np.random.default_rng(t)
        for B in (1, 3, 64, 200, 7, 64):
            X = r.uniform(-2, 2, (B, len(n.inputs))).astype(np.float32)
            _, st = dls[t].activate(X, outputs=False, state=True)
            assert bitwise_equal(st, oracle.eval_batch(d, X)), (t, B)
    _run([worker] * len(corpus))
    for dl in dls:
        dl.free()
    for dev in devs:
        dev.close()


def test_one_handle_distinct_layouts(oracle, corpus):
    dls = [A.DeviceLayout.from_network(n) for n, _ in corpus]

    def worker(t):
        n, d = corpus[t]
        r = np.random.default_rng(10 + t)
        for B in (64, 1, 130, 5):
            X = r.uniform(-2, 2, (B, len(n.inputs))).astype(np.float32)
            out, st = dls[t].activate(X, outputs=True, state=True)
            want = oracle.eval_batch(d, X)
            assert bitwise_equal(st, want) and bitwise_equal(out, want[:, n.outputs]), (t, B)
    _run([worker] * len(corpus))
    for dl in dls:
        dl.free()


def test_one_layout_distinct_states(oracle, corpus):
    n, d = corpus[0]
    dl = A.DeviceLayout.from_network(n)

    def worker(t):
        r = np.random.default_rng(20 + t)
        for it in range(12):
            B = (1, 64, 17)[it % 3]
            X = r.uniform(-2, 2, (B, len(n.inputs))).astype(np.float32)
            _, st = dl.activate(X, outputs=False, state=True)
            assert bitwise_equal(st, oracle.eval_batch(d, X)), (t, it)
    _run([worker] * 6)
    dl.free()
