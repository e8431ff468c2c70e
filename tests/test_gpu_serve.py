"""The resident batch-1 server (asnn_dev_server_*, csrc/serve.cuh): a
persistent one-CTA kernel holding one layout in shared memory and answering
activations through a doorbell in page-locked host memory.  Same contract as
asnn_dev_activate (eval.cpp:49-87): outputs bitwise equal to the oracle (the
reference's eval order and sigmoid32), arity errors mapped to
InputArityMismatch, many requests in a row, start/stop/restart, and a layout
freed under a live server."""
from __future__ import annotations

import time

import numpy as np
import pytest

import paper_2005_04347_b200 as A

pytestmark = pytest.mark.gpu


def _net(seed, hidden=188, conns=1000, depth=8, n_in=8, n_out=4):
    return A.generate(A.GenSpec(n_in, n_out, hidden, conns, depth, -1.0, 1.0, seed))


def _expect(oracle, net, X):
    lay = oracle.layout(net)
    st = oracle.eval_batch(lay, X)
    return st[:, np.asarray(net.outputs)]


@pytest.mark.parametrize("seed", [1, 7, 2005])
def test_server_bitwise_many_requests(oracle, seed):
    net = _net(seed)
    dl = A.DeviceLayout.from_network(net, device=0)
    rng = np.random.default_rng(seed)
    X = rng.uniform(-2, 2, (64, len(net.inputs))).astype(np.float32)
    want = _expect(oracle, net, X)
    with dl.serve(max_vec=1) as srv:
        for i in range(64):
            got = srv.activate(X[i:i + 1])
            assert np.array_equal(got.view(np.uint32), want[i:i + 1].view(np.uint32)), f"request {i}"
    dl.free()


def test_server_batches_and_config1(oracle):
    # config 1's exact spec (BASELINE configs[0]): 16 inputs, 4 outputs, 980 hidden, 10k connections
    net = A.generate(A.GenSpec(16, 4, 980, 10000, 10, -1.0, 1.0, 1))
    dl = A.DeviceLayout.from_network(net, device=0)
    rng = np.random.default_rng(3)
    X = rng.uniform(-2, 2, (40, len(net.inputs))).astype(np.float32)
    want = _expect(oracle, net, X)
    srv = dl.serve(max_vec=8)
    at = 0
    for nv in (1, 8, 3, 5, 1, 8, 8, 6):
        got = srv.activate(X[at:at + nv])
        assert np.array_equal(got.view(np.uint32), want[at:at + nv].view(np.uint32)), (at, nv)
        at += nv
    with pytest.raises(A.InputArityMismatch):
        srv.activate(X[:1, :-1])
    with pytest.raises(ValueError):
        srv.activate(np.zeros((9, len(net.inputs)), np.float32))  # more than max_vec
    # still serving after the rejected calls
    got = srv.activate(X[:1])
    assert np.array_equal(got.view(np.uint32), want[:1].view(np.uint32))
    srv.close()
    # restart on the same layout
    with dl.serve() as srv2:
        got = srv2.activate(X[5:6])
        assert np.array_equal(got.view(np.uint32), want[5:6].view(np.uint32))
    dl.free()


def test_server_zero_row_and_layout_free(oracle):
    # a hand-built layout whose rows reference an id with no position (zero row)
    d = oracle.layout(_net(11))
    free_ids = np.setdiff1d(np.arange(d["id_bound"], dtype=np.uint32), d["node_ids"])
    assert free_ids.size, "the generator left no unassigned id"
    in_nodes = d["in_nodes"].copy()
    in_nodes[len(in_nodes) // 2] = free_ids[0]
    lay = A.LayeredLayout(d["total_layers"], d["layer_offsets"], d["node_ids"], d["row_ptr"],
                          in_nodes, d["in_weights"], d["input_order"], d["dropped_connections"],
                          d["id_bound"], np.asarray(d["node_ids"][-2:], np.uint32))
    dl = A.DeviceLayout.from_layout(lay, device=0)
    X = np.random.default_rng(0).uniform(-2, 2, (4, len(d["input_order"]))).astype(np.float32)
    out_ref, _ = dl.activate(X)
    srv = dl.serve(max_vec=4)
    got = srv.activate(X)
    assert np.array_equal(got.view(np.uint32), out_ref.view(np.uint32))
    dl.free()  # stops the live server
    srv.close()  # no-op after the layout stopped it


def test_server_rejects_populations_and_reports_latency(oracle):
    nets = [_net(s, hidden=60, conns=200, depth=4) for s in (1, 2)]
    dl = A.DeviceLayout.from_population(nets, device=0)
    with pytest.raises(A.BackendUnavailable):
        dl.serve()
    dl.free()
    net = _net(5)
    dl = A.DeviceLayout.from_network(net, device=0)
    x = np.random.default_rng(1).uniform(-2, 2, (1, len(net.inputs))).astype(np.float32)
    with dl.serve() as srv:
        for _ in range(20):
            srv.activate(x)
        t0 = time.perf_counter()
        for _ in range(200):
            srv.activate(x)
        us = (time.perf_counter() - t0) / 200 * 1e6
        tm = srv.timings()
    print(f"resident server: {us:.1f} us per vector from Python; last call {tm}")
    assert us < 1000.0
    dl.free()
