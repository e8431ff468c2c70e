"""Parity at BASELINE.json's full sizes.  Configs 2, 3 and 5: every vector
(every network) bitwise against the oracle's eval_sequential.  Config 4
(10M nodes, ~495M edges, batch 64) through size-independent properties --
the oracle cannot sweep this network in test time, so:
  * self-consistency (test_eval.cpp:109-134): every sampled node recomputes
    bit for bit from the finished id-indexed state with the oracle's
    activate_node restatement -- including the heaviest rows, whose sums the
    device split into segments across levels, and rows of the last levels;
  * determinism: a second sweep gives identical outputs;
  * the declared outputs equal the state at the output ids (read_outputs)."""
from __future__ import annotations

import numpy as np
import pytest

import bench
import paper_2005_04347_b200 as A

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_config4_self_consistency(oracle):
    net = bench.make_network("c4", 1.0)[0]
    assert len(net.source) > 490_000_000
    dl = A.DeviceLayout.from_network(net)
    B = 64
    assert dl.plan(B)["strategy"] == "segments"
    X = np.random.default_rng(4).uniform(-2, 2, (B, len(net.inputs))).astype(np.float32)
    out, st = dl.activate(X, outputs=True, state=True)
    out2, _ = dl.activate(X, outputs=True, state=False)
    assert np.array_equal(out.view(np.uint32), out2.view(np.uint32))
    assert np.array_equal(out.view(np.uint32), st[:, net.outputs].view(np.uint32))
    lay = dl.download()
    rp = lay.row_ptr.astype(np.int64)
    deg = np.diff(rp)
    n_pos = len(lay.node_ids)
    sensors = int(lay.layer_offsets[1])
    rng = np.random.default_rng(9)
    heavy = np.argsort(deg)[-300:]                       # segmented rows
    last = np.arange(int(lay.layer_offsets[-2]), n_pos)[:500]
    sample = np.unique(np.concatenate([rng.integers(sensors, n_pos, 3000), heavy, last]))
    sample = sample[sample >= sensors].astype(np.uint32)
    d = dict(layer_offsets=lay.layer_offsets, node_ids=lay.node_ids, row_ptr=lay.row_ptr,
             in_nodes=lay.in_nodes, in_weights=lay.in_weights, input_order=lay.input_order)
    for b in (0, 37, 63):
        rec = oracle.recompute(d, X[b], st[b], sample)
        got = st[b][lay.node_ids[sample]]
        assert np.array_equal(rec.view(np.uint32), got.view(np.uint32)), b


@pytest.mark.parametrize("cfg,check", [("c2", 1024), ("c3", 256)])
def test_config_full_size_bitwise(oracle, cfg, check):
    """Configs 2 and 3 at BASELINE.json's full size, activated with the full
    batch through the strategy the engine picks (per-level k_rows for C2,
    pipelined K-cta for C3); `check` vectors (all of them) compared with the
    oracle's eval_sequential bit for bit, state and outputs."""
    net = bench.make_network(cfg, 1.0)[0]
    B = bench.CONFIGS[cfg][1]
    dl = A.DeviceLayout.from_network(net)
    X = np.random.default_rng(11).uniform(-2, 2, (B, len(net.inputs))).astype(np.float32)
    out, st = dl.activate(X, outputs=True, state=True)
    d = oracle.layout(net)
    rows = np.sort(np.random.default_rng(12).choice(B, check, replace=False))
    want = oracle.eval_batch(d, X[rows])
    assert np.array_equal(st[rows].view(np.uint32), want.view(np.uint32))
    assert np.array_equal(out[rows].view(np.uint32), want[:, net.outputs].view(np.uint32))
    dl.free()


def test_config5_population_full_size_bitwise(oracle):
    """Config 5 at full size: 10k networks x 128 vectors in one K-cta launch;
    every network's outputs compared with the oracle bit for bit (state for
    every 50th network)."""
    nets = bench.make_network("c5", 1.0)
    B = bench.CONFIGS["c5"][1]
    rng = np.random.default_rng(13)
    X = [rng.uniform(-2, 2, (B, len(n.inputs))).astype(np.float32) for n in nets]
    dl = A.DeviceLayout.from_population(nets)
    out, _ = dl.activate(np.concatenate([x.reshape(-1) for x in X]), outputs=True, n_vec=B)
    out = np.asarray(out).reshape(-1)
    off = 0
    for g, (n, x) in enumerate(zip(nets, X)):
        k = len(n.outputs)
        got = out[off:off + B * k].reshape(B, k)
        off += B * k
        d = oracle.layout(n)
        want = oracle.eval_batch(d, x)
        assert np.array_equal(got.view(np.uint32), want[:, n.outputs].view(np.uint32)), g
    dl.free()
