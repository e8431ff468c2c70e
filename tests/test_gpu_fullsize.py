"""Parity at BASELINE.json's full sizes.

Configs 1 and 4 against the REFERENCE itself: tests/golden/fullsize_<cfg>.npz
holds the digests the unmodified reference produced on the same seeded
network (tests/golden/make_fullsize.py: its own compute_required / segment /
flatten, ~20 min for config 4, and eval_parallel on every vector of the batch):
the device layout (levels, node order, rows, weights, input order, dropped
count) and every vector's full id-indexed state must hash identically.

Configs 2, 3 and 5: every vector (every network) bitwise against the oracle's
eval_sequential.  Config 4 additionally through size-independent properties:
  * self-consistency (test_eval.cpp:109-134): every sampled node recomputes
    bit for bit from the finished id-indexed state with the oracle's
    activate_node restatement -- including the heaviest rows, whose sums the
    device split into segments across levels, and rows of the last levels;
  * determinism: a second sweep gives identical outputs;
  * the declared outputs equal the state at the output ids (read_outputs)."""
from __future__ import annotations

import pathlib

import numpy as np
import pytest

import bench
import paper_2005_04347_b200 as A

def _fixture_module():
    import importlib.util
    path = pathlib.Path(__file__).resolve().parent / "golden" / "make_fullsize.py"
    spec = importlib.util.spec_from_file_location("make_fullsize", path)
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


_fx = _fixture_module()
layout_digest, state_digest = _fx.layout_digest, _fx.state_digest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("cfg", ["c1", "c4"])
def test_config_against_reference_golden(cfg):
    """compute_required / segment / flatten and eval_parallel of the reference
    (segmentation.cpp:20-101, layout.cpp:12-83, eval.cpp:49-80) vs the device,
    bit for bit, at the config's full size and full batch (64 vectors)."""
    g = np.load(GOLDEN / f"fullsize_{cfg}.npz")
    net = bench.make_network(cfg, 1.0)[0]
    dl = A.DeviceLayout.from_network(net)
    lay = dl.download()
    assert len(lay.node_ids) == int(g["node_count"])
    assert len(lay.in_nodes) == int(g["edge_count"])
    assert lay.total_layers == int(g["total_layers"])
    assert lay.dropped_connections == int(g["dropped"])
    assert lay.id_bound == int(g["id_bound"])
    assert layout_digest(dict(layer_offsets=lay.layer_offsets, node_ids=lay.node_ids,
                              row_ptr=lay.row_ptr, in_nodes=lay.in_nodes,
                              in_weights=lay.in_weights, input_order=lay.input_order)) \
        == str(g["layout_sha256"])
    del lay
    assert len(A.compute_required(net).members) == int(g["required_count"])
    X = g["x"]
    outputs = np.asarray(net.outputs)
    want_out = g["outputs"]
    # the whole batch in one sweep, then in slices of 16 (other kernels / pitches)
    for lo, hi in ((0, X.shape[0]), (0, 16), (48, 64)):
        out, st = dl.activate(X[lo:hi], outputs=True, state=True)
        assert np.array_equal(out.view(np.uint32), want_out[lo:hi].view(np.uint32))
        for b in range(hi - lo):
            assert state_digest(st[b]) == str(g["state_sha256"][lo + b]), (lo + b)
            assert np.array_equal(st[b][outputs].view(np.uint32), want_out[lo + b].view(np.uint32))
        del st
    dl.free()


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
