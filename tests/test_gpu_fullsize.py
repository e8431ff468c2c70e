"""Parity at BASELINE.json's full size (config 4: 10M nodes, ~495M edges,
batch 64) through size-independent properties -- the oracle cannot sweep
this network in test time, so:
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
