"""Heavy rows split into segments across the levels of their sources
(csrc/segments.cuh): the partial fp32 sums parked between levels must give
bit-for-bit the reference's uninterrupted sum (eval.cpp:16-23), whatever the
cut points, the segment lengths and the kernel (k_rows / k_heavy) that runs
each segment."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from conftest import bitwise_equal, rel_close  # noqa: F401

pytestmark = pytest.mark.gpu


def check_bitwise(oracle, net, B, thr, seg_min, seg_long, seed=0):
    d = oracle.layout(net)
    dl = A.DeviceLayout.from_network(net)
    X = np.random.default_rng(seed + B).uniform(-2, 2, (B, len(net.inputs))).astype(np.float32)
    dev = A.Device.get(0)
    old = {k: os.environ.get(k) for k in ("ASNN_SEG_MIN", "ASNN_SEG_LONG")}
    os.environ["ASNN_SEG_MIN"] = str(seg_min)
    os.environ["ASNN_SEG_LONG"] = str(seg_long)
    dev.set_sweep_mode(1)
    try:
        dev.set_heavy_threshold(thr)
        assert dl.plan(B)["strategy"] == "segments"
        out, st = dl.activate(X, outputs=True, state=True)
    finally:
        dev.set_heavy_threshold(512)
        dev.set_sweep_mode(0)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    want = oracle.eval_batch(d, X)
    assert bitwise_equal(st, want), float(np.max(np.abs(st - want)))
    assert bitwise_equal(out, st[:, net.outputs])
    dl.free()


@pytest.mark.parametrize("B", [8, 16, 32, 64, 128, 256])
@pytest.mark.parametrize("thr,seg_min,seg_long", [(16, 1, 512), (16, 8, 32), (64, 64, 512), (32, 4, 16)])
def test_banded_powerlaw_segments(oracle, B, thr, seg_min, seg_long):
    """Banded power-law DAG (config 4's shape, small): ids ascend with the
    level, so heavy rows are cut into many segments; seg_long small sends
    some segments (with partial sums in and out) through k_heavy."""
    net = A.generate_powerlaw(6000, 12, 32, 16, 150_000, 2.1, 11)
    check_bitwise(oracle, net, B, thr, seg_min, seg_long)


def test_shuffled_ids_segments(oracle):
    """Node ids in random order: a row's source ids no longer follow the
    levels, the prefix max jumps early and most rows stay in one segment."""
    net = A.generate_powerlaw(4000, 10, 16, 8, 80_000, 2.1, 5)
    rng = np.random.default_rng(7)
    perm = rng.permutation(int(net.nodes.max()) + 1).astype(np.uint32)
    shuffled = A.Network(np.sort(perm[net.nodes]), perm[net.inputs], perm[net.outputs], perm[net.source],
                         perm[net.target], net.weight)
    check_bitwise(oracle, shuffled, 64, 16, 1, 64)


def test_reference_generator_segments(oracle):
    """The reference's own generator (netgen.cpp:71-157) at a deep shape."""
    rng = A.SplitMix64(4242)
    net = A.generate(A.random_spec(rng, 3000, 40000))
    check_bitwise(oracle, net, 128, 16, 2, 48)
