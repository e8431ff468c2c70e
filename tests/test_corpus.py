"""Synthetic corpora: the package's generate() is byte-identical to the
reference's (netgen.cpp:71-157); the config-2/4 shapes are deterministic and
have the structure DESIGN.md states.  CPU only."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from conftest import load_golden


def digest(net):
    h = hashlib.sha256()
    for a in (net.nodes, net.inputs, net.outputs, net.source, net.target, net.weight.view(np.uint32)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_generate_matches_reference_digests():
    g = load_golden("corpus_digest.npz")
    for row, wr, dg in zip(g["spec"], g["wrange"], g["digest"]):
        spec = A.GenSpec(int(row[0]), int(row[1]), int(row[2]), int(row[3]), int(row[4]),
                         float(wr[0]), float(wr[1]), int(row[5]))
        assert digest(A.generate(spec)) == str(dg)


def test_generate_matches_live_reference(ref):
    rng = A.SplitMix64(20260810)
    for _ in range(25):
        spec = A.random_spec(rng, 10, 20000)
        a = ref.generate(spec).arrays()
        net = A.generate(spec)
        for k in ("nodes", "inputs", "outputs", "source", "target"):
            assert np.array_equal(a[k], getattr(net, k))
        assert np.array_equal(a["weight"].view(np.uint32), net.weight.view(np.uint32))
    assert A.max_connections(A.GenSpec(4, 2, 30, 0, 6)) == ref.L.ref_max_connections(4, 2, 30, 6)


def test_generate_infeasible_specs():
    # test_netgen.cpp:111-147
    with pytest.raises(A.InfeasibleSpec):
        A.generate(A.GenSpec(0, 1, 0, 1, 2))
    with pytest.raises(A.InfeasibleSpec):
        A.generate(A.GenSpec(1, 1, 5, 10, 2))
    with pytest.raises(A.InfeasibleSpec):
        A.generate(A.GenSpec(1, 1, 1, 10, 5))
    with pytest.raises(A.InfeasibleSpec):
        A.generate(A.GenSpec(2, 1, 10, 5, 4))          # fewer edges than non-inputs
    with pytest.raises(A.InfeasibleSpec):
        A.generate(A.GenSpec(2, 1, 2, 1000, 4))        # over capacity


def test_generate_shape_and_depth(oracle):
    # test_netgen.cpp:47-60: exact depth and edge count
    spec = A.GenSpec(16, 4, 980, 10000, 10, seed=1)
    net = A.generate(spec)
    assert len(net.source) == 10000 and len(net.nodes) == 1000
    _, n = oracle.segment(net)
    assert n == 10


def test_mlp_shape(oracle):
    net = A.generate_mlp(12, 50, 0.3, 7)
    assert len(net.nodes) == 600 and len(net.inputs) == 50 and len(net.outputs) == 50
    assert np.all(net.source // 50 + 1 == net.target // 50)      # adjacent layers only
    level, n = oracle.segment(net)
    assert n == 12 and np.array_equal(level, net.nodes // 50)
    assert digest(net) == digest(A.generate_mlp(12, 50, 0.3, 7))


def test_powerlaw_shape(oracle):
    net = A.generate_powerlaw(20000, 10, 64, 32, 400000, 2.1, 5)
    assert len(net.nodes) == 20000
    e = len(net.source)
    assert 0.7 * 400000 < e < 1.3 * 400000
    # target-major, sources ascending and unique within a row
    assert np.all(np.diff(net.target.astype(np.int64)) >= 0)
    same = net.target[1:] == net.target[:-1]
    assert np.all(net.source[1:][same] > net.source[:-1][same])
    level, n = oracle.segment(net)
    assert n == 10
    assert np.all(level != 0xFFFFFFFF)              # every node reaches an output
    deg = np.bincount(net.target, minlength=20000)[64:]
    assert deg.max() > 10 * np.median(deg)          # heavy tail
    assert digest(net) == digest(A.generate_powerlaw(20000, 10, 64, 32, 400000, 2.1, 5))


@pytest.mark.parametrize("shape", [
    (3, 2, 12, 1.0, 4),      # full capacity: the dense branch takes every free pair
    (3, 2, 12, 0.8, 4),      # dense (more than half the free pairs)
    (1, 1, 6, 0.9, 5),       # one input: band 1 has no free source besides its mandatory one
    (5, 3, 0, 1.0, 2),       # depth 2, no hidden band
    (5, 3, 0, 0.6, 2),
    (2, 2, 40, 0.55, 8),
    (8, 4, 200, 0.3, 6),     # sparse, rejection with duplicates
])
def test_generate_dense_and_edge_specs_match_reference(ref, shape):
    """The dense branch (netgen.cpp:115-128, a shuffled prefix of the free
    pairs) and the sparse one (:129-141) near their switch-over and at the
    capacity limit, against the reference's own generate."""
    i, o, h, frac, d = shape
    cap = A.max_connections(A.GenSpec(i, o, h, 0, d))
    lo = h + o
    for seed in range(6):
        conn = max(lo, int(lo + (cap - lo) * frac))
        spec = A.GenSpec(i, o, h, conn, d, -2.0, 2.0, 1000 + seed)
        a = ref.generate(spec).arrays()
        net = A.generate(spec)
        for k in ("nodes", "inputs", "outputs", "source", "target"):
            assert np.array_equal(a[k], getattr(net, k)), (shape, seed, k)
        assert np.array_equal(a["weight"].view(np.uint32), net.weight.view(np.uint32))
