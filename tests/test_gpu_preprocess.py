"""Device preprocessing parity: compute_required / segment (GPU Kahn) /
flatten (GPU radix-sort CSR build) against the reference-generated golden
fixtures and the oracle.  Integer work: bit-exact or it fails."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from conftest import bitwise_equal, rel_close

pytestmark = pytest.mark.gpu
UN = 0xFFFFFFFF


def device_levels(net):
    dev = A.Device.get(0)
    import ctypes as C
    from paper_2005_04347_b200 import _lib
    level = np.zeros(len(net.nodes), np.uint32)
    n = C.c_uint32()
    d = net.desc()
    dev.check(dev.lib.asnn_dev_segment(dev.h, C.byref(d), None, _lib.ptr(level, C.c_uint32),
                                       C.byref(n)))
    return level, n.value


def same_layout(lay: A.LayeredLayout, d: dict):
    assert lay.total_layers == d["total_layers"]
    for k in ("layer_offsets", "node_ids", "row_ptr", "in_nodes"):
        assert np.array_equal(getattr(lay, k).astype(np.uint64), d[k].astype(np.uint64)), k
    assert bitwise_equal(lay.in_weights, d["in_weights"])
    assert np.array_equal(lay.input_order, d["input_order"])
    assert lay.dropped_connections == d["dropped_connections"]
    assert lay.id_bound == d["id_bound"]


def test_fixtures():
    # test_segmentation.cpp:10-48 through the mirror API
    net = A.make_network([0, 1], [2], [(0, 2, 0.5), (1, 2, -0.25)])
    a = A.segment(net, A.compute_required(net))
    assert [l.tolist() for l in a.layers] == [[0, 1], [2]] and a.unassigned.size == 0
    net = A.make_network([0], [3], [(0, 1, 1.0), (0, 2, 0.5), (1, 2, -1.0), (2, 3, 0.75),
                                    (0, 3, 0.25)])
    a = A.segment(net)
    assert [l.tolist() for l in a.layers] == [[0], [1], [2], [3]]
    lay = A.flatten(net, a)
    assert lay.row(3)[0].tolist() == [0, 2] and lay.row(3)[1].tolist() == [0.25, 0.75]
    net = A.make_network([0], [2], [(0, 2, 1.0), (0, 3, 1.0)])
    req = A.compute_required(net)
    assert req.members.tolist() == [0, 2]
    a = A.segment(net, req)
    assert [l.tolist() for l in a.layers] == [[0], [2]] and a.unassigned.tolist() == [3]
    assert a.layer_of(3) is None and a.layer_of(2) == 1 and a.layer_of(99) is None
    lay = A.flatten(net, a)
    assert lay.dropped_connections == 1 and lay.id_bound == 4 and lay.node_count() == 2
    net = A.make_network([0], [2], [(3, 2, 1.0)], [0])
    a = A.segment(net)
    assert A.unassigned_outputs(net, a) == [2]
    with pytest.raises(A.OutputUnreachable):
        A.flatten(net, a)
    with pytest.raises(A.OutputUnreachable):
        A.DeviceLayout.from_network(net)
    net = A.make_network([5, 30], [90], [(5, 90, 1.0), (30, 90, 1.0)])
    lay = A.flatten(net)
    assert lay.id_bound == 91 and lay.row(2)[0].tolist() == [5, 30]


def test_adversarial_against_reference(oracle, adversarial_nets):
    for case in adversarial_nets:
        net = case["net"]
        req = A.compute_required(net)
        assert np.array_equal(req.members, case["required"])
        level, n = device_levels(net)
        assert np.array_equal(level, case["level"])
        if case["flatten_ok"]:
            dl = A.DeviceLayout.from_network(net)
            same_layout(dl.download(0), oracle.layout(net))
            assert dl.info()["dropped_connections"] == case["dropped"]
            out, st = dl.activate(case["x"][None, :], outputs=True, state=True)
            assert rel_close(st[0], case["op"]).all()
        else:
            with pytest.raises(A.OutputUnreachable):
                A.DeviceLayout.from_network(net)


def test_verify_corpus_layouts(oracle, verify_corpus):
    for case in verify_corpus:
        net = A.generate(case["spec"])
        dl = A.DeviceLayout.from_network(net)
        lay = dl.download(0)
        h = hashlib.sha256()
        for a in (lay.layer_offsets, lay.node_ids, lay.row_ptr, lay.in_nodes,
                  lay.in_weights.view(np.uint32)):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == case["csr_digest"]
        assert np.diff(lay.layer_offsets).tolist() == case["layer_sizes"]
        assert np.array_equal(lay.node_ids, case["members"])


def test_random_specs_levels(oracle):
    rng = A.SplitMix64(32)
    for _ in range(40):
        net = A.generate(A.random_spec(rng, 50, 30000))
        level, n = device_levels(net)
        ol, on = oracle.segment(net)
        assert n == on and np.array_equal(level, ol)


def test_shuffled_edges_and_sparse_ids(oracle):
    """Edge order must not matter (rows are sorted by source id) and ids may
    be sparse (node_index binary search path)."""
    rng = np.random.default_rng(8)
    base = A.generate(A.GenSpec(6, 3, 400, 5000, 12, seed=77))
    perm = rng.permutation(len(base.source))
    remap = np.sort(rng.choice(10 ** 6, size=len(base.nodes), replace=False)).astype(np.uint32)
    net = A.Network(remap[base.nodes], remap[base.inputs], remap[base.outputs],
                    remap[base.source[perm]], remap[base.target[perm]], base.weight[perm])
    dl = A.DeviceLayout.from_network(net)
    same_layout(dl.download(0), oracle.layout(net))


def test_deep_chain_and_wide_fan():
    # 3000-level chain with skip edges; and one node with 200k predecessors
    n = 3000
    src = list(range(n - 1)) + list(range(0, n - 2, 7))
    dst = list(range(1, n)) + [i + 2 for i in range(0, n - 2, 7)]
    net = A.make_network([0], [n - 1], list(zip(src, dst, [0.5] * len(src))))
    level, nl = device_levels(net)
    assert nl == n and np.array_equal(level, np.arange(n))
    k = 200_000
    net = A.make_network(list(range(k)), [k], [(i, k, 1e-3) for i in range(k)])
    level, nl = device_levels(net)
    assert nl == 2 and level[k] == 1


@pytest.mark.parametrize("mode", [1, 2])
def test_population_matches_single_networks(oracle, mode):
    rng = A.SplitMix64(5)
    nets = [A.generate(A.GenSpec(8, 4, 188, 1000, 8, seed=rng.next())) for _ in range(50)]
    pop = A.DeviceLayout.from_population(nets)
    A.Device.get(0).set_sweep_mode(mode)
    info = pop.info()
    assert info["n_networks"] == 50
    X = np.random.default_rng(1).uniform(-2, 2, (50, 16, 8)).astype(np.float32)
    out, st = pop.activate(X, outputs=True, state=True, n_vec=16)
    k = 0
    ko = 0
    for g, net in enumerate(nets):
        d = oracle.layout(net)
        same_layout(pop.download(g), d)
        ref = oracle.eval_batch(d, X[g])
        got = st.reshape(-1)[k:k + 16 * d["id_bound"]].reshape(16, d["id_bound"])
        k += 16 * d["id_bound"]
        assert rel_close(got, ref).all()
        o = out.reshape(-1)[ko:ko + 16 * 4].reshape(16, 4)
        ko += 16 * 4
        assert bitwise_equal(o, got[:, net.outputs])
    A.Device.get(0).set_sweep_mode(0)
