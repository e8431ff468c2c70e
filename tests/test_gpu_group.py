"""Multi-GPU sharding inside the engine (csrc/group.cu) on one
B200: a group that lists device 0 several times runs every shard on the same
GPU with the copy-engine gather, a one-device group exercises the NCCL
loader and a one-rank communicator.  Every result is compared bitwise with
the oracle's eval_sequential (eval.cpp:39-47)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from conftest import bitwise_equal
from paper_2005_04347_b200.shard import batch_slice, population_shard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("B", [1, 7, 64, 130])
def test_batch_sharded_group_bitwise(oracle, devices, B):
    net = A.generate(A.GenSpec(12, 5, 1500, 15000, 14, seed=71 + B))
    d = oracle.layout(net)
    X = np.random.default_rng(B).uniform(-2, 2, (B, len(net.inputs))).astype(np.float32)
    grp = A.DeviceGroup(devices)
    assert grp.gather == ("single device" if len(devices) == 1 else "copy engines")
    gl = grp.layout(net)
    out, st = gl.activate(X, state=True)
    want = oracle.eval_batch(d, X)
    assert bitwise_equal(st, want)
    assert bitwise_equal(out, want[:, net.outputs])
    # the partition is shard.py's rule
    for i in range(len(devices)):
        sh = gl.shard(i, B)
        lo, hi = batch_slice(B, len(devices), i)
        assert sh["vecs"] == hi - lo and sh["x_off"] == lo * len(net.inputs)
        assert sh["out_off"] == lo * len(net.outputs)
    # resident path: staged inputs, sweeps + gathers, outputs read back
    gl.stage(X, B)
    ms = gl.sweep(3)
    assert ms > 0
    assert bitwise_equal(gl.read_outputs().reshape(B, -1), want[:, net.outputs])
    gl.free()
    grp.close()


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_population_sharded_group_bitwise(oracle, devices):
    rng = A.SplitMix64(505)
    nets = [A.generate(A.GenSpec(6, 3, 90, 600, 6, seed=rng.next())) for _ in range(25)]
    V = 16
    Xs = [np.random.default_rng(g).uniform(-2, 2, (V, len(n.inputs))).astype(np.float32)
          for g, n in enumerate(nets)]
    grp = A.DeviceGroup(devices)
    gl = grp.population(nets)
    out, st = gl.activate(np.concatenate([x.reshape(-1) for x in Xs]), n_vec=V, state=True)
    o = s = 0
    for g, (n, x) in enumerate(zip(nets, Xs)):
        d = oracle.layout(n)
        want = oracle.eval_batch(d, x)
        k, idb = len(n.outputs), d["id_bound"]
        assert bitwise_equal(out[o:o + V * k].reshape(V, k), want[:, n.outputs]), g
        assert bitwise_equal(st[s:s + V * idb].reshape(V, idb), want), g
        o += V * k
        s += V * idb
    owned = [population_shard(len(nets), len(devices), i) for i in range(len(devices))]
    assert sum(owned, []) == list(range(len(nets)))
    gl.free()
    grp.close()


def test_group_sweep_options_and_errors(oracle):
    net = A.generate(A.GenSpec(4, 2, 300, 2500, 30, seed=9))
    d = oracle.layout(net)
    X = np.random.default_rng(1).uniform(-2, 2, (9, len(net.inputs))).astype(np.float32)
    grp = A.DeviceGroup([0, 0])
    gl = grp.layout(net)
    for mode in (1, 2, 3):
        grp.set_sweep_mode(mode)
        out, _ = gl.activate(X)
        assert bitwise_equal(out, oracle.eval_batch(d, X)[:, net.outputs]), mode
    grp.set_sweep_mode(0)
    with pytest.raises(A.InputArityMismatch):
        gl.activate(X[:, :-1])
    gl.free()
    grp.close()


def test_nccl_one_rank_allgather():
    """The NCCL path end to end on one GPU: libnccl resolved at run time, a
    one-rank communicator, the in-place all-gather on the engine's stream."""
    import torch
    uid = A.comm_unique_id()
    assert len(uid) == 128
    dev = A.Device(0)
    dev.comm_init(uid, 1, 0)
    buf = torch.arange(10, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    dev.allgather(buf.data_ptr(), buf.data_ptr(), [10])
    dev.synchronize()
    assert torch.equal(buf.cpu(), torch.arange(10, dtype=torch.float32))
    dev.close()
