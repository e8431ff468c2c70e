"""Multi-process (world_size 2, gloo, CPU) coverage of the sharding plumbing
of paper_2005_04347_b200/shard.py: batch slices, population deal, the
variable-length output all-gather and reassembly.  The per-shard compute in
these CPU tests is the oracle (the stand-in for each rank's GPU); on a B200
each rank runs the engine and the gather uses NCCL (bench.py)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2005_04347_b200.shard import assemble_population, batch_slice, population_shard


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_batch_slice_partitions():
    for n in range(0, 40):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                lo, hi = batch_slice(n, world, r)
                assert 0 <= lo <= hi <= n
                assert hi - lo in (n // world, n // world + 1)
                cover.extend(range(lo, hi))
            assert cover == list(range(n))


def test_population_shard_partitions():
    for n in (0, 1, 7, 100):
        for world in (1, 2, 8):
            got = sorted(g for r in range(world) for g in population_shard(n, world, r))
            assert got == list(range(n))
    per_rank = [[np.full(2, g) for g in population_shard(9, 2, r)] for r in range(2)]
    out = assemble_population(per_rank, 9, 2)
    assert [int(o[0]) for o in out] == list(range(9))


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import paper_2005_04347_b200 as A
    from oracle.bind import Oracle
    from paper_2005_04347_b200.shard import gather_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        # batch sharding of one network, uneven batch
        net = A.generate(A.GenSpec(6, 3, 400, 4000, 9, seed=11))
        lay = o.layout(net)
        X = np.random.default_rng(0).uniform(-2, 2, (7, 6)).astype(np.float32)
        lo, hi = batch_slice(7, world, rank)
        local = o.eval_batch(lay, X[lo:hi])[:, net.outputs] if hi > lo else \
            np.zeros((0, len(net.outputs)), np.float32)
        full = gather_rows(torch.from_numpy(np.ascontiguousarray(local)), world).numpy()
        want = o.eval_batch(lay, X)[:, net.outputs]
        ok_batch = np.array_equal(full.view(np.uint32), want.view(np.uint32))
        # population sharding, each network with its own vectors
        rng = A.SplitMix64(5)
        nets = [A.generate(A.GenSpec(4, 2, 40, 200, 5, seed=rng.next())) for _ in range(5)]
        Xs = [np.random.default_rng(g).uniform(-2, 2, (3, 4)).astype(np.float32) for g in range(5)]
        mine = population_shard(5, world, rank)
        blocks = [o.eval_batch(o.layout(nets[g]), Xs[g])[:, nets[g].outputs] for g in mine]
        local = np.concatenate(blocks).reshape(-1, 3, 2) if blocks else np.zeros((0, 3, 2), np.float32)
        allr = gather_rows(torch.from_numpy(np.ascontiguousarray(local)), world).numpy()
        # rank-order concatenation -> per rank lists -> population order
        per_rank, k = [], 0
        for r in range(world):
            cnt = len(population_shard(5, world, r))
            per_rank.append(list(allr[k:k + cnt]))
            k += cnt
        pop = assemble_population(per_rank, 5, world)
        ok_pop = all(np.array_equal(pop[g], o.eval_batch(o.layout(nets[g]), Xs[g])[:, nets[g].outputs])
                     for g in range(5))
        q.put((rank, ok_batch, ok_pop))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_reassembly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert res == [(0, True, True), (1, True, True)]
