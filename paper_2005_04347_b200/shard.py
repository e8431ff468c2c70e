"""Multi-GPU partitioning of the activation sweep.

A network's level-synchronous sweep does not shard without a per-layer
exchange, so the engine shards what is independent:

* batch sharding -- every rank holds a full layout replica and activates a
  contiguous slice of the input vectors; no traffic during the sweep;
* population sharding -- a contiguous, balanced slice of the networks per
  rank, each network with all of its vectors (so the gathered outputs are in
  population order).

The only collective is the final gather of the declared outputs.  Inside
the engine (csrc/group.cu) it is an NCCL all-gather on the engine's stream
(asnn_dev_comm_init / asnn_dev_allgather for one process per GPU,
asnn_group_* for one process driving several); gather_rows below is the
torch.distributed form used by the CPU (gloo) tests and by the one-GPU
functional mode, where NCCL cannot put two ranks on one device.  The
partition functions here and group.cu's `balanced` are the same rule.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def batch_slice(n_vec: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of the input vectors rank `rank` activates: contiguous and
    balanced (the first n_vec % world ranks take one extra vector)."""
    base, rem = divmod(n_vec, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def population_shard(n_networks: int, world: int, rank: int) -> List[int]:
    """Indices of the networks rank `rank` owns: a contiguous balanced slice
    (asnn_group_build_population's partition)."""
    lo, hi = batch_slice(n_networks, world, rank)
    return list(range(lo, hi))


def gather_rows(local, world: int, group=None):
    """All-gather variable-length row blocks (a torch tensor [rows, ...] on
    the backend's device) in rank order; returns the concatenation on every
    rank.  Blocks are padded to the largest one for the collective."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    n = torch.tensor([local.shape[0]], device=local.device, dtype=torch.int64)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def assemble_population(per_rank: Sequence[Sequence[np.ndarray]], n_networks: int,
                        world: int) -> List[np.ndarray]:
    """Per-network outputs back in population order from the per-rank lists
    of population_shard()."""
    out: List[Optional[np.ndarray]] = [None] * n_networks
    for r in range(world):
        for k, g in enumerate(population_shard(n_networks, world, r)):
            out[g] = per_rank[r][k]
    return out  # type: ignore[return-value]


class BatchShardedLayout:
    """A layout replica on this rank's GPU that activates its slice of a
    batch and all-gathers the declared outputs (NCCL)."""

    def __init__(self, device_layout, world: int, rank: int, group=None):
        self.dl = device_layout
        self.world, self.rank, self.group = world, rank, group
        self.n_out = device_layout.info()["n_outputs"]

    def activate(self, X: np.ndarray) -> np.ndarray:
        """X: the full batch [n_vec][n_in] (host).  Returns the full
        [n_vec][n_out] outputs on every rank."""
        import torch
        lo, hi = batch_slice(X.shape[0], self.world, self.rank)
        out, _ = self.dl.activate(X[lo:hi], outputs=True, state=False)
        t = torch.from_numpy(out).to(f"cuda:{torch.cuda.current_device()}")
        return gather_rows(t, self.world, self.group).cpu().numpy()
