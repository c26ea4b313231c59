"""Multi-GPU partitioning: one process per GPU, torch.distributed.

* PDHG gate-sharding: rank r owns a contiguous block of gates (their y_i, d_i,
  warps); every rank holds the replicated x, z, zbar and computes the identical
  prox step locally, so the only exchange per iteration is one allreduce(sum)
  of the image-sized partial sum of D_i^* A_i^* dy_i (NCCL over NVLink), after
  which every rank applies z += dz, zbar = z + theta*dz (all p_i = 1 in PDHG).
* Batch slices (C5): independent units, ``slice_shard`` splits them with no
  data-path collective.
* SPDHG of a single problem does not shard (one gate per iteration,
  strictly sequential): replicas only.
"""

from __future__ import annotations

from typing import Protocol

import numpy as np

__all__ = ["gate_shard", "slice_shard", "sharded_epochs", "ShardedPDHG", "run_pdhg_sharded"]


def _block(count: int, world: int, rank: int) -> tuple[int, int]:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid world size / rank")
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gate_shard(num_gates: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced gate block [lo, hi) of ``rank`` (20/8 -> 3,3,3,3,2,2,2,2)."""
    return _block(num_gates, world, rank)


def slice_shard(num_slices: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice block of ``rank`` for the batch workload (no collective)."""
    return _block(num_slices, world, rank)


class ShardWorker(Protocol):
    def local_iteration(self):
        """Run the local gates of one PDHG iteration; return the partial dz tensor."""

    def finish(self, dz) -> None:
        """Apply the globally reduced dz: z += dz; zbar = z + theta*dz."""


def sharded_epochs(worker: ShardWorker, epochs: int, group=None) -> None:
    """PDHG epochs with one allreduce(sum) of the image-sized update per iteration."""
    import torch.distributed as dist

    for _ in range(epochs):
        dz = worker.local_iteration()
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(dz, op=dist.ReduceOp.SUM, group=group)
        worker.finish(dz)


class ShardedPDHG:
    """GPU worker: the fused K1..K4 kernels on the local gate block."""

    def __init__(self, config, problem, rank: int, world: int, keep_projections=False):
        from .engine import Engine

        if config.mode != "pdhg":
            raise ValueError("gate sharding applies to pdhg (spdhg runs as replicas)")
        if config.num_gates != problem.num_gates:
            raise ValueError("config and problem disagree on the gate count")
        self.lo, self.hi = gate_shard(problem.num_gates, world, rank)
        if self.hi <= self.lo:
            raise ValueError("more ranks than gates")
        self.engine = Engine([problem.operators], [problem.data], gate_range=(self.lo, self.hi),
                             keep_projections=keep_projections)
        self.engine.set_params(config)
        self.engine.reset()
        self.alpha = problem.alpha
        self.theta = config.theta
        self.dz = self.engine.torch.zeros_like(self.engine.x)

    def local_iteration(self):
        eng = self.engine
        eng.iteration(eng.items_pdhg(epoch_ctr=True), self.alpha, dz=self.dz)
        return self.dz

    def finish(self, dz):
        self.engine.z_update(dz, self.theta)
        self.engine.advance_epoch()


def run_pdhg_sharded(config, problem, group=None):
    """PDHG over the ranks of ``group``; returns x (float64 numpy) on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    w = ShardedPDHG(config, problem, rank, world)
    sharded_epochs(w, config.epochs, group)
    from .solvers import _raise_status

    _raise_status(w.engine)
    return np.asarray(w.engine.x[0].double().cpu().numpy())
