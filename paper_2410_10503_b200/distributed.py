"""Multi-GPU partitioning: one process per GPU, torch.distributed.

* PDHG gate-sharding: rank r owns a contiguous block of gates (their y_i, d_i,
  warps); every rank holds the replicated x, z, zbar and computes the identical
  prox step locally, so the only exchange per iteration is the sum of the
  image-sized partials D_i^* A_i^* dy_i, after which every rank applies
  z += dz, zbar = z + theta*dz (all p_i = 1 in PDHG).  Two exchanges:
  ``"p2p"`` (default on GPUs) — K4 writes the partial into a peer-visible
  symmetric buffer and the fused ``mct_exchange_*`` kernels sum the peers'
  partials over NVLink inside the z update (``P2PExchange``); ``"nccl"`` — an
  NCCL allreduce(sum) followed by ``mct_iter_z_update``.
* Batch slices (C5): independent units, ``slice_shard`` splits them with no
  data-path collective.
* SPDHG of a single problem does not shard (one gate per iteration,
  strictly sequential): replicas only.
"""

from __future__ import annotations

from typing import Protocol

import numpy as np

__all__ = ["gate_shard", "unit_shard", "half_angle_rows", "slice_shard", "sharded_epochs", "ShardedPDHG", "run_pdhg_sharded",
           "P2PExchange", "exchange_schedule"]


def _block(count: int, world: int, rank: int) -> tuple[int, int]:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid world size / rank")
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gate_shard(num_gates: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced gate block [lo, hi) of ``rank`` (20/8 -> 3,3,3,3,2,2,2,2)."""
    return _block(num_gates, world, rank)


def unit_shard(num_gates: int, world: int, rank: int):
    """Half-gate units of ``rank`` (gate-sharded PDHG balanced to half a gate).

    The 2N units (gate g, half h) are split into contiguous balanced blocks; a rank
    gets the full gates [lo, hi) whose both halves it owns, plus at most one half
    gate ``(g, part)`` at either end (part 1 = first half of the angle pairs, 2 =
    second).  Returns ``(lo, hi, half)`` with ``half`` None when the block is
    gate-aligned (e.g. 20 gates on 1, 2 or 4 ranks; 40 on 8)."""
    ulo, uhi = _block(2 * num_gates, world, rank)
    if uhi <= ulo:
        raise ValueError("more ranks than half-gate units")
    lo, hi = (ulo + 1) // 2, uhi // 2
    half = None
    if ulo % 2 == 1:
        half = (ulo // 2, 2)
    if uhi % 2 == 1:
        if half is not None:  # cannot happen with balanced blocks
            raise ValueError("a rank would own two half gates")
        half = (uhi // 2, 1)
    return lo, hi, half


def half_angle_rows(num_angles: int, part: int) -> list[int]:
    """Sinogram rows (angles) of half ``part`` (1 or 2) of a gate: the mirror pairs
    (q, A-q) with q < 1 + P//2 plus the self-paired angles 0 (and A/2) for part 1,
    the remaining pairs for part 2 (P = (A-1)//2; csrc mct_half_q)."""
    if part not in (1, 2):
        raise ValueError("part must be 1 or 2")
    A = int(num_angles)
    npairs = (A - 1) // 2
    hq = 1 + npairs // 2
    if part == 1:
        qs, singles = range(1, hq), [0] + ([A // 2] if A % 2 == 0 and A >= 2 else [])
    else:
        qs, singles = range(hq, npairs + 1), []
    return sorted(singles + list(qs) + [A - q for q in qs])


def slice_shard(num_slices: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice block of ``rank`` for the batch workload (no collective)."""
    return _block(num_slices, world, rank)


def exchange_schedule(epoch: int) -> tuple[int, int]:
    """(flag value, buffer parity) of the p2p exchange of PDHG iteration ``epoch``
    (0-based): flags count from 1 (pads start zeroed) and the partial buffers
    alternate, so a rank rewrites a buffer only after every peer has posted the
    next iteration (see csrc/exchange_kernels.cu)."""
    if epoch < 0:
        raise ValueError("epoch must be >= 0")
    return epoch + 1, (epoch + 1) % 2


def _align(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


class P2PExchange:
    """Peer-memory exchange of gate-sharded PDHG partials (``mct_exchange_*``).

    One symmetric allocation per rank holds two partial buffers (iteration
    parity) and a signal pad of ``world`` uint64 slots; ``rendezvous`` maps every
    peer's allocation into this process (NVLink / NVSwitch peer addresses).
    """

    def __init__(self, n: int, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        from . import _lib

        self.torch, self._lib = torch, _lib
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.n = int(n)
        part = _align(4 * self.n)
        pad_off = 2 * part
        dev = torch.device("cuda", torch.cuda.current_device())
        self.buf = symm.empty(pad_off + _align(8 * self.world), dtype=torch.uint8, device=dev)
        self.buf.zero_()
        self.handle = symm.rendezvous(self.buf, self.group)
        peers = [int(p) for p in self.handle.buffer_ptrs]
        if len(peers) != self.world:
            raise RuntimeError("symmetric-memory rendezvous returned a wrong peer count")
        i64 = torch.int64
        self.parts_dev = [torch.tensor([p + k * part for p in peers], dtype=i64, device=dev)
                          for k in (0, 1)]
        self.pads_dev = torch.tensor([p + pad_off for p in peers], dtype=i64, device=dev)
        self.my_pad = self.buf.data_ptr() + pad_off
        self.partials = [self.buf[k * part:k * part + 4 * self.n].view(torch.float32)
                         for k in (0, 1)]
        self.failed = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = 0  # iterations exchanged so far
        torch.cuda.synchronize()
        dist.barrier(self.group)  # every pad is zero before the first post

    def partial(self):
        """The buffer K4 writes this iteration's partial into."""
        return self.partials[exchange_schedule(self.epoch)[1]]

    def exchange(self, z, zbar, theta: float) -> None:
        """Post this rank's partial, then z += sum_q partial_q, zbar = z + theta*sum."""
        L, lib = self._lib.load(), self._lib
        flag, parity = exchange_schedule(self.epoch)
        st = lib.stream_handle()
        lib.check(L.mct_exchange_post(lib.ptr(self.pads_dev), self.world, self.rank, flag, st))
        lib.check(L.mct_exchange_z_update(lib.ptr(self.parts_dev[parity]), self.my_pad,
                                          self.world, flag, self.n, lib.ptr(z), lib.ptr(zbar),
                                          float(theta), lib.ptr(self.failed), st))
        self.epoch += 1

    def check(self) -> None:
        if int(self.failed.item()):
            raise RuntimeError("p2p exchange timed out waiting for a peer's partial")


class ShardWorker(Protocol):
    def local_iteration(self):
        """Run the local gates of one PDHG iteration; return the partial dz tensor."""

    def finish(self, dz) -> None:
        """Apply the globally reduced dz: z += dz; zbar = z + theta*dz."""


def sharded_epochs(worker: ShardWorker, epochs: int, group=None) -> None:
    """PDHG epochs with one image-sized sum per iteration (allreduce, or the
    worker's own p2p exchange inside ``finish``)."""
    import torch.distributed as dist

    nccl = getattr(worker, "exchange", "nccl") == "nccl"
    for _ in range(epochs):
        dz = worker.local_iteration()
        if (nccl and dist.is_available() and dist.is_initialized()
                and dist.get_world_size(group) > 1):
            dist.all_reduce(dz, op=dist.ReduceOp.SUM, group=group)
        worker.finish(dz)


class ShardedPDHG:
    """GPU worker: the fused K1..K4 kernels on the local gate block."""

    def __init__(self, config, problem, rank: int, world: int, keep_projections=False,
                 exchange: str = "nccl", group=None):
        from .engine import Engine

        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        if config.mode != "pdhg":
            raise ValueError("gate sharding applies to pdhg (spdhg runs as replicas)")
        if config.num_gates != problem.num_gates:
            raise ValueError("config and problem disagree on the gate count")
        # half-gate units: every rank gets 2N/world units (whole gates + at most one
        # half gate), so 20 gates on 8 ranks is 2.5 gates each instead of 3 or 2
        self.lo, self.hi, self.half = unit_shard(problem.num_gates, world, rank)
        if self.hi <= self.lo and self.half is None:
            raise ValueError("more ranks than half-gate units")
        # gates whose data this rank reads (contiguous: the half gate is lo-1 or hi)
        hg = [self.half[0]] if self.half is not None else []
        self.data_lo = min([self.lo] + hg)
        self.data_hi = max([self.hi] + [g + 1 for g in hg])
        self.engine = Engine([problem.operators], [problem.data], gate_range=(self.lo, self.hi),
                             keep_projections=keep_projections, half=self.half)
        self.engine.set_params(config)
        self.engine.reset()
        self.alpha = problem.alpha
        self.theta = config.theta
        self.exchange = exchange
        self.p2p = P2PExchange(self.engine.x.numel(), group) if exchange == "p2p" else None
        self.dz = None if self.p2p else self.engine.torch.zeros_like(self.engine.x)

    def partial_buffer(self):
        """Where K4 writes this iteration's partial sum (shape of x)."""
        return self.p2p.partial().view(self.engine.x.shape) if self.p2p else self.dz

    def local_iteration(self):
        eng = self.engine
        dz = self.partial_buffer()
        eng.iteration(eng.items_pdhg(epoch_ctr=True), self.alpha, dz=dz)
        return dz

    def reduce_update(self, dz, group=None):
        """Sum the partials over the ranks and apply the z / z-bar update."""
        if self.p2p:
            self.p2p.exchange(self.engine.z, self.engine.zbar, self.theta)
            return
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(dz, op=dist.ReduceOp.SUM, group=group)
        self.engine.z_update(dz, self.theta)

    def finish(self, dz):
        if self.p2p:
            self.p2p.exchange(self.engine.z, self.engine.zbar, self.theta)
        else:
            self.engine.z_update(dz, self.theta)
        self.engine.advance_epoch()

    def check(self):
        if self.p2p:
            self.p2p.check()

    def p2p_failed_anywhere(self, group=None) -> bool:
        """True when any rank's p2p exchange timed out (collective over the group)."""
        import torch.distributed as dist

        flag = self.engine.torch.zeros(1, dtype=self.engine.torch.int32,
                                       device=self.engine.device)
        if self.p2p is not None:
            flag.copy_(self.p2p.failed)
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        return bool(int(flag.item()))

    def fallback_to_nccl(self):
        """Switch this worker to the NCCL exchange and restart from the zero state."""
        self.p2p = None
        self.exchange = "nccl"
        self.dz = self.engine.torch.zeros_like(self.engine.x)
        self.engine.reset()


def run_pdhg_sharded(config, problem, group=None, exchange: str = "nccl"):
    """PDHG over the ranks of ``group``; returns x (float64 numpy) on every rank.

    ``exchange="p2p"`` needs an initialised NCCL process group (symmetric-memory
    rendezvous); ``"nccl"`` also runs without one (single process).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    w = ShardedPDHG(config, problem, rank, world, exchange=exchange, group=group)
    sharded_epochs(w, config.epochs, group)
    from .solvers import _raise_status

    # A timed-out peer wait leaves the waiting rank's z / zbar stale, and its later
    # partials corrupt every rank: agree on the failure collectively so that every
    # rank raises, not only the one whose wait timed out.
    if w.p2p is not None and w.p2p_failed_anywhere(group):
        raise RuntimeError("p2p exchange timed out waiting for a peer's partial "
                           "(on at least one rank); the iterate is invalid")
    _raise_status(w.engine)
    return np.asarray(w.engine.x[0].double().cpu().numpy())
