"""CPU tier: the multi-GPU host logic with gloo, world_size 2 and 3.

The gate-sharded PDHG protocol of paper_2410_10503_b200.distributed (contiguous
blocks of half-gate units, replicated prox step, one allreduce(sum) of the image-sized update
per iteration, then z += dz; zbar = z + theta*dz) is driven here by an
oracle-backed worker (test infrastructure) and must reproduce the
single-process PDHG trajectory of the reference restatement.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import solver as osolver
from paper_2410_10503_b200 import workloads
from paper_2410_10503_b200.distributed import (gate_shard, half_angle_rows, sharded_epochs,
                                               slice_shard, unit_shard)


def test_gate_shard_blocks():
    assert [gate_shard(20, 8, r) for r in range(8)] == [
        (0, 3), (3, 6), (6, 9), (9, 12), (12, 14), (14, 16), (16, 18), (18, 20)]
    assert [gate_shard(40, 8, r)[1] - gate_shard(40, 8, r)[0] for r in range(8)] == [5] * 8
    assert gate_shard(4, 1, 0) == (0, 4)
    assert [slice_shard(64, 8, r) for r in (0, 7)] == [(0, 8), (56, 64)]
    with pytest.raises(ValueError):
        gate_shard(4, 2, 2)


@pytest.mark.parametrize("gates", [1, 2, 3, 4, 5, 7, 10, 20, 40])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 6, 7, 8])
def test_unit_shard_covers_every_half_gate_once(gates, world):
    """Half-gate units: every (gate, half) is owned by exactly one rank, ranks hold
    2N/world units (+-1), at most one half gate each, adjacent to their full gates."""
    if 2 * gates < world:
        with pytest.raises(ValueError):
            [unit_shard(gates, world, r) for r in range(world)]
        return
    seen = []
    for r in range(world):
        lo, hi, half = unit_shard(gates, world, r)
        units = [(g, h) for g in range(lo, hi) for h in (1, 2)]
        if half is not None:
            g, part = half
            assert part in (1, 2) and (g == lo - 1 or g == hi)
            units.append(half)
        assert abs(len(units) - 2 * gates / world) < 1
        seen += units
    assert sorted(seen) == [(g, h) for g in range(gates) for h in (1, 2)]
    assert unit_shard(20, 8, 0) == (0, 2, (2, 1)) and unit_shard(20, 8, 1) == (3, 5, (2, 2))
    assert all(unit_shard(40, 8, r)[2] is None for r in range(8))


@pytest.mark.parametrize("A", [1, 2, 3, 36, 37, 720])
def test_half_angle_rows_partition(A):
    a, b = half_angle_rows(A, 1), half_angle_rows(A, 2)
    assert sorted(a + b) == list(range(A))
    assert not set(a) & set(b)


class OracleShardWorker:
    """Same protocol as distributed.ShardedPDHG (half-gate units: whole gates plus at
    most one gate restricted to half of its angles), computed by the fp64 oracle."""

    def __init__(self, cfg, alpha, ops, data, rank, world):
        self.cfg, self.alpha, self.ops, self.data = cfg, alpha, ops, data
        self.lo, self.hi, half = unit_shard(len(ops), world, rank)
        # (gate, sinogram-row mask or None)
        self.units = [(i, None) for i in range(self.lo, self.hi)]
        if half is not None:
            mask = np.zeros(data[half[0]].shape[0], dtype=bool)
            mask[half_angle_rows(len(mask), half[1])] = True
            self.units.append((half[0], mask))
        shape = ops[0].domain_shape
        self.x = np.zeros(shape)
        self.z = np.zeros(shape)
        self.zbar = np.zeros(shape)
        self.y = {i: np.zeros(data[i].shape) for i, _ in self.units}

    def local_iteration(self):
        c = self.cfg
        n = len(self.ops)
        self.x_new = osolver.prox_g(self.alpha, c.tau, self.x - c.tau * self.zbar)
        dz = np.zeros_like(self.x)
        for i, mask in self.units:
            proj = self.ops[i].apply(self.x_new)
            y_new = osolver.prox_fstar(n, self.data[i], c.sigmas[i], self.y[i] + c.sigmas[i] * proj)
            if mask is not None:  # this rank owns only these angles of gate i
                y_new = np.where(mask[:, None], y_new, self.y[i])
            dz += self.ops[i].adjoint_apply(y_new - self.y[i])
            self.y[i] = y_new
        return torch.from_numpy(dz)

    def finish(self, dz):
        d = dz.numpy()
        self.z = self.z + d
        self.zbar = self.z + self.cfg.theta * d
        self.x = self.x_new


class OracleP2PWorker(OracleShardWorker):
    """The p2p protocol of distributed.P2PExchange, emulated on CPU: partials in
    parity buffers, exchange = gather every rank's buffer of this parity and sum in
    rank order inside the z update (the arithmetic of exchange_update_kernel)."""

    exchange = "p2p"

    def __init__(self, *a):
        super().__init__(*a)
        from paper_2410_10503_b200.distributed import exchange_schedule

        self.schedule = exchange_schedule
        self.bufs = [torch.zeros(self.x.shape, dtype=torch.float64) for _ in range(2)]
        self.epoch = 0

    def local_iteration(self):
        dz = super().local_iteration()
        buf = self.bufs[self.schedule(self.epoch)[1]]
        buf.copy_(dz)
        return buf

    def finish(self, dz):
        parts = [torch.zeros_like(dz) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, self.bufs[self.schedule(self.epoch)[1]])
        s = parts[0].clone()
        for q in parts[1:]:
            s += q
        super().finish(s)
        self.epoch += 1


def _problem():
    cfgw = workloads.WorkloadConfig("dist", 40, 36, 59, 5, "dense", 4, 1e-2, 6, peak=2.0)
    inp = workloads.slice_inputs(cfgw, 0)
    geom = oracle.Geometry(*cfgw.geometry_args)
    ops = oracle.gate_operators(geom, inp.gates)
    clean = [op.apply(inp.phantom.astype(np.float64)) for op in ops]
    data = [d.astype(np.float64) for d in workloads.noisy_data(clean, inp.seed)]
    norms = [osolver.power_method(op, iterations=30) for op in ops]
    cfg = osolver.default_config("pdhg", norms, cfgw.alpha, cfgw.epochs,
                                 stacked_norm_sq=osolver.stacked_norm_sq(ops, iterations=30))
    return cfg, cfgw.alpha, ops, data


def _worker(rank, world, port, out_path, kind="nccl"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, alpha, ops, data = _problem()
        cls = OracleP2PWorker if kind == "p2p" else OracleShardWorker
        w = cls(cfg, alpha, ops, data, rank, world)
        sharded_epochs(w, cfg.epochs)
        if rank == 0:
            np.save(out_path, w.x)
        else:
            np.save(out_path.replace(".npy", f"_r{rank}.npy"), w.x)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind,world", [("nccl", 2), ("p2p", 2), ("nccl", 3)])
def test_gate_sharded_pdhg_gloo_matches_single_process(tmp_path, kind, world):
    """5 gates on 2 ranks (2.5 each: gate 2 split by angle halves) or 3 ranks."""
    out = str(tmp_path / "x.npy")
    mp.spawn(_worker, args=(world, _free_port(), out, kind), nprocs=world, join=True)
    x0 = np.load(out)
    for r in range(1, world):
        # replicated primal stays identical on every rank
        assert np.array_equal(x0, np.load(out.replace(".npy", f"_r{r}.npy")))
    cfg, alpha, ops, data = _problem()
    st, _ = osolver.run(cfg, alpha, ops, data, diagnostics=False)
    assert np.linalg.norm(x0 - st.x) <= 1e-12 * np.linalg.norm(st.x)


def test_p2p_exchange_schedule():
    """Flags start at 1 (pads are zeroed) and increase by one per iteration; the
    partial buffers alternate, so a buffer is rewritten two iterations later —
    after every peer has posted the iteration in between (exchange_kernels.cu)."""
    from paper_2410_10503_b200.distributed import exchange_schedule

    sched = [exchange_schedule(e) for e in range(6)]
    assert [f for f, _ in sched] == [1, 2, 3, 4, 5, 6]
    assert [p for _, p in sched] == [1, 0, 1, 0, 1, 0]
    for e in range(4):
        assert exchange_schedule(e)[1] == exchange_schedule(e + 2)[1]
        assert exchange_schedule(e)[1] != exchange_schedule(e + 1)[1]
    with pytest.raises(ValueError):
        exchange_schedule(-1)
