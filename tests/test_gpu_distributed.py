"""GPU tier: the real gate-sharded PDHG worker (distributed.ShardedPDHG) in separate
processes.

Each rank is its own process with its own CUDA context on the one visible B200
(gpurun leases one GPU), runs K1..K4 on its half-gate units through the C-ABI and
joins the image-sized partial sum through ``torch.distributed`` (gloo backend on
CUDA tensors: NCCL refuses two ranks on one device).  No kernel waits on another
rank's kernel (the exchange is a host collective), so the ranks cannot deadlock
the device (B200_PROFILING.md: spinning peer waits between processes sharing one
GPU raise Xid 109).  The cross-device p2p flag handshake therefore stays covered
by the emulated-rank test (test_gpu_solver.py::test_p2p_exchange_emulated_ranks).

Bar: every rank ends with identical bits, within 1e-6 of the single-process run()
(the partial sums are added in a different order than K4's gate lanes).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(m):
    from paper_2410_10503_b200 import workloads

    cfgw = workloads.WorkloadConfig("shard_small", 96, 90, 137, 5, "dense", 6, 1e-2, 6, peak=4.0)
    problem, _, _ = m.simulate.workload_problem(cfgw, 0)
    norms = [m.power_method(op, iterations=20, seed=0) for op in problem.operators]
    stacked = m.stacked_norm_sq(problem.operators, iterations=20, seed=0)
    cfg = m.default_config("pdhg", norms, cfgw.alpha, cfgw.epochs, stacked_norm_sq=stacked)
    return cfg, problem


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2410_10503_b200 as m
        from paper_2410_10503_b200.distributed import run_pdhg_sharded, unit_shard

        m.build_native()
        cfg, problem = _problem(m)
        x = run_pdhg_sharded(cfg, problem, exchange="nccl")  # allreduce over the group
        np.save(os.path.join(out_dir, f"x_r{rank}.npy"), x)
        np.save(os.path.join(out_dir, f"units_r{rank}.npy"),
                np.array(unit_shard(problem.num_gates, world, rank), dtype=object),
                allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pdhg_processes_match_single_process(tmp_path, world):
    """5 dense gates on 2 ranks (2.5 gates each: gate 2 split into its two angle
    halves) and on 3 ranks (1.67 gates each), 6 PDHG epochs."""
    import torch.multiprocessing as mp

    import paper_2410_10503_b200 as m

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    xs = [np.load(tmp_path / f"x_r{r}.npy") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(xs[0], xs[r]), f"rank {r} diverged from rank 0"
    halves = [np.load(tmp_path / f"units_r{r}.npy", allow_pickle=True)[2] for r in range(world)]
    assert any(h is not None for h in halves)  # a half-gate unit was exercised
    m.build_native()
    cfg, problem = _problem(m)
    x_run, _ = m.run(cfg, problem, diagnostics=False)
    assert np.linalg.norm(x_run) > 0
    assert np.linalg.norm(xs[0] - x_run) <= 1e-6 * np.linalg.norm(x_run)
