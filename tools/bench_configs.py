#!/usr/bin/env python
"""Throughput of every BASELINE.json config on one GPU (supplements bench.py's C3 line).

    python tools/bench_configs.py [--configs c1,c2,c3,c4,c5] [--epochs K] [--out profiles/r01/configs.json]

Per config: PDHG and/or SPDHG epochs/s (CUDA graphs, CUDA events, warm-up 3,
solver work only), C4 additionally the standalone A_i / A_i^* / D_i / D_i^*
operator sweep, C5 the 64-slice batched SPDHG (one launch per kernel for all
slices).  Step sizes come from device power iterations (20 its, slice 0;
C5 scales them by 1.1 so every slice's steps stay admissible).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2410_10503_b200 as m  # noqa: E402
from paper_2410_10503_b200 import workloads  # noqa: E402
from paper_2410_10503_b200.engine import Engine  # noqa: E402


def events(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def epoch_rate(problems, cfgs, mode, epochs):
    S = len(problems)
    eng = Engine([p.operators for p in problems], [p.data for p in problems],
                 max_items=S if mode == "spdhg" else None)
    eng.set_params(cfgs[0])
    eng.reset()
    if mode == "spdhg":
        eng.set_sequences(np.stack([m.draw_sequence(c, (epochs + 3) * c.num_gates) for c in cfgs]))
    g = eng.epoch_graph(mode, problems[0].alpha)
    for _ in range(3):
        g.replay()
    ms = events(g.replay, epochs)
    primal, dual = eng.read_status()
    assert primal is None and dual is None, (primal, dual)
    del g, eng
    torch.cuda.empty_cache()
    return 1000.0 / ms, ms


def run_config(name, epochs):
    cfg = workloads.CONFIGS[name]
    out = {"config": name, "n": cfg.n, "angles": cfg.num_angles, "bins": cfg.num_bins,
           "gates": cfg.num_gates, "motion": cfg.motion, "batch": cfg.batch}
    t0 = time.time()
    problem, truth, _ = m.simulate.workload_problem(cfg, 0)
    norms = [m.power_method(op, iterations=20) for op in problem.operators]
    out["setup_s"] = time.time() - t0
    S = cfg.samples
    if name == "c4":
        # standalone operator sweep (A_i, A_i^*, D_i, D_i^*) on gate 0
        op = problem.operators[0]
        x = torch.rand(op.domain_shape, device="cuda")
        y = torch.rand(op.range_shape, device="cuda")
        ray = op.outer
        w = op.inner
        sweep = {
            "A_i": events(lambda: op.apply_device(x), 5),
            "A_i^*": events(lambda: op.adjoint_device(y), 5),
            "A": events(lambda: ray.apply_device(x), 5),
            "A^*": events(lambda: ray.adjoint_device(y), 5),
            "D_i": events(lambda: w.apply_device(x), 20),
            "D_i^*": events(lambda: w.adjoint_device(x), 20),
        }
        out["operator_ms"] = sweep
        out["A_samples_per_s"] = S / (sweep["A"] * 1e-3)
    if cfg.batch > 1:
        probs = [problem] + [m.simulate.workload_problem(cfg, s)[0] for s in range(1, cfg.batch)]
        norms = [1.1 * v for v in norms]
        cfgs = [m.default_config("spdhg", norms, cfg.alpha, epochs, seed=cfg.seed + s)
                for s in range(cfg.batch)]
        out["setup_s"] = time.time() - t0
        rate, ms = epoch_rate(probs, cfgs, "spdhg", epochs)
        out["spdhg_batch_epochs_per_s"] = rate
        out["spdhg_batch_slice_epochs_per_s"] = rate * cfg.batch
        out["ms_per_epoch"] = ms
        out["joseph_samples_per_s"] = 2 * S * cfg.num_gates * cfg.batch / (ms * 1e-3)
        return out
    for mode in cfg.modes if name != "c1" else ("pdhg", "spdhg"):
        stacked = m.stacked_norm_sq(problem.operators, iterations=20) if mode == "pdhg" else None
        c = m.default_config(mode, norms, cfg.alpha, epochs, seed=cfg.seed,
                             stacked_norm_sq=stacked)
        rate, ms = epoch_rate([problem], [c], mode, epochs)
        out[f"{mode}_epochs_per_s"] = rate
        out[f"{mode}_ms_per_epoch"] = ms
        out[f"{mode}_joseph_samples_per_s"] = 2 * S * cfg.num_gates / (ms * 1e-3)
        # the public API with per-epoch diagnostics on (objective + rmse to the
        # phantom every epoch; SURVEY §8d "also report a diagnostics-on number")
        diag_epochs = 200 if name in ("c1", "c2") else 50  # includes run()'s own setup
        cd = m.default_config(mode, norms, cfg.alpha, diag_epochs, seed=cfg.seed,
                              stacked_norm_sq=stacked)
        m.run(cd, problem, truth=truth)  # warm (graphs, diagnostics buffers)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        _, rec = m.run(cd, problem, truth=truth)
        torch.cuda.synchronize()
        out[f"{mode}_run_diagnostics_epochs_per_s"] = diag_epochs / (time.perf_counter() - t1)
        out[f"{mode}_run_final_objective"] = rec.objective[-1]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    m.build_native()
    res = []
    for name in args.configs.split(","):
        r = run_config(name, args.epochs)
        print(json.dumps(r), flush=True)
        res.append(r)
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
