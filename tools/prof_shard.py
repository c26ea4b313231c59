"""Per-kernel times of one gate-sharded PDHG iteration for local gate counts
k = 2, 2.5, 3, 5, 10, 20 (what one rank of an N-GPU run executes at C3; k.5 = k
whole gates + one half-gate unit), eager launches with CUDA events between the
kernels (K4 in partial mode)."""
import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_10503_b200 as m  # noqa: E402
from paper_2410_10503_b200 import _lib, workloads  # noqa: E402
from paper_2410_10503_b200.engine import Engine, KernelTimer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--locals", default="2,2.5,3,5,10,20")
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
cfg = workloads.CONFIGS[args.config]
inp = workloads.slice_inputs(cfg, 0)
geom = m.Geometry(*cfg.geometry_args)
ops = m.gate_operators(geom, inp.gates)
rng = np.random.default_rng(0)
data = [rng.standard_normal(geom.sino_shape).astype(np.float32) for _ in ops]
problem = m.Problem.from_parts(cfg.alpha, ops, data)
norm = float(np.sqrt(0.966 * cfg.num_angles * cfg.n))
c = m.default_config("pdhg", [norm] * cfg.num_gates, cfg.alpha, 1,
                     stacked_norm_sq=norm**2 * cfg.num_gates)
L = _lib.load()
stream = torch.cuda.current_stream()
out = {}
for kk in args.locals.split(","):
    k = int(float(kk))
    half = (k, 1) if float(kk) != k else None
    eng = Engine([problem.operators], [problem.data], gate_range=(0, k), half=half)
    eng.set_params(c)
    eng.reset()
    dz = torch.zeros_like(eng.x)
    items = eng.items_pdhg(epoch_ctr=True)
    per = []
    for it in range(args.iters + 3):
        timer = KernelTimer(torch, stream)
        eng.iteration(items, cfg.alpha, dz=dz, mark=timer)
        eng.z_update(dz, c.theta)
        eng.advance_epoch()
        if it >= 3:
            per.append(timer)
    torch.cuda.synchronize()
    t = np.array([tm.times_ms() for tm in per])
    med = np.median(t, 0)
    out[kk] = {"K1": round(float(med[0]) * 1e3, 1), "K2": round(float(med[1]) * 1e3, 1),
              "K3": round(float(med[2]) * 1e3, 1), "K4": round(float(med[3]) * 1e3, 1),
              "sum_us": round(float(med.sum()) * 1e3, 1)}
    print(kk, json.dumps(out[kk]))
    del eng
