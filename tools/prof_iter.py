"""Profiling driver: C3-shaped fused iterations without setup noise.

Builds the C3 gate family (20 dense warps), random data, analytic step sizes,
then runs `--iters` eager iterations (4 launches each: pack_kernel,
fwd_kernel<1>, adj_kernel<0>, update_kernel<1>).  Used under ncu so launch
counts are predictable:  -k regex:'fwd_kernel|adj_kernel|pack_kernel|update_kernel'
-s 4 -c 4  captures the second iteration.
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--mode", default="pdhg")
args = ap.parse_args()

import torch  # noqa: E402

import paper_2410_10503_b200 as m  # noqa: E402
from paper_2410_10503_b200 import workloads  # noqa: E402
from paper_2410_10503_b200.engine import Engine  # noqa: E402

cfg = workloads.CONFIGS[args.config]
inp = workloads.slice_inputs(cfg, 0)
geom = m.Geometry(*cfg.geometry_args)
ops = m.gate_operators(geom, inp.gates)
rng = np.random.default_rng(0)
data = [rng.standard_normal(geom.sino_shape).astype(np.float32) for _ in ops]
problem = m.Problem.from_parts(cfg.alpha, ops, data)
norm = float(np.sqrt(0.966 * cfg.num_angles * cfg.n))
c = m.default_config(args.mode, [norm] * cfg.num_gates, cfg.alpha, 1)
eng = Engine([problem.operators], [problem.data])
eng.set_params(c)
eng.reset()
if args.mode == "spdhg":
    eng.set_sequences(m.draw_sequence(c, 4 * cfg.num_gates)[None])
torch.cuda.synchronize()
for k in range(args.iters):
    if args.mode == "pdhg":
        eng.iteration(eng.items_pdhg(iteration=k + 1), cfg.alpha)
    else:
        eng.iteration(eng.items_spdhg(k), cfg.alpha)
torch.cuda.synchronize()
print("ok", eng.read_status())
