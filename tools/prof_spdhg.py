"""SPDHG iteration breakdown: per-kernel CUDA-event times (eager) vs the graph epoch.

Prints, for the chosen workload, the average duration of K1..K4 of a single-gate
SPDHG iteration (events recorded between the launches on the launching stream)
and the per-epoch time of the captured CUDA graph, so the launch / tail
overhead of the graph is visible as (graph epoch - N * sum(K)).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--epochs", type=int, default=20)
args = ap.parse_args()

import ctypes  # noqa: E402

import torch  # noqa: E402

import paper_2410_10503_b200 as m  # noqa: E402
from paper_2410_10503_b200 import _lib, workloads  # noqa: E402
from paper_2410_10503_b200.engine import Engine, KernelTimer  # noqa: E402

cfg = workloads.CONFIGS[args.config]
inp = workloads.slice_inputs(cfg, 0)
geom = m.Geometry(*cfg.geometry_args)
ops = m.gate_operators(geom, inp.gates)
rng = np.random.default_rng(0)
data = [rng.standard_normal(geom.sino_shape).astype(np.float32) for _ in ops]
problem = m.Problem.from_parts(cfg.alpha, ops, data)
norm = float(np.sqrt(0.966 * cfg.num_angles * cfg.n))
c = m.default_config("spdhg", [norm] * cfg.num_gates, cfg.alpha, args.epochs + 10)
eng = Engine([problem.operators], [problem.data])
eng.set_params(c)
eng.reset()
eng.set_sequences(m.draw_sequence(c)[None])
L = _lib.load()
N = cfg.num_gates
stream = torch.cuda.current_stream()


def iteration(k, timer=None):
    eng.iteration(eng.items_spdhg(k), cfg.alpha, mark=timer)


for k in range(2 * N):
    iteration(k % N)
torch.cuda.synchronize()
K = args.epochs * N
timers = [KernelTimer(torch, stream) for _ in range(K)]
for k in range(K):
    iteration(k % N, timers[k])
torch.cuda.synchronize()
per = np.array([t.times_ms() for t in timers])
eng.reset()
g = eng.epoch_graph("spdhg", cfg.alpha)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(args.epochs):
    g.replay()
e.record()
torch.cuda.synchronize()
graph_ms = s.elapsed_time(e) / args.epochs
out = {
    "config": args.config,
    "kernel_ms": dict(zip(["K1", "K2", "K3", "K4"], per.mean(0).tolist())),
    "kernel_ms_median": dict(zip(["K1", "K2", "K3", "K4"], np.median(per, 0).tolist())),
    "eager_iter_ms": float(per.sum(1).mean()),
    "graph_epoch_ms": graph_ms,
    "graph_iter_ms": graph_ms / N,
    "overhead_per_iter_ms": graph_ms / N - float(np.median(per, 0).sum()),
    "status": eng.read_status(),
}
print(json.dumps(out))
