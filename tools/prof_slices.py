"""Small-grid tax of single-gate SPDHG: per-kernel CUDA-event times of one SPDHG
iteration for S independent slices in the same launches (S = 1, 2, 4, 8 copies of the
C3 problem, one gate each per iteration), printed per slice.  S = 1 is the SPDHG
bench; a per-slice time falling with S is the launch's ramp / tail / fragmentation
cost that a single-gate iteration pays."""
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

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
SLICES = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
inp = workloads.slice_inputs(cfg, 0)
geom = m.Geometry(*cfg.geometry_args)
ops = m.gate_operators(geom, inp.gates)
rng = np.random.default_rng(0)
data = [rng.standard_normal(geom.sino_shape).astype(np.float32) for _ in ops]
problem = m.Problem.from_parts(cfg.alpha, ops, data)
norm = float(np.sqrt(0.966 * cfg.num_angles * cfg.n))
c = m.default_config("spdhg", [norm] * cfg.num_gates, cfg.alpha, 50)
L = _lib.load()
out = {}
for S in SLICES:
    eng = Engine([problem.operators] * S, [problem.data] * S, max_items=S)
    eng.set_params(c)
    eng.reset()
    eng.set_sequences(np.stack([m.draw_sequence(c, 60 * cfg.num_gates)] * S))
    stream = torch.cuda.current_stream()

    def iteration(k, timer=None):
        eng.iteration(eng.items_spdhg(k), cfg.alpha, mark=timer)

    for k in range(2 * cfg.num_gates):
        iteration(k % cfg.num_gates)
    torch.cuda.synchronize()
    K = 2 * cfg.num_gates
    timers = [KernelTimer(torch, stream) for _ in range(K)]
    for k in range(K):
        iteration(k % cfg.num_gates, timers[k])
    torch.cuda.synchronize()
    per = np.median([t.times_ms() for t in timers], axis=0)
    out[S] = {n: round(1000 * float(v) / S, 1) for n, v in zip(("K1", "K2", "K3", "K4"), per)}
    out[S]["sum"] = round(sum(out[S][n] for n in ("K1", "K2", "K3", "K4")), 1)
    del eng
    torch.cuda.empty_cache()
print(json.dumps({"config": cfg.name, "unit": "us per slice-iteration", "per_S": out}))
