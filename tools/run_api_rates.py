"""Wall-clock rates of the public ``run()`` API (warm engine, one run timed) for
C1 and C3, PDHG and SPDHG, with diagnostics off / on / on + rmse to the phantom.
Step sizes from the analytic norm estimate ||A||^2 ~ 0.966*A*n (timing only)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_10503_b200 as m  # noqa: E402
from paper_2410_10503_b200 import workloads  # noqa: E402

for name, epochs in (("c1", 400), ("c3", 50)):
    cfg = workloads.CONFIGS[name]
    problem, truth, _ = m.simulate.workload_problem(cfg, 0)
    norm = float(np.sqrt(0.966 * cfg.num_angles * cfg.n))
    for mode in ("pdhg", "spdhg"):
        c = m.default_config(mode, [norm] * cfg.num_gates, cfg.alpha, epochs, seed=1,
                             stacked_norm_sq=norm**2 * cfg.num_gates if mode == "pdhg" else None)
        for kw in (dict(diagnostics=False), dict(diagnostics=True),
                   dict(diagnostics=True, truth=truth)):
            m.run(c, problem, **kw)
            torch.cuda.synchronize()
            t = time.perf_counter()
            m.run(c, problem, **kw)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            print(name, mode, epochs, sorted(kw), round(epochs / dt, 1), "epochs/s")
