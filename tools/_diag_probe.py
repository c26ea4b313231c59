import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2410_10503_b200 as m
from paper_2410_10503_b200 import workloads
for name, E in (('c1', 400), ('c3', 50)):
    cfg = workloads.CONFIGS[name]
    problem, truth, inp = m.simulate.workload_problem(cfg, 0)
    norm = float(np.sqrt(0.966 * cfg.num_angles * cfg.n))
    for mode in ('pdhg', 'spdhg'):
        c = m.default_config(mode, [norm]*cfg.num_gates, cfg.alpha, E, seed=1, stacked_norm_sq=norm**2*cfg.num_gates if mode=='pdhg' else None)
        for kw in (dict(diagnostics=False), dict(diagnostics=True), dict(diagnostics=True, truth=truth)):
            m.run(c, problem, **kw); torch.cuda.synchronize()
            t = time.perf_counter(); m.run(c, problem, **kw); torch.cuda.synchronize()
            dt = time.perf_counter()-t
            print(name, mode, E, list(kw), round(E/dt, 1), 'epochs/s')
