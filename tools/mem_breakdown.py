"""Device memory of one PDHG engine per config: device-wide usage deltas
(cudaMemGetInfo, so the C-ABI's own cudaMalloc'ed plans count too) after building the
gated operators' plans (warp fields + transposed D^* lists) and after the engine
(data, duals, state, workspace); torch-allocator bytes beside them."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2410_10503_b200 as m  # noqa: E402
from paper_2410_10503_b200 import workloads  # noqa: E402
from paper_2410_10503_b200.engine import Engine  # noqa: E402


def used():
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    return total - free


out = {}
torch.zeros(1, device="cuda")
for name in sys.argv[1:] or ["c3", "c4"]:
    cfg = workloads.CONFIGS[name]
    u0, t0 = used(), torch.cuda.memory_allocated()
    problem, _, _ = m.simulate.workload_problem(cfg, 0)
    ws_plans = []
    for op in problem.operators:
        w = getattr(op, "inner", None)
        if w is not None and hasattr(w, "plan"):
            ws_plans.append(w.plan())
    u1 = used()
    eng = Engine([problem.operators], [problem.data])
    u2, t2 = used(), torch.cuda.memory_allocated()
    nnz = sum(int(w.nnz) for w in eng.family._warps[0] if w is not None and hasattr(w, "nnz"))
    out[name] = {"plans_bytes": u1 - u0, "engine_bytes": u2 - u1, "total_bytes": u2 - u0,
                 "engine_torch_bytes": t2 - t0, "workspace_bytes": int(eng.ws.numel()),
                 "transposed_list_entries": nnz}
    del eng, problem, ws_plans
    torch.cuda.empty_cache()
print(json.dumps(out))
