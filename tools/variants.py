"""Tuning aid (not product): build -D variants of the sm_100a library here (nvcc
cross-compiles) and time them on the GPU box without rebuilding there.

    python tools/variants.py build name1="-DADJ_PPT2=2" name2="-DFWD_MIN_BLOCKS_M=8" ...
    python tools/variants.py run [--steps 50]      # on the GPU box

``build`` writes paper_2410_10503_b200/_native/var/<name>.so (git-ignored, travels
with the gpurun snapshot) plus the ptxas log; ``run`` times every built variant (and
the default library) with bench.py through MCT_LIB and prints one line per variant:
PDHG / SPDHG epochs/s and the per-kernel event times of the PDHG step.
"""

import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
VAR = ROOT / "paper_2410_10503_b200" / "_native" / "var"


def build_one(name, defs):
    from paper_2410_10503_b200 import build as b

    VAR.mkdir(parents=True, exist_ok=True)
    out = VAR / f"{name}.so"
    cmd = [b._nvcc(), *b.ARCH_FLAGS, *b.NVCC_FLAGS, *defs.split(), "-I", str(ROOT / "include"),
           "-o", str(out)] + [str(s) for s in b.sources()]
    p = subprocess.run(cmd, capture_output=True, text=True)
    (VAR / f"{name}.log").write_text(defs + "\n" + p.stdout + p.stderr)
    return name, p.returncode


def run(steps, extra):
    names = ["default"] + sorted(p.stem for p in VAR.glob("*.so"))
    for name in names:
        env = dict(os.environ)
        if name != "default":
            env["MCT_LIB"] = str(VAR / f"{name}.so")
        p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--no-cpu-baseline", "--no-e2e",
                            "--steps", str(steps), "--warmup", "5", *extra], capture_output=True,
                           text=True, env=env, cwd=ROOT)
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
            ker = d.get("kernel_ms") or d.get("kernel_ms_per_epoch_rank0")
            sp = (d.get("spdhg") or {}).get("value")
            print(name, round(d["value"], 1), {k[:2]: round(v, 4) for k, v in ker.items()},
                  "spdhg", round(sp, 1) if sp else None, flush=True)
        except Exception:
            print(name, "FAILED", p.stderr[-400:].replace("\n", " | "), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        jobs = [a.split("=", 1) for a in sys.argv[2:]]
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            for name, rc in ex.map(lambda j: build_one(*j), jobs):
                print(name, "ok" if rc == 0 else "BUILD FAILED")
    else:
        steps = 50
        extra = []
        args = sys.argv[2:]
        if args and args[0] == "--steps":
            steps = int(args[1])
            args = args[2:]
        run(steps, args)
