"""In-tree build of the sm_100a C-ABI library (no JIT cache, no pip install).

``build_native()`` compiles ``csrc/*.cu`` with nvcc for ``sm_100a`` into
``paper_2410_10503_b200/_native/libmctomo_b200.so``; the built ``.so`` is
git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
NATIVE_DIR = PKG / "_native"
LIB_NAME = "libmctomo_b200.so"
LIB_PATH = NATIVE_DIR / LIB_NAME

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC,-O2",
    "-Xptxas",
    "-v",
    "-shared",
    "-cudart",
    "static",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the sm_100a library cannot be built")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "mctomo_b200.h"]
    return any(p.stat().st_mtime > t for p in deps if p.is_file())


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile the CUDA library for sm_100a (idempotent unless sources changed)."""
    if not force and not _stale():
        return LIB_PATH
    NATIVE_DIR.mkdir(parents=True, exist_ok=True)
    tmp = LIB_PATH.with_suffix(".so.tmp")
    extra = os.environ.get("MCT_NVCC_EXTRA", "").split()  # tuning experiments only
    cmd = [_nvcc(), *ARCH_FLAGS, *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-o", str(tmp)]
    cmd += [str(s) for s in sources()]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = NATIVE_DIR / "build.log"
    log.write_text(" ".join(cmd) + "\n\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
