"""CPU tier: the C-ABI library builds, loads without a GPU and exports every
symbol include/mctomo_b200.h declares; argument errors map to ValueError
before any device work (linops.py:59-73 error behaviour)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2410_10503_b200 import _lib
from paper_2410_10503_b200.build import LIB_PATH, build_native

HEADER = Path(__file__).resolve().parent.parent / "include" / "mctomo_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(mct_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    build_native()
    assert LIB_PATH.exists()
    L = _lib.load()
    assert L.mct_abi_version() == 2


def test_every_declared_symbol_is_exported_and_bound():
    L = ctypes.CDLL(str(LIB_PATH))
    names = declared_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(names)


def test_sm100a_cubin_embedded():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("args,msg", [
    ((0, 8, 4, 8, 1.0), "rows"),
    ((8, 8, 0, 8, 1.0), "num_angles"),
    ((8, 8, 4, 8, -1.0), "detector_spacing"),
    ((32768, 32768, 4, 8, 1.0), "2\\^29 pixels"),
])
def test_plan_validation_maps_to_value_error(args, msg):
    L = _lib.load()
    h = ctypes.c_void_p()
    c = np.ones(8)
    with pytest.raises(ValueError, match=msg):
        _lib.check(L.mct_ray_plan_create(ctypes.byref(h), *args, c.ctypes.data, c.ctypes.data,
                                         c.astype(np.uint8).ctypes.data))
    assert not h


def test_null_arguments_rejected():
    L = _lib.load()
    with pytest.raises(ValueError):
        _lib.check(L.mct_ray_forward(None, None, None, 1, None, None))
    with pytest.raises(ValueError):
        _lib.check(L.mct_reduce(None, None, 10, 1, 10, 0, None, None, None))
    with pytest.raises(ValueError):
        _lib.check(L.mct_warp_plan_create_dilatation(ctypes.byref(ctypes.c_void_p()), 4, 4, 0.0))


def _build_c_demo(tmp_path):
    import shutil
    import subprocess

    cc = shutil.which("cc") or shutil.which("gcc")
    cuda = Path("/usr/local/cuda")
    if cc is None or not (cuda / "include" / "cuda_runtime.h").exists():
        pytest.skip("no C compiler / CUDA headers")
    build_native()
    root = HEADER.parent.parent
    exe = tmp_path / "c_abi_demo"
    cmd = [cc, "-O2", "-I", str(root / "include"), "-I", str(cuda / "include"),
           str(root / "examples" / "c_abi_demo.c"), "-L", str(LIB_PATH.parent), "-lmctomo_b200",
           "-L", str(cuda / "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{LIB_PATH.parent}",
           "-o", str(exe)]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_c_abi_demo_compiles_without_python_types(tmp_path):
    """examples/c_abi_demo.c uses the boundary from plain C (no torch, no Python)."""
    assert _build_c_demo(tmp_path).exists()


@pytest.mark.gpu
def test_c_abi_demo_runs(tmp_path):
    import subprocess

    exe = _build_c_demo(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "rel =" in out.stdout
