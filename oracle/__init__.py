"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product package).

CPU restatement of the reference algorithm for the motion-compensated PDHG/SPDHG
hot path of arXiv 2410.10503 (`mctomo`, /root/reference/pkg/src/mctomo):

* ``mctomo_oracle.c`` (fp64 C, built by ``build()``) restates the Joseph ray
  transform A / A^* (projector.py:126-217) and the warp D / D^* (motion.py:132-194)
  plus the dense-field warp restatement (src = p + phi(p)).
* ``solver.py`` restates the solver layer in numpy: prox maps
  (functionals.py:40-68), ``default_config`` (solvers.py:198-247), ``step``
  (solvers.py:316-366), ``run`` (solvers.py:369-432), ``power_method`` /
  ``stacked_norm_sq`` (linops.py:215-289), ``sample_gates`` (solvers.py:298-313).

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the *imported reference itself*
(``tests/golden/make_golden.py``), including bitwise known-answer cases.

Allowed importers: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs — as the checker or as the timed CPU
baseline, never as the product path.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD_DIR = HERE / "_build"
LIB_PATH = BUILD_DIR / "libmctomo_oracle.so"
SRC = HERE / "mctomo_oracle.c"

RIGID, DILATATION, DENSE = 1, 2, 3


def build(force: bool = False) -> Path:
    """Compile the fp64 C restatement (gcc, OpenMP, no FMA contraction)."""
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB_PATH
    BUILD_DIR.mkdir(exist_ok=True)
    cmd = [
        "gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
        "-fno-fast-math", "-o", str(LIB_PATH) + ".tmp", str(SRC), "-lm",
    ]
    subprocess.run(cmd, check=True)
    os.replace(str(LIB_PATH) + ".tmp", LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.c_void_p
        u8 = ctypes.c_void_p
        i, d = ctypes.c_int, ctypes.c_double
        L.orc_ray_forward.argtypes = [i, i, i, i, d, dp, dp, u8, dp, dp, i]
        L.orc_ray_adjoint.argtypes = [i, i, i, i, d, dp, dp, u8, dp, dp, i]
        L.orc_warp_forward.argtypes = [i, i, i, d, d, d, d, d, fp, dp, dp]
        L.orc_warp_adjoint.argtypes = [i, i, i, d, d, d, d, d, fp, dp, dp]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Geometry:
    """projector.Geometry restated (projector.py:39-103)."""

    rows: int
    cols: int
    num_angles: int
    num_bins: int
    detector_spacing: float

    @property
    def angles(self) -> np.ndarray:
        return np.arange(self.num_angles) * (math.pi / self.num_angles)  # :73

    @property
    def bin_centers(self) -> np.ndarray:
        offsets = np.arange(self.num_bins) - (self.num_bins - 1) / 2.0  # :78
        return offsets * self.detector_spacing

    @property
    def image_shape(self):
        return (self.rows, self.cols)

    @property
    def sino_shape(self):
        return (self.num_angles, self.num_bins)

    def tables(self):
        ang = self.angles
        cos = np.ascontiguousarray(np.cos(ang))
        sin = np.ascontiguousarray(np.sin(ang))
        rdom = np.ascontiguousarray((np.abs(cos) >= sin).astype(np.uint8))  # :130
        return cos, sin, rdom


class RayTransform:
    """Oracle A / A^* (projector.py:186-217), weights computed on the fly."""

    def __init__(self, geom: Geometry, threads: int | None = None):
        self.geom = geom
        self.domain_shape = geom.image_shape
        self.range_shape = geom.sino_shape
        self._cos, self._sin, self._rdom = geom.tables()
        self.threads = threads or 1

    def _args(self):
        g = self.geom
        return (g.rows, g.cols, g.num_angles, g.num_bins, float(g.detector_spacing),
                _dp(self._cos), _dp(self._sin), self._rdom.ctypes.data)

    def apply(self, x):
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        assert x.shape == self.domain_shape
        out = np.empty(self.range_shape)
        lib().orc_ray_forward(*self._args(), _dp(x), _dp(out), int(self.threads))
        return out

    def adjoint_apply(self, y):
        y = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
        assert y.shape == self.range_shape
        out = np.empty(self.domain_shape)
        lib().orc_ray_adjoint(*self._args(), _dp(y), _dp(out), int(self.threads))
        return out


class Warp:
    """Oracle D / D^* (motion.py:111-194) and the dense restatement."""

    def __init__(self, shape, kind, rotation=0.0, translation=(0.0, 0.0), scale=1.0, phi=None):
        self.domain_shape = self.range_shape = (int(shape[0]), int(shape[1]))
        self.kind = kind
        cs, sn = math.cos(rotation), math.sin(rotation)
        if abs(cs) < 1e-15:  # motion.py:142-147 right-angle snap
            cs = 0.0
        if abs(sn) < 1e-15:
            sn = 0.0
        self._p = (float(cs), float(sn), float(translation[0]), float(translation[1]), float(scale))
        self.identity = kind != DENSE and rotation == 0.0 and tuple(translation) == (0.0, 0.0) \
            and scale == 1.0
        self.phi = None
        if kind == DENSE:
            self.phi = np.ascontiguousarray(np.asarray(phi, dtype=np.float32))
            assert self.phi.shape == (2,) + self.domain_shape

    def _call(self, fn, v):
        v = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
        out = np.empty(self.domain_shape)
        phi = self.phi.ctypes.data if self.phi is not None else None
        fn(self.kind, self.domain_shape[0], self.domain_shape[1], *self._p, phi, _dp(v), _dp(out))
        return out

    def apply(self, x):
        if self.identity:  # motion.py:180-181
            return np.array(x, dtype=np.float64, copy=True)
        return self._call(lib().orc_warp_forward, x)

    def adjoint_apply(self, y):
        if self.identity:  # motion.py:187-188
            return np.array(y, dtype=np.float64, copy=True)
        return self._call(lib().orc_warp_adjoint, y)


class Composed:
    """linops.ComposedMap restated (linops.py:105-123)."""

    def __init__(self, outer, inner):
        self.outer, self.inner = outer, inner
        self.domain_shape = inner.domain_shape
        self.range_shape = outer.range_shape

    def apply(self, x):
        return self.outer.apply(self.inner.apply(x))

    def adjoint_apply(self, y):
        return self.inner.adjoint_apply(self.outer.adjoint_apply(y))


def warp_from_spec(shape, spec):
    """Build an oracle warp from a workload gate spec (dict)."""
    kind = spec["kind"]
    if kind == "rigid":
        return Warp(shape, RIGID, rotation=spec["rotation"], translation=spec["translation"])
    if kind == "dilatation":
        return Warp(shape, DILATATION, scale=spec["scale"])
    if kind == "dense":
        return Warp(shape, DENSE, phi=spec["phi"])
    raise ValueError(kind)


def gate_operators(geom: Geometry, specs, threads: int | None = None):
    """simulate.gate_operators restated (simulate.py:172-188)."""
    base = RayTransform(geom, threads)
    ops = []
    for spec in specs:
        w = warp_from_spec(geom.image_shape, spec)
        ops.append(base if getattr(w, "identity", False) else Composed(base, w))
    return ops
