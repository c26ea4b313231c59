"""Displacement warps D_i and D_i^* on sm_100a (mirror of mctomo.motion).

Reference: motion.py:36-242.  ``MotionParams`` / ``motion_sequence`` are the same
host-side types.  ``WarpOperator`` resamples by inverse mapping with bilinear
interpolation and zero fill (motion.py:132-183); its adjoint is a deterministic
gather that re-evaluates the forward's exact fp64 source coordinates, so the
pair is an exact transpose up to fp32 summation (motion.py:185-194 is a
scatter).  Identity parameters short-circuit to a bitwise copy.

``DenseWarpOperator`` adds the dense non-rigid field the BASELINE configs need
(not in the reference): src(p) = p + phi(p) with phi a (2, rows, cols) fp32
pull-back displacement in pixels, same interpolation scheme; its adjoint uses a
transposed gather list built once on the device.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linops import LinearMap

__all__ = [
    "MotionParams",
    "WarpOperator",
    "DenseWarpOperator",
    "WarpBase",
    "motion_sequence",
    "warp_from_spec",
    "RIGID_TERMINAL_ROTATION",
    "RIGID_TERMINAL_TRANSLATION",
    "DILATATION_TERMINAL_GROWTH",
]

KINDS = ("rigid", "dilatation")
RIGID_TERMINAL_ROTATION = 0.15
RIGID_TERMINAL_TRANSLATION = (5.0, 3.0)
DILATATION_TERMINAL_GROWTH = 0.04


@dataclass(frozen=True)
class MotionParams:
    """One motion state (reference motion.py:48-108)."""

    kind: str
    rotation: float = 0.0
    translation: tuple[float, float] = (0.0, 0.0)
    scale: float = 1.0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"kind must be one of {KINDS}, got {self.kind!r}")
        values = (self.rotation, *self.translation, self.scale)
        if not all(math.isfinite(v) for v in values):
            raise ValueError("motion parameters must be finite")
        if not self.scale > 0:
            raise ValueError("scale must be positive")
        if self.kind == "rigid" and self.scale != 1.0:
            raise ValueError("rigid motion fixes scale = 1")
        if self.kind == "dilatation" and (self.rotation != 0.0 or self.translation != (0.0, 0.0)):
            raise ValueError("dilatation uses only scale")

    @classmethod
    def identity(cls) -> "MotionParams":
        return cls(kind="rigid")

    def is_identity(self) -> bool:
        return self.rotation == 0.0 and self.translation == (0.0, 0.0) and self.scale == 1.0

    def to_dict(self) -> dict:
        return {"kind": self.kind, "rotation": self.rotation,
                "translation": list(self.translation), "scale": self.scale}

    @classmethod
    def from_dict(cls, payload: dict) -> "MotionParams":
        return cls(kind=payload["kind"], rotation=float(payload["rotation"]),
                   translation=(float(payload["translation"][0]),
                                float(payload["translation"][1])),
                   scale=float(payload["scale"]))


class _WarpPlan:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                _lib.load().mct_warp_plan_destroy(self.handle)
        except Exception:
            pass


class WarpBase(LinearMap):
    """Common device plumbing of the warp operators."""

    _identity = False

    def _make_plan(self):  # pragma: no cover - abstract
        raise NotImplementedError

    def plan(self):
        torch = _lib.require_cuda()
        dev = torch.cuda.current_device()
        plans = self.__dict__.setdefault("_plans", {})
        p = plans.get(dev)
        if p is None:
            p = plans[dev] = _WarpPlan(self._make_plan())
        return p

    @property
    def is_identity_warp(self) -> bool:
        return self._identity

    def apply_device(self, x):
        if self._identity:
            return x.clone()
        out = x.new_empty(self.domain_shape)
        _lib.check(_lib.load().mct_warp_forward(self.plan().handle, _lib.ptr(x), _lib.ptr(out),
                                                _lib.stream_handle()))
        return out

    def adjoint_device(self, y):
        if self._identity:
            return y.clone()
        out = y.new_empty(self.domain_shape)
        _lib.check(_lib.load().mct_warp_adjoint(self.plan().handle, _lib.ptr(y), _lib.ptr(out),
                                                _lib.stream_handle()))
        return out

    def apply(self, x):
        if self._identity and not type(x).__module__.startswith("torch"):
            return self._check_domain(x).copy()  # motion.py:180-181 bitwise copy
        return super().apply(x)

    def adjoint_apply(self, y):
        if self._identity and not type(y).__module__.startswith("torch"):
            return self._check_range(y).copy()
        return super().adjoint_apply(y)


class WarpOperator(WarpBase):
    """Rigid / dilatation warp of a fixed-size image (reference motion.py:111-194)."""

    def __init__(self, params: MotionParams, shape: tuple[int, int]):
        if len(shape) != 2 or shape[0] < 1 or shape[1] < 1:
            raise ValueError(f"invalid image shape {shape}")
        self.params = params
        self.domain_shape = (int(shape[0]), int(shape[1]))
        self.range_shape = self.domain_shape
        self._identity = params.is_identity()

    def _make_plan(self):
        L = _lib.load()
        h = ctypes.c_void_p()
        rows, cols = self.domain_shape
        p = self.params
        if self._identity:
            _lib.check(L.mct_warp_plan_create_identity(ctypes.byref(h), rows, cols))
        elif p.kind == "rigid":
            cos, sin = math.cos(p.rotation), math.sin(p.rotation)
            # motion.py:142-147: snap right angles to exact permutations
            if abs(cos) < 1e-15:
                cos = 0.0
            if abs(sin) < 1e-15:
                sin = 0.0
            _lib.check(L.mct_warp_plan_create_rigid(ctypes.byref(h), rows, cols, cos, sin,
                                                    float(p.translation[0]),
                                                    float(p.translation[1])))
        else:
            _lib.check(L.mct_warp_plan_create_dilatation(ctypes.byref(h), rows, cols,
                                                         float(p.scale)))
        return h


class DenseWarpOperator(WarpBase):
    """Dense non-rigid warp src(p) = p + phi(p) (restates motion.py:155-194)."""

    def __init__(self, phi):
        phi = np.asarray(phi)
        if phi.ndim != 3 or phi.shape[0] != 2 or phi.shape[1] < 1 or phi.shape[2] < 1:
            raise ValueError(f"displacement field must have shape (2, rows, cols), got {phi.shape}")
        if not np.all(np.isfinite(phi)):
            raise ValueError("displacement field must be finite")
        self.phi = np.ascontiguousarray(phi, dtype=np.float32)
        self.domain_shape = (int(phi.shape[1]), int(phi.shape[2]))
        self.range_shape = self.domain_shape
        self._identity = False

    def _make_plan(self):
        torch = _lib.require_cuda()
        L = _lib.load()
        h = ctypes.c_void_p()
        phi_dev = torch.from_numpy(self.phi).cuda()
        rows, cols = self.domain_shape
        _lib.check(L.mct_warp_plan_create_dense(ctypes.byref(h), rows, cols, _lib.ptr(phi_dev),
                                                _lib.stream_handle()))
        return h

    @property
    def nnz(self) -> int:
        return int(_lib.load().mct_warp_plan_nnz(self.plan().handle))


def warp_from_spec(shape, spec) -> WarpBase:
    """Warp operator from a workload gate spec dict (see workloads.py)."""
    if isinstance(spec, MotionParams):
        return WarpOperator(spec, shape)
    kind = spec["kind"]
    if kind == "dense":
        return DenseWarpOperator(spec["phi"])
    if kind == "rigid":
        return WarpOperator(MotionParams("rigid", float(spec["rotation"]),
                                         tuple(float(t) for t in spec["translation"])), shape)
    if kind == "dilatation":
        return WarpOperator(MotionParams("dilatation", scale=float(spec["scale"])), shape)
    raise ValueError(f"unknown gate kind {kind!r}")


def motion_sequence(kind: str, num_gates: int, magnitude: float = 1.0) -> list[MotionParams]:
    """Linear ramp from the identity (reference motion.py:197-242)."""
    if kind not in KINDS:
        raise ValueError(f"kind must be one of {KINDS}, got {kind!r}")
    if num_gates < 1:
        raise ValueError("num_gates must be >= 1")
    if not math.isfinite(magnitude):
        raise ValueError("magnitude must be finite")
    fractions = np.linspace(0.0, 1.0, num_gates) if num_gates > 1 else np.array([0.0])
    seq = []
    for f in fractions:
        f = float(f)
        if kind == "rigid":
            seq.append(MotionParams(
                kind="rigid", rotation=f * magnitude * RIGID_TERMINAL_ROTATION,
                translation=(f * magnitude * RIGID_TERMINAL_TRANSLATION[0],
                             f * magnitude * RIGID_TERMINAL_TRANSLATION[1])))
        else:
            seq.append(MotionParams(kind="dilatation",
                                    scale=1.0 + f * magnitude * DILATATION_TERMINAL_GROWTH))
    return seq
