"""Joseph parallel-beam ray transform A, A^* on sm_100a (mirror of mctomo.projector).

Reference: projector.py:39-233.  ``Geometry`` is the same frozen dataclass
(validation, angles, bin centres, presets).  ``RayTransform`` keeps the
reference semantics — pixel (r, c) centred at (r-(rows-1)/2, c-(cols-1)/2),
angle theta integrating along (cos, sin), bins along (-sin, cos), one sample per
row (|cos| >= sin) or per column otherwise, linear interpolation across the
other axis weighted by the step length — but computes the weights on the fly in
the CUDA kernels instead of materialising 48*A*B*n bytes of tables, and
implements A^* as a deterministic transpose-gather instead of a scatter.

``GatedOperator`` is A_i = A o D_i (simulate.gate_operators / linops.compose)
with the warp fused into the projector's input packing.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .linops import LinearMap

__all__ = ["Geometry", "RayTransform", "GatedOperator", "ray_transform", "forward", "adjoint"]


@dataclass(frozen=True)
class Geometry:
    """Parallel-beam acquisition geometry (reference projector.py:39-103)."""

    rows: int
    cols: int
    num_angles: int
    num_bins: int
    detector_spacing: float

    def __post_init__(self):
        for name in ("rows", "cols", "num_angles", "num_bins"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if not (self.detector_spacing > 0):
            raise ValueError("detector_spacing must be positive")

    @property
    def angles(self) -> np.ndarray:
        """Projection angles in radians, strictly increasing in [0, pi)."""
        return np.arange(self.num_angles) * (math.pi / self.num_angles)

    @property
    def bin_centers(self) -> np.ndarray:
        offsets = np.arange(self.num_bins) - (self.num_bins - 1) / 2.0
        return offsets * self.detector_spacing

    @property
    def detector_span(self) -> float:
        return self.num_bins * self.detector_spacing

    @property
    def image_shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    @property
    def sino_shape(self) -> tuple[int, int]:
        return (self.num_angles, self.num_bins)

    @classmethod
    def default(cls) -> "Geometry":
        spacing = 100.0 * math.sqrt(2.0) / 200.0
        return cls(100, 100, 200, 200, spacing)

    @classmethod
    def fast(cls) -> "Geometry":
        spacing = 64.0 * math.sqrt(2.0) / 128.0
        return cls(64, 64, 128, 128, spacing)

    def angle_tables(self):
        """cos, sin, rows-dominant flags exactly as projector.py:127-130."""
        ang = self.angles
        cos = np.ascontiguousarray(np.cos(ang), dtype=np.float64)
        sin = np.ascontiguousarray(np.sin(ang), dtype=np.float64)
        rdom = np.ascontiguousarray((np.abs(cos) >= sin).astype(np.uint8))
        return cos, sin, rdom


class _RayPlan:
    """Owner of one device ``mct_ray_plan`` (per CUDA device)."""

    def __init__(self, geom: Geometry):
        torch = _lib.require_cuda()
        L = _lib.load()
        cos, sin, rdom = geom.angle_tables()
        h = ctypes.c_void_p()
        _lib.check(L.mct_ray_plan_create(ctypes.byref(h), geom.rows, geom.cols, geom.num_angles,
                                         geom.num_bins, float(geom.detector_spacing),
                                         cos.ctypes.data, sin.ctypes.data, rdom.ctypes.data))
        self.handle = h
        self.device = torch.cuda.current_device()
        self.item_bytes = int(L.mct_ray_workspace_bytes(h, 1))

    def workspace_bytes(self, items: int) -> int:
        """Workspace bytes for launches of up to `items` items (gate-pair blocks)."""
        return int(_lib.load().mct_ray_workspace_bytes(self.handle, int(items)))

    def set_ring_pairs(self, pairs: int) -> None:
        """Cap the gate-pair regions a workspace of this plan holds (less memory, more
        K1-K3 chunks per iteration, same results).  Call before any workspace or engine
        of this plan exists: the workspace layout follows it."""
        _lib.check(_lib.load().mct_ray_plan_set_ring_pairs(self.handle, int(pairs)))

    def __del__(self):
        try:
            if self.handle:
                _lib.load().mct_ray_plan_destroy(self.handle)
        except Exception:
            pass


class RayTransform(LinearMap):
    """The parallel-beam projection operator for a fixed geometry.

    Immutable; each call draws its own (zeroed) workspace from the caching
    allocator, so concurrent calls on distinct outputs are safe
    (reference projector.py:186-199).
    """

    def __init__(self, geom: Geometry):
        self.geom = geom
        self.domain_shape = geom.image_shape
        self.range_shape = geom.sino_shape
        self._plans: dict[int, _RayPlan] = {}

    def plan(self) -> _RayPlan:
        torch = _lib.require_cuda()
        dev = torch.cuda.current_device()
        p = self._plans.get(dev)
        if p is None:
            p = self._plans[dev] = _RayPlan(self.geom)
        return p

    def workspace(self, items: int):
        """Zeroed workspace for `items` items, cached per (device, stream).

        The kernels overwrite every interior element they read and never write
        the zero pads, so a workspace can be reused by any later call issued on
        the same stream (calls on other streams get their own buffer).
        """
        torch = _lib.require_cuda()
        need = self.plan().workspace_bytes(items)
        cache = self.__dict__.setdefault("_ws", {})
        key = (torch.cuda.current_device(), _lib.stream_handle())
        ws = cache.get(key)
        if ws is None or ws.numel() < need:
            ws = cache[key] = torch.zeros(need, dtype=torch.uint8, device="cuda")
        return ws

    def forward_batch(self, x):
        """A on a (batch, rows, cols) fp32 CUDA tensor -> (batch, A, B)."""
        torch = _lib.require_cuda()
        b = x.shape[0]
        out = torch.empty((b,) + self.range_shape, dtype=torch.float32, device=x.device)
        ws = self.workspace(b)
        _lib.check(_lib.load().mct_ray_forward(self.plan().handle, _lib.ptr(x), _lib.ptr(out), b,
                                               _lib.ptr(ws), _lib.stream_handle()))
        return out

    def adjoint_batch(self, y):
        """A^* on a (batch, A, B) fp32 CUDA tensor -> (batch, rows, cols)."""
        torch = _lib.require_cuda()
        b = y.shape[0]
        out = torch.empty((b,) + self.domain_shape, dtype=torch.float32, device=y.device)
        ws = self.workspace(b)
        _lib.check(_lib.load().mct_ray_adjoint(self.plan().handle, _lib.ptr(y), _lib.ptr(out), b,
                                               _lib.ptr(ws), _lib.stream_handle()))
        return out

    def apply_device(self, x):
        return self.forward_batch(x.reshape((1,) + self.domain_shape))[0]

    def adjoint_device(self, y):
        return self.adjoint_batch(y.reshape((1,) + self.range_shape))[0]


class GatedOperator(LinearMap):
    """A_i = A o D_i with the warp fused into the projector input packing.

    Behaves like the reference ``compose(base, WarpOperator(...))``
    (simulate.py:184-185, linops.py:105-132): ``outer`` / ``inner`` are exposed.
    """

    def __init__(self, outer: RayTransform, inner):
        self.outer = outer
        self.inner = inner
        self.domain_shape = tuple(inner.domain_shape)
        self.range_shape = tuple(outer.range_shape)
        self._fams: dict[int, object] = {}

    def _family(self):
        from .engine import Family  # local import: engine imports projector

        torch = _lib.require_cuda()
        dev = torch.cuda.current_device()
        f = self._fams.get(dev)
        if f is None:
            f = self._fams[dev] = Family(self.outer, [[self.inner]])
        return f

    def apply_device(self, x):
        torch = _lib.require_cuda()
        fam = self._family()
        out = torch.empty(self.range_shape, dtype=torch.float32, device=x.device)
        ws = self.outer.workspace(1)
        _lib.check(_lib.load().mct_gated_forward(fam.handle, 0, 0, _lib.ptr(x), _lib.ptr(out),
                                                 _lib.ptr(ws), _lib.stream_handle()))
        return out

    def adjoint_device(self, y):
        torch = _lib.require_cuda()
        fam = self._family()
        out = torch.empty(self.domain_shape, dtype=torch.float32, device=y.device)
        ws = self.outer.workspace(1)
        _lib.check(_lib.load().mct_gated_adjoint(fam.handle, 0, 0, _lib.ptr(y), _lib.ptr(out),
                                                 _lib.ptr(ws), _lib.stream_handle()))
        return out


@lru_cache(maxsize=4)
def ray_transform(geom: Geometry) -> RayTransform:
    """Return the (cached) ray transform for ``geom`` (projector.py:220-223)."""
    return RayTransform(geom)


def forward(geom: Geometry, x):
    return ray_transform(geom).apply(x)


def adjoint(geom: Geometry, y):
    return ray_transform(geom).adjoint_apply(y)
