"""Operator contract and combinators on the device (mirror of mctomo.linops).

Same surface as the reference (linops.py:39-307): ``LinearMap`` with
``domain_shape`` / ``range_shape`` / ``apply`` / ``adjoint_apply``,
``ComposedMap`` / ``compose``, ``GramSumMap``, ``power_method``,
``stacked_norm_sq``, ``adjoint_mismatch``.

B200 design: every operator of this package computes on the GPU through the
sm_100a C-ABI.  ``apply`` / ``adjoint_apply`` accept either

* numpy arrays (the reference contract: float64 in, a *new* float64 array out,
  input never mutated, ``ValueError`` on a shape mismatch) — values are rounded
  to fp32 on the device, or
* torch CUDA fp32 tensors (the fast path; returns a new CUDA tensor).

``apply_device`` / ``adjoint_device`` are the tensor-level hooks subclasses
implement.  Power iteration and the Gram sums run on the device with the
library's fixed-order fp64 reductions.
"""

from __future__ import annotations

import warnings
from abc import ABC, abstractmethod
from typing import Sequence

import numpy as np

from . import _lib

__all__ = [
    "LinearMap",
    "IdentityMap",
    "DiagonalMap",
    "StackedMap",
    "ComposedMap",
    "GramSumMap",
    "compose",
    "power_method",
    "stacked_norm_sq",
    "adjoint_mismatch",
    "device_dot",
]


def _is_tensor(v) -> bool:
    return type(v).__module__.startswith("torch")


def device_dot(a, b=None, mode: int = _lib.REDUCE_DOT) -> float:
    """Deterministic fp64 reduction of fp32 device tensors (one value)."""
    torch = _lib.require_cuda()
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    bp = _lib.ptr(b) if b is not None else None
    _lib.check(_lib.load().mct_reduce(_lib.ptr(a), bp, a.numel(), 1, a.numel(), mode,
                                      _lib.ptr(out), _lib.ptr(_lib.scratch(a.device)),
                                      _lib.stream_handle()))
    return float(out.item())


class LinearMap(ABC):
    """A linear map between real coordinate grids (reference linops.py:39-73)."""

    domain_shape: tuple[int, ...]
    range_shape: tuple[int, ...]

    # ---- device hooks --------------------------------------------------
    @abstractmethod
    def apply_device(self, x):
        """Evaluate on a contiguous fp32 CUDA tensor of ``domain_shape``."""

    @abstractmethod
    def adjoint_device(self, y):
        """Transpose on a contiguous fp32 CUDA tensor of ``range_shape``."""

    # ---- reference contract --------------------------------------------
    def apply(self, x):
        if _is_tensor(x):
            return self.apply_device(self._check_tensor(x, self.domain_shape, "domain"))
        x = self._check_domain(x)
        return self._roundtrip(self.apply_device, x)

    def adjoint_apply(self, y):
        if _is_tensor(y):
            return self.adjoint_device(self._check_tensor(y, self.range_shape, "range"))
        y = self._check_range(y)
        return self._roundtrip(self.adjoint_device, y)

    def _roundtrip(self, fn, arr: np.ndarray) -> np.ndarray:
        torch = _lib.require_cuda()
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).cuda()
        return fn(t).double().cpu().numpy()

    def _check_domain(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != tuple(self.domain_shape):
            raise ValueError(f"expected domain shape {tuple(self.domain_shape)}, got {x.shape}")
        return x

    def _check_range(self, y) -> np.ndarray:
        y = np.asarray(y, dtype=np.float64)
        if y.shape != tuple(self.range_shape):
            raise ValueError(f"expected range shape {tuple(self.range_shape)}, got {y.shape}")
        return y

    @staticmethod
    def _check_tensor(t, shape, what):
        torch = _lib.require_cuda()
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"expected {what} shape {tuple(shape)}, got {tuple(t.shape)}")
        if not t.is_cuda:
            raise ValueError("tensor inputs must live on a CUDA device")
        if t.dtype != torch.float32:
            t = t.float()
        return t.contiguous()


class IdentityMap(LinearMap):
    """Identity on a grid (reference linops.py:76-87); a device copy."""

    def __init__(self, shape):
        self.domain_shape = tuple(int(n) for n in shape)
        self.range_shape = self.domain_shape

    def apply_device(self, x):
        return x.clone()

    def adjoint_device(self, y):
        return y.clone()


class DiagonalMap(LinearMap):
    """Elementwise multiplication by a fixed array, self-adjoint (linops.py:90-102).

    The diagonal lives on the device in fp32.
    """

    def __init__(self, diag):
        self.diag = np.asarray(diag, dtype=np.float64).copy()
        self.domain_shape = self.diag.shape
        self.range_shape = self.diag.shape
        self._dev = None

    def _d(self):
        if self._dev is None:
            torch = _lib.require_cuda()
            self._dev = torch.from_numpy(self.diag.astype(np.float32)).cuda()
        return self._dev

    def apply_device(self, x):
        return x * self._d()

    def adjoint_device(self, y):
        return y * self._d()


class StackedMap(LinearMap):
    """Row stack of maps sharing one domain and one range (linops.py:135-169).

    ``apply`` stacks the block outputs along a new leading axis; ``adjoint_apply``
    sums the block adjoints in block order (device axpby, fixed order).
    """

    def __init__(self, blocks: Sequence[LinearMap]):
        blocks = tuple(blocks)
        if not blocks:
            raise ValueError("StackedMap needs at least one block")
        dom, rng = tuple(blocks[0].domain_shape), tuple(blocks[0].range_shape)
        for k, b in enumerate(blocks):
            if tuple(b.domain_shape) != dom:
                raise ValueError(f"block {k} domain {tuple(b.domain_shape)} != {dom}")
            if tuple(b.range_shape) != rng:
                raise ValueError(f"block {k} range {tuple(b.range_shape)} != {rng}")
        self.blocks = blocks
        self.domain_shape = dom
        self.range_shape = (len(blocks),) + rng

    def apply_device(self, x):
        torch = _lib.require_cuda()
        return torch.stack([b.apply_device(x) for b in self.blocks])

    def adjoint_device(self, y):
        L = _lib.load()
        out = self.blocks[0].adjoint_device(y[0].contiguous()).clone()
        for b, yk in zip(self.blocks[1:], y[1:]):
            g = b.adjoint_device(yk.contiguous())
            _lib.check(L.mct_axpby(out.numel(), 1.0, _lib.ptr(g), 1.0, _lib.ptr(out),
                                   _lib.stream_handle()))
        return out


class ComposedMap(LinearMap):
    """Composition ``outer o inner`` (reference linops.py:105-123)."""

    def __init__(self, outer: LinearMap, inner: LinearMap):
        if tuple(inner.range_shape) != tuple(outer.domain_shape):
            raise ValueError(
                "cannot compose: inner range "
                f"{tuple(inner.range_shape)} != outer domain {tuple(outer.domain_shape)}")
        self.outer = outer
        self.inner = inner
        self.domain_shape = tuple(inner.domain_shape)
        self.range_shape = tuple(outer.range_shape)

    def apply_device(self, x):
        return self.outer.apply_device(self.inner.apply_device(x))

    def adjoint_device(self, y):
        return self.inner.adjoint_device(self.outer.adjoint_device(y))


def compose(outer: LinearMap, inner: LinearMap) -> ComposedMap:
    """``x -> outer(inner(x))`` (reference linops.py:126-132).

    A ray transform composed with a warp becomes the fused
    :class:`~paper_2410_10503_b200.projector.GatedOperator` (A_i = A o D_i with the
    warp written straight into the projector's padded input layout).
    """
    from .motion import WarpBase
    from .projector import GatedOperator, RayTransform

    if isinstance(outer, RayTransform) and isinstance(inner, WarpBase):
        if tuple(inner.range_shape) != tuple(outer.domain_shape):
            raise ValueError(
                "cannot compose: inner range "
                f"{tuple(inner.range_shape)} != outer domain {tuple(outer.domain_shape)}")
        return GatedOperator(outer, inner)
    return ComposedMap(outer, inner)


class GramSumMap(LinearMap):
    """``x -> c*x + sum_i w_i B_i^T B_i x`` (reference linops.py:172-212)."""

    def __init__(self, blocks: Sequence[LinearMap], weights: Sequence[float] | None = None,
                 identity_coefficient: float = 0.0):
        blocks = tuple(blocks)
        if not blocks:
            raise ValueError("GramSumMap needs at least one block")
        dom = tuple(blocks[0].domain_shape)
        for k, b in enumerate(blocks):
            if tuple(b.domain_shape) != dom:
                raise ValueError(f"block {k} domain {tuple(b.domain_shape)} != {dom}")
        if weights is None:
            weights = (1.0,) * len(blocks)
        weights = tuple(float(w) for w in weights)
        if len(weights) != len(blocks):
            raise ValueError("one weight per block required")
        self.blocks = blocks
        self.weights = weights
        self.identity_coefficient = float(identity_coefficient)
        self.domain_shape = dom
        self.range_shape = dom

    def apply_device(self, x):
        L = _lib.load()
        out = x.clone()
        n = out.numel()
        st = _lib.stream_handle()
        # out = c * x
        _lib.check(L.mct_axpby(n, 0.0, _lib.ptr(x), self.identity_coefficient, _lib.ptr(out), st))
        for w, b in zip(self.weights, self.blocks):
            g = b.adjoint_device(b.apply_device(x))
            _lib.check(L.mct_axpby(n, w, _lib.ptr(g), 1.0, _lib.ptr(out), st))
        return out

    def adjoint_device(self, y):
        return self.apply_device(y)


def power_method(op: LinearMap, iterations: int = 100, seed: int = 0,
                 rtol: float = 1e-10) -> float:
    """Operator norm by power iteration on the Gram (reference linops.py:215-272).

    Same seeded start (``default_rng(seed).standard_normal``), stopping rule and
    degenerate-case warnings; the Gram applications, norms and Rayleigh
    quotients run on the device (fp32 vectors, fp64 fixed-order reductions).
    """
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if not isinstance(op, LinearMap):
        return _foreign_power_method(op, iterations, seed, rtol)
    torch = _lib.require_cuda()
    rng = np.random.default_rng(seed)
    b0 = rng.standard_normal(op.domain_shape)
    nb = float(np.linalg.norm(b0))
    if nb == 0.0:
        warnings.warn("degenerate start vector; returning 0", RuntimeWarning)
        return 0.0
    b = torch.from_numpy((b0 / nb).astype(np.float32)).cuda()
    L = _lib.load()
    rayleigh = 0.0
    for _ in range(iterations):
        w = op.adjoint_device(op.apply_device(b))
        bb = device_dot(b, b)
        new_rayleigh = device_dot(b, w) / bb
        nw = float(np.sqrt(device_dot(w, w)))
        if nw == 0.0:
            warnings.warn("power iteration degenerated to zero vector; returning 0",
                          RuntimeWarning)
            return 0.0
        _lib.check(L.mct_axpby(w.numel(), 1.0 / nw, _lib.ptr(w), 0.0, _lib.ptr(b),
                               _lib.stream_handle()))
        if new_rayleigh > 0 and abs(new_rayleigh - rayleigh) <= rtol * new_rayleigh:
            rayleigh = new_rayleigh
            break
        rayleigh = new_rayleigh
    return float(np.sqrt(max(rayleigh, 0.0)))


def _foreign_power_method(op, iterations: int, seed: int, rtol: float) -> float:
    """power_method for a map that is not one of this package's device operators
    (any object with the reference's LinearMap contract: numpy ``apply`` /
    ``adjoint_apply``).  The Gram applications are the foreign map's own; this only
    sequences them with the same seeded start and stopping rule (linops.py:250-272)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(tuple(op.domain_shape))
    norm0 = float(np.linalg.norm(v))
    if norm0 == 0.0:
        warnings.warn("degenerate start vector; returning 0", RuntimeWarning)
        return 0.0
    v = v / norm0
    lam = 0.0
    for _ in range(iterations):
        gv = np.asarray(op.adjoint_apply(op.apply(v)), dtype=np.float64)
        lam_new = float(np.vdot(v, gv)) / float(np.vdot(v, v))
        gnorm = float(np.linalg.norm(gv))
        if gnorm == 0.0:
            warnings.warn("power iteration degenerated to zero vector; returning 0",
                          RuntimeWarning)
            return 0.0
        v = gv / gnorm
        converged = lam_new > 0 and abs(lam_new - lam) <= rtol * lam_new
        lam = lam_new
        if converged:
            break
    return float(np.sqrt(max(lam, 0.0)))


class _ForeignGramSum:
    """sum_i B_i^T B_i over maps outside this package (numpy contract)."""

    def __init__(self, blocks):
        self.blocks = tuple(blocks)
        self.domain_shape = self.range_shape = tuple(self.blocks[0].domain_shape)

    def apply(self, x):
        out = np.zeros(self.domain_shape)
        for b in self.blocks:
            out += np.asarray(b.adjoint_apply(b.apply(x)), dtype=np.float64)
        return out

    adjoint_apply = apply


def stacked_norm_sq(blocks: Sequence[LinearMap], iterations: int = 100, seed: int = 0) -> float:
    """Squared norm of the row stack = lambda_max(sum_i B_i^T B_i) (linops.py:275-289)."""
    blocks = tuple(blocks)
    if not all(isinstance(b, LinearMap) for b in blocks):
        return _foreign_power_method(_ForeignGramSum(blocks), iterations, seed, 1e-10)
    return power_method(GramSumMap(blocks), iterations=iterations, seed=seed)


def adjoint_mismatch(op: LinearMap, pairs: int = 20, seed: int = 0) -> float:
    """Worst relative defect of <Ax, y> = <x, A^T y> (reference linops.py:292-307)."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(pairs):
        x = rng.standard_normal(op.domain_shape).astype(np.float32).astype(np.float64)
        y = rng.standard_normal(op.range_shape).astype(np.float32).astype(np.float64)
        lhs = float(np.vdot(op.apply(x), y))
        rhs = float(np.vdot(x, op.adjoint_apply(y)))
        scale = max(abs(lhs), abs(rhs), np.finfo(np.float64).tiny)
        worst = max(worst, abs(lhs - rhs) / scale)
    return worst
