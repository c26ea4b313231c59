"""Gated operator families, norm estimation and synthetic data on the device.

Mirror of mctomo.simulate (simulate.py:1-314):

* ``gate_operators`` (A_i = A o D_i, identity gates reuse the bare ray
  transform, ``compensated=False`` gives the no-MC baseline) and
  ``estimate_norms`` (per-gate power iteration, stacked norm, base norm) — on
  the GPU;
* ``generate`` (simulate.py:191-239): d_i = A(D_i x) + eps_i with the device
  forward projector and the device noise kernel (``mct_gaussian_field``: the
  pinned Philox4x64-10 + Box-Muller recipe, uniforms bit-identical to numpy),
  returning the reference's ``GatedDataset``; ``NoiseModel``, the presets
  ``rigid_preset`` / ``nonrigid_preset`` and the test phantoms ``make_phantom``
  (simulate.py:62-100, host numpy, bit-identical to the reference's);
* ``gaussian_field`` — the host recipe (bit-exact with the reference), and
  ``gaussian_field_device`` — the same field computed on the GPU;
* ``simulate_data`` / ``workload_problem`` — BASELINE workload data.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .linops import LinearMap, compose, power_method, stacked_norm_sq
from .motion import DenseWarpOperator, MotionParams, motion_sequence, warp_from_spec
from .projector import Geometry, ray_transform
from .workloads import _grids, gaussian_field, noisy_data

__all__ = ["PHANTOM_KINDS", "make_phantom", "NoiseModel", "GatedDataset", "gaussian_field",
           "gaussian_field_device", "generate", "gate_operators", "estimate_norms",
           "rigid_preset", "nonrigid_preset", "simulate_data", "workload_problem"]

PHANTOM_KINDS = ("nested_shells", "thorax")

# thorax regions (centre u, centre v, radius u, radius v) in units of the
# longer half-extent (simulate.py:44-47)
THORAX_BODY = (0.0, 0.0, 0.92, 0.72)
THORAX_LUNGS = ((-0.02, -0.42, 0.34, 0.26), (-0.02, 0.42, 0.34, 0.26))
THORAX_SPINE = (0.62, 0.0, 0.16, 0.12)


def _inside(uu, vv, region) -> np.ndarray:
    cu, cv, ru, rv = region
    return ((uu - cu) / ru) ** 2 + ((vv - cv) / rv) ** 2 <= 1.0


def make_phantom(kind: str, rows: int, cols: int) -> np.ndarray:
    """Deterministic test phantom in [0, 1] (simulate.py:62-100).

    Layers are painted in order, later ones overwrite: ``nested_shells`` is an
    oval shell with a five-lobed ridge around a dense core; ``thorax`` a tissue
    ellipse with two lungs, a spine disc and ten rib dots.
    """
    if kind not in PHANTOM_KINDS:
        raise ValueError(f"kind must be one of {PHANTOM_KINDS}, got {kind!r}")
    if min(rows, cols) < 16:
        raise ValueError("phantom grids must be at least 16x16")
    uu, vv = _grids(rows, cols)
    img = np.zeros((rows, cols))
    if kind == "nested_shells":
        r = np.hypot(uu / 0.88, vv / 0.78)
        lobes = 0.55 + 0.10 * np.cos(5.0 * np.arctan2(vv, uu))
        layers = [
            (r <= 1.0, 0.85),
            (r <= 0.92, 0.30),
            ((np.abs(r - lobes) <= 0.07) & (r <= 0.92), 0.95),
            (r <= 0.22, 0.65),
            (np.abs(r - 0.30) <= 0.04, 0.15),
        ]
    else:
        layers = [(_inside(uu, vv, THORAX_BODY), 0.55)]
        layers += [(_inside(uu, vv, lung), 0.12) for lung in THORAX_LUNGS]
        layers.append((_inside(uu, vv, THORAX_SPINE), 0.95))
        for k in range(10):  # ribs along the body outline
            ang = -0.8 * math.pi / 2 + k * (1.6 * math.pi / 2) / 9
            centre = (0.78 * math.cos(ang + math.pi / 2), 0.62 * math.sin(ang + math.pi / 2))
            layers.append((_inside(uu, vv, (*centre, 0.045, 0.045)), 0.85))
    for mask, value in layers:
        img[mask] = value
    return np.clip(img, 0.0, 1.0)


@dataclass(frozen=True)
class NoiseModel:
    """Gaussian sinogram noise, per-gate variance sigma^2 / N (simulate.py:103-110)."""

    sigma: float

    def __post_init__(self):
        if not (math.isfinite(self.sigma) and self.sigma >= 0):
            raise ValueError("sigma must be finite and >= 0")


@dataclass
class GatedDataset:
    """N gates of (motion state, noisy sinogram) plus provenance (simulate.py:137-169).

    Gate 1 (index 0) carries the identity motion; ``truth`` is the phantom in
    that reference state.
    """

    geometry: Geometry
    truth: np.ndarray
    motion: list
    sinograms: list
    sigma: float
    master_seed: int
    phantom_kind: str | None = None
    magnitude: float | None = None

    @property
    def num_gates(self) -> int:
        return len(self.motion)

    def __post_init__(self):
        if len(self.motion) == 0:
            raise ValueError("at least one gate required")
        if len(self.sinograms) != len(self.motion):
            raise ValueError("one sinogram per motion state required")
        if not self.motion[0].is_identity():
            raise ValueError("gate 1 must carry the identity motion")
        want = tuple(self.geometry.sino_shape)
        for k, sino in enumerate(self.sinograms):
            if tuple(np.shape(sino)) != want:
                raise ValueError(f"gate {k} sinogram shape {np.shape(sino)} != {want}")


def gaussian_field_device(shape, master_seed: int, gate_index: int, scale: float = 1.0,
                          base=None, dtype: str = "float64"):
    """``base + scale * gaussian_field(shape, master_seed, gate_index)`` on the GPU.

    Returns a CUDA tensor (fp64 or fp32).  Same stream as the host recipe
    (Philox4x64-10 keyed (master_seed mod 2^64, gate_index), uniforms
    bit-identical); the Box-Muller transcendental functions are CUDA's, within a
    few ulp of the host libm.  ``base`` is an optional fp32 CUDA tensor of
    ``shape`` (e.g. a clean sinogram).
    """
    if gate_index < 0:
        raise ValueError("gate_index must be >= 0")
    torch = _lib.require_cuda()
    shape = tuple(int(v) for v in np.atleast_1d(shape))
    tdtype = {"float64": torch.float64, "float32": torch.float32}[dtype]
    out = torch.empty(shape, dtype=tdtype, device="cuda")
    bp = None
    if base is not None:
        if tuple(base.shape) != shape or base.dtype != torch.float32 or not base.is_cuda:
            raise ValueError("base must be a CUDA fp32 tensor of the field's shape")
        base = base.contiguous()
        bp = _lib.ptr(base)
    _lib.check(_lib.load().mct_gaussian_field(
        int(master_seed) % (1 << 64), int(gate_index), out.numel(), float(scale), bp,
        _lib.ptr(out), 1 if dtype == "float64" else 0, _lib.stream_handle()))
    return out


def generate(phantom, motion: list, geom: Geometry, noise: NoiseModel | None = None,
             master_seed: int = 0, phantom_kind: str | None = None,
             magnitude: float | None = None) -> GatedDataset:
    """Simulated gated acquisition (simulate.py:191-239), computed on the GPU.

    clean_i = A(D_i x) by the device gated operators (fp32), then
    d_i = clean_i + (sigma/sqrt(N)) * field_i by the device noise kernel in
    fp64; ``noise=None`` sets sigma to 2% of the brightest noiseless bin.
    Sinograms are returned as float64 numpy arrays like the reference's.
    """
    torch = _lib.require_cuda()
    phantom = np.asarray(phantom, dtype=np.float64)
    if phantom.shape != tuple(geom.image_shape):
        raise ValueError(f"phantom shape {phantom.shape} != geometry image {geom.image_shape}")
    if not motion:
        raise ValueError("motion list must be nonempty")
    if not motion[0].is_identity():
        raise ValueError("gate 1 must carry the identity motion")
    ops = gate_operators(geom, motion, compensated=True)
    x = torch.from_numpy(phantom.astype(np.float32)).cuda()
    clean = [op.apply_device(x) for op in ops]
    sigma = noise.sigma if noise is not None else 0.02 * max(float(c.max()) for c in clean)
    gate_sigma = sigma / math.sqrt(len(motion))
    sinos = [gaussian_field_device(geom.sino_shape, master_seed, k, gate_sigma, base=c)
             .cpu().numpy() for k, c in enumerate(clean)]
    return GatedDataset(geometry=geom, truth=phantom.copy(), motion=list(motion),
                        sinograms=sinos, sigma=float(sigma), master_seed=int(master_seed),
                        phantom_kind=phantom_kind, magnitude=magnitude)


def _preset(kind: str, num_gates: int, phantom_kind: str, size: str, sigma, seed: int,
            magnitude: float) -> GatedDataset:
    geoms = {"default": Geometry.default, "fast": Geometry.fast}
    if size not in geoms:
        raise ValueError(f"size must be 'default' or 'fast', got {size!r}")
    geom = geoms[size]()
    return generate(make_phantom(phantom_kind, geom.rows, geom.cols),
                    motion_sequence(kind, num_gates, magnitude), geom,
                    NoiseModel(sigma) if sigma is not None else None, master_seed=seed,
                    phantom_kind=phantom_kind, magnitude=magnitude)


def rigid_preset(size: str = "default", sigma: float | None = None, seed: int = 0,
                 magnitude: float = 1.0) -> GatedDataset:
    """20-gate rigid-motion dataset on the nested_shells phantom (simulate.py:296-303)."""
    return _preset("rigid", 20, "nested_shells", size, sigma, seed, magnitude)


def nonrigid_preset(size: str = "default", sigma: float | None = None, seed: int = 0,
                    magnitude: float = 1.0) -> GatedDataset:
    """10-gate dilatation dataset on the thorax phantom (simulate.py:306-314)."""
    return _preset("dilatation", 10, "thorax", size, sigma, seed, magnitude)


def _is_identity(spec) -> bool:
    if isinstance(spec, MotionParams):
        return spec.is_identity()
    if isinstance(spec, dict) and spec.get("kind") in ("rigid", "dilatation"):
        return (float(spec.get("rotation", 0.0)) == 0.0
                and tuple(spec.get("translation", (0.0, 0.0))) == (0.0, 0.0)
                and float(spec.get("scale", 1.0)) == 1.0)
    return False


def gate_operators(geom: Geometry, motion: Sequence, compensated: bool = True) -> list[LinearMap]:
    """Gated forward operators A o D_i (reference simulate.py:172-188).

    ``motion`` entries may be ``MotionParams`` (rigid / dilatation), dense
    displacement fields (arrays of shape (2, rows, cols)) or workload spec
    dicts.
    """
    base = ray_transform(geom)
    ops: list[LinearMap] = []
    for spec in motion:
        if not compensated or _is_identity(spec):
            ops.append(base)
            continue
        if isinstance(spec, np.ndarray):
            warp = DenseWarpOperator(spec)
        else:
            warp = warp_from_spec(geom.image_shape, spec)
        ops.append(compose(base, warp))
    return ops


def estimate_norms(geom: Geometry, motion: Sequence, iterations: int = 100, seed: int = 0,
                   operators: Sequence[LinearMap] | None = None) -> dict:
    """Power-iteration norm estimates (reference simulate.py:242-265), on the GPU."""
    ops = list(operators) if operators is not None else gate_operators(geom, motion, True)
    gate_norms = [float(power_method(op, iterations=iterations, seed=seed)) for op in ops]
    stacked = float(stacked_norm_sq(ops, iterations=iterations, seed=seed))
    base = float(power_method(ray_transform(geom), iterations=iterations, seed=seed))
    return {
        "gate_norms": gate_norms,
        "stacked_norm_sq": stacked,
        "base_norm_sq": base * base,
        "power_iterations": int(iterations),
        "power_seed": int(seed),
    }


def simulate_data(operators: Sequence[LinearMap], phantom: np.ndarray, seed: int,
                  level: float = 0.01) -> list[np.ndarray]:
    """d_i = A_i x + (sigma/sqrt(N)) * gaussian_field(i), sigma = level*max|A_i x|."""
    clean = [np.asarray(op.apply(np.asarray(phantom, dtype=np.float64))) for op in operators]
    return noisy_data(clean, seed, level)


def workload_problem(cfg, slice_index: int = 0, data=None):
    """(Problem, truth, SliceInputs) of one slice of a BASELINE workload config.

    ``data`` may supply precomputed sinograms (e.g. committed golden inputs);
    otherwise they are simulated with the device forward projector.
    """
    from .solvers import Problem
    from .workloads import slice_inputs

    inp = slice_inputs(cfg, slice_index)
    geom = Geometry(*cfg.geometry_args)
    ops = gate_operators(geom, inp.gates, compensated=True)
    if data is None:
        data = simulate_data(ops, inp.phantom, inp.seed)
    return Problem.from_parts(cfg.alpha, ops, data), inp.phantom, inp
