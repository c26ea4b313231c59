"""Seeded synthetic workloads of BASELINE.json's configs.

BASELINE.json names no public dataset: these seeded inputs *are* the workload.
Everything here is host-side input generation in numpy (fp64, rounded to fp32
once so the GPU path and the fp64 oracle consume identical values).

* phantom: random ellipses on the reference's normalised [-1, 1] grid
  (simulate._grids, simulate.py:50-55), painted in draw order and clipped to
  [0, 1] like simulate.make_phantom (simulate.py:76-99);
* rigid gates (C1): rotation U[-5, 5] deg, translation U[-3, 3]^2 px;
* dense gates (C2-C5): sum of 6 Gaussian bumps (sigma 30 px, N(0, I2)
  amplitudes) rescaled to a peak displacement peak*U[0.5, 1];
* noise: the reference's documented Philox + Box-Muller recipe
  (simulate.gaussian_field, simulate.py:113-133), restated bit-exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    n: int
    num_angles: int
    num_bins: int
    num_gates: int
    motion: str          # "rigid" | "dense"
    ellipses: int
    alpha: float
    epochs: int
    peak: float | None = None
    batch: int = 1
    seed: int = 0
    modes: tuple = ("pdhg", "spdhg")

    @property
    def geometry_args(self):
        return (self.n, self.n, self.num_angles, self.num_bins, 1.0)

    @property
    def samples(self) -> int:
        """S = A*B*n Joseph samples per A application."""
        return self.num_angles * self.num_bins * self.n


# BASELINE.json "configs" (C1..C5); ellipse counts 12 where BASELINE leaves them unstated
CONFIGS = {
    "c1": WorkloadConfig("c1", 128, 180, 183, 4, "rigid", 8, 1e-2, 20),
    "c2": WorkloadConfig("c2", 256, 360, 363, 10, "dense", 12, 1e-2, 50, peak=4.0,
                         modes=("spdhg",)),
    "c3": WorkloadConfig("c3", 512, 720, 729, 20, "dense", 16, 5e-3, 50, peak=6.0),
    "c4": WorkloadConfig("c4", 1024, 1440, 1453, 40, "dense", 12, 5e-3, 5, peak=8.0,
                         modes=("pdhg",)),
    "c5": WorkloadConfig("c5", 512, 720, 729, 10, "dense", 12, 1e-2, 30, peak=6.0, batch=64,
                         modes=("spdhg",)),
}


def _grids(rows: int, cols: int):
    # simulate._grids (simulate.py:50-55): [-1, 1] on the longer half-extent
    half = (max(rows, cols) - 1) / 2.0
    u = (np.arange(rows) - (rows - 1) / 2.0) / half
    v = (np.arange(cols) - (cols - 1) / 2.0) / half
    return np.meshgrid(u, v, indexing="ij")


def ellipse_phantom(n: int, count: int, seed: int) -> np.ndarray:
    """Random-ellipse phantom in [0, 1], fp32-rounded."""
    rng = np.random.default_rng([seed, 0])
    centres = rng.uniform(-0.6, 0.6, size=(count, 2))
    axes = rng.uniform(0.08, 0.45, size=(count, 2))
    angles = rng.uniform(0.0, math.pi, size=count)
    values = rng.uniform(0.1, 1.0, size=count)
    uu, vv = _grids(n, n)
    img = np.zeros((n, n))
    for (cu, cv), (ru, rv), th, val in zip(centres, axes, angles, values):
        du, dv = uu - cu, vv - cv
        a = math.cos(th) * du + math.sin(th) * dv
        b = -math.sin(th) * du + math.cos(th) * dv
        img[(a / ru) ** 2 + (b / rv) ** 2 <= 1.0] = val
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def rigid_gates(num_gates: int, seed: int) -> list[dict]:
    """C1 rigid gates: rotation U[-5, 5] deg, translation U[-3, 3]^2 px."""
    rng = np.random.default_rng([seed, 1])
    gates = []
    for _ in range(num_gates):
        rot = math.radians(rng.uniform(-5.0, 5.0))
        tr = (float(rng.uniform(-3.0, 3.0)), float(rng.uniform(-3.0, 3.0)))
        gates.append({"kind": "rigid", "rotation": float(rot), "translation": tr})
    return gates


def bump_field(n: int, peak: float, seed: int, gate: int, bumps: int = 6,
               sigma_px: float = 30.0) -> np.ndarray:
    """Smooth pull-back displacement (2, n, n) fp32 in pixels (row, col)."""
    rng = np.random.default_rng([seed, 2, gate])
    centres = rng.uniform(0.0, n, size=(bumps, 2))
    amps = rng.standard_normal(size=(bumps, 2))
    target = peak * rng.uniform(0.5, 1.0)
    r = np.arange(n, dtype=np.float64)
    phi = np.zeros((2, n, n))
    for (cr, cc), (ar, ac) in zip(centres, amps):
        g = np.exp(-((r[:, None] - cr) ** 2 + (r[None, :] - cc) ** 2) / (2.0 * sigma_px ** 2))
        phi[0] += ar * g
        phi[1] += ac * g
    mag = float(np.sqrt(phi[0] ** 2 + phi[1] ** 2).max())
    if mag > 0:
        phi *= target / mag
    return phi.astype(np.float32)


def dense_gates(n: int, num_gates: int, peak: float, seed: int) -> list[dict]:
    return [{"kind": "dense", "phi": bump_field(n, peak, seed, i)} for i in range(num_gates)]


def gaussian_field(shape, master_seed: int, gate_index: int) -> np.ndarray:
    """Philox + Box-Muller recipe of simulate.gaussian_field (simulate.py:113-133)."""
    if gate_index < 0:
        raise ValueError("gate_index must be >= 0")
    key = np.array([master_seed % (1 << 64), gate_index], dtype=np.uint64)
    uniform = np.random.Generator(np.random.Philox(key=key))
    count = int(np.prod(shape))
    pairs = (count + 1) // 2
    u1 = uniform.random(pairs)
    u2 = uniform.random(pairs)
    radius = np.sqrt(-2.0 * np.log1p(-u1))
    angle = 2.0 * np.pi * u2
    samples = np.empty(2 * pairs)
    samples[0::2] = radius * np.cos(angle)
    samples[1::2] = radius * np.sin(angle)
    return samples[:count].reshape(shape)


def noisy_data(clean: list[np.ndarray], seed: int, level: float = 0.01) -> list[np.ndarray]:
    """d_i = clean_i + (sigma/sqrt(N)) * field_i, sigma = level*max|clean| (fp32)."""
    n = len(clean)
    sigma = level * max(float(np.abs(c).max()) for c in clean)
    gate_sigma = sigma / math.sqrt(n)
    return [
        (np.asarray(c, dtype=np.float64) + gate_sigma * gaussian_field(c.shape, seed, k)).astype(
            np.float32)
        for k, c in enumerate(clean)
    ]


@dataclass
class SliceInputs:
    """Inputs of one slice: phantom, gate specs (dicts), seed."""

    seed: int
    phantom: np.ndarray
    gates: list = field(default_factory=list)


def slice_inputs(cfg: WorkloadConfig, slice_index: int = 0) -> SliceInputs:
    seed = cfg.seed + slice_index
    phantom = ellipse_phantom(cfg.n, cfg.ellipses, seed)
    if cfg.motion == "rigid":
        gates = rigid_gates(cfg.num_gates, seed)
    else:
        gates = dense_gates(cfg.n, cfg.num_gates, float(cfg.peak), seed)
    return SliceInputs(seed=seed, phantom=phantom, gates=gates)
