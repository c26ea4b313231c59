"""Gated operator families, norm estimation and synthetic data on the device.

Mirror of the hot-path parts of mctomo.simulate (simulate.py:172-265):
``gate_operators`` (A_i = A o D_i, identity gates reuse the bare ray transform,
``compensated=False`` gives the no-MC baseline) and ``estimate_norms``
(per-gate power iteration, stacked norm, base norm — all on the GPU).
``gaussian_field`` is the reference's pinned Philox + Box-Muller recipe.
``simulate_data`` produces d_i = A(D_i x) + noise for the BASELINE workloads
with the device forward projector.
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np

from .linops import LinearMap, compose, power_method, stacked_norm_sq
from .motion import DenseWarpOperator, MotionParams, WarpOperator, warp_from_spec
from .projector import Geometry, ray_transform
from .workloads import gaussian_field, noisy_data

__all__ = ["gate_operators", "estimate_norms", "gaussian_field", "simulate_data",
           "workload_problem"]


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
