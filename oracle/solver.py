"""ORACLE — TEST INFRASTRUCTURE ONLY.  numpy fp64 restatement of the solver layer.

Follows the reference *code* (not the SPEC):
functionals.prox_g / prox_fstar (functionals.py:40-68), moduli (:115-126),
SolverConfig admissibility (solvers.py:149-187), default_config (:198-247),
sample_gates (:298-313), step (:316-366), run (:369-419), _epoch_objective
(:422-432), power_method (linops.py:215-272), stacked_norm_sq (:275-289).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

RHO = 0.99  # solvers.py:63


class DivergenceError(RuntimeError):
    pass


def prox_g(alpha, tau, v):
    return np.asarray(v, dtype=np.float64) / (1.0 + 2.0 * alpha * tau)  # functionals.py:48


def prox_fstar(n, data, sigma, v):
    return (np.asarray(v, dtype=np.float64) - sigma * np.asarray(data, dtype=np.float64)) / (
        1.0 + sigma * n / 2.0)  # functionals.py:66


def g_value(alpha, x):
    x = np.asarray(x, dtype=np.float64)
    return float(alpha * np.vdot(x, x))


def fit_value(n, data, y):
    diff = np.asarray(y, dtype=np.float64) - np.asarray(data, dtype=np.float64)
    return float(np.vdot(diff, diff)) / n


def moduli(alpha, n):
    return 2.0 * alpha, n / 2.0


@dataclass(frozen=True)
class Config:
    mode: str
    sigmas: tuple
    tau: float
    theta: float
    probs: tuple
    epochs: int
    seed: int
    gate_norms: tuple
    stacked_norm_sq: float | None = None

    @property
    def num_gates(self):
        return len(self.sigmas)

    @property
    def iterations_per_epoch(self):
        return 1 if self.mode == "pdhg" else self.num_gates


def default_config(mode, gate_norms, alpha, epochs, seed=0, stacked_norm_sq=None):
    gate_norms = tuple(float(v) for v in gate_norms)
    n = len(gate_norms)
    mu_g, mu_fstar = moduli(alpha, n)
    gamma = math.sqrt(mu_g / mu_fstar)  # solvers.py:224
    if mode == "pdhg":
        probs = (1.0,) * n
        s2 = stacked_norm_sq if stacked_norm_sq is not None else sum(v * v for v in gate_norms)
        s = math.sqrt(s2)
        sigmas = (gamma * RHO / s,) * n
        tau = RHO / (gamma * s)
    elif mode == "spdhg":
        probs = (1.0 / n,) * n
        sigmas = tuple(gamma * RHO / v for v in gate_norms)
        tau = RHO / (gamma * max(v / p for v, p in zip(gate_norms, probs)))
    else:
        raise ValueError(mode)
    return Config(mode, sigmas, tau, 1.0, probs, int(epochs), int(seed), gate_norms,
                  stacked_norm_sq)


def sample_gates(rng, probs, mode):
    if mode == "pdhg":
        return tuple(range(len(probs)))
    p = np.asarray(probs, dtype=np.float64)
    return (int(rng.choice(len(probs), p=p / p.sum())),)  # solvers.py:312


@dataclass
class State:
    x: np.ndarray
    y: list
    z: np.ndarray
    zbar: np.ndarray
    iteration: int = 0
    epoch: float = 0.0
    fwd_calls: int = 0
    adj_calls: int = 0
    last_projections: dict = field(default_factory=dict)

    @classmethod
    def zeros(cls, image_shape, data):
        return cls(np.zeros(image_shape), [np.zeros(d.shape) for d in data],
                   np.zeros(image_shape), np.zeros(image_shape))


def step(state, config, alpha, operators, data, draw):
    """solvers.step restated (solvers.py:316-366)."""
    n = len(operators)
    x_new = prox_g(alpha, config.tau, state.x - config.tau * state.zbar)
    if not np.isfinite(x_new).all():
        raise DivergenceError(f"non-finite primal iterate at iteration {state.iteration + 1}")
    subset = draw()
    while len(subset) == 0:
        subset = draw()
    state.last_projections = {}
    deltas = []
    for i in subset:
        op = operators[i]
        projected = op.apply(x_new)
        state.fwd_calls += 1
        state.last_projections[i] = projected
        y_new = prox_fstar(n, data[i], config.sigmas[i], state.y[i] + config.sigmas[i] * projected)
        if not np.isfinite(y_new).all():
            raise DivergenceError(
                f"non-finite dual iterate (gate {i}) at iteration {state.iteration + 1}")
        delta_z = op.adjoint_apply(y_new - state.y[i])
        state.adj_calls += 1
        state.y[i] = y_new
        deltas.append((i, delta_z))
    for _, delta_z in deltas:
        state.z += delta_z
    state.zbar = state.z.copy()
    for i, delta_z in deltas:
        state.zbar += (config.theta / config.probs[i]) * delta_z
    state.x = x_new
    state.iteration += 1
    state.epoch += len(subset) / n
    return state


def objective(alpha, operators, data, x):
    n = len(operators)
    total = g_value(alpha, x)
    for op, d in zip(operators, data):
        total += fit_value(n, d, op.apply(x))
    return total


def run(config, alpha, operators, data, diagnostics=True, on_epoch=None):
    """solvers.run restated (solvers.py:369-432); returns (state, objectives)."""
    data = [np.asarray(d, dtype=np.float64) for d in data]
    state = State.zeros(operators[0].domain_shape, data)
    rng = np.random.default_rng(config.seed)
    n = len(operators)
    guard = 1e6 * max(sum(fit_value(n, d, np.zeros_like(d)) for d in data),
                      np.finfo(np.float64).tiny)
    objectives = []

    def draw():
        return sample_gates(rng, config.probs, config.mode)

    for epoch_index in range(1, config.epochs + 1):
        for _ in range(config.iterations_per_epoch):
            step(state, config, alpha, operators, data, draw)
        if diagnostics:
            if config.mode == "pdhg" and len(state.last_projections) == n:
                obj = g_value(alpha, state.x) + sum(
                    fit_value(n, data[i], state.last_projections[i]) for i in range(n))
            else:
                obj = objective(alpha, operators, data, state.x)
            if not math.isfinite(obj) or obj > guard:
                raise DivergenceError(
                    f"objective {obj:.3e} exceeded the divergence guard at epoch {epoch_index} "
                    f"(iteration {state.iteration})")
            objectives.append(obj)
        if on_epoch is not None:
            on_epoch(epoch_index, state)
    return state, objectives


def power_method(op, iterations=100, seed=0, rtol=1e-10):
    """linops.power_method restated (linops.py:215-272)."""
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(op.domain_shape)
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return 0.0
    b /= nb
    rayleigh = 0.0
    for _ in range(iterations):
        w = op.adjoint_apply(op.apply(b))
        new_rayleigh = float(np.vdot(b, w)) / float(np.vdot(b, b))
        nw = float(np.linalg.norm(w))
        if nw == 0.0:
            return 0.0
        b = w / nw
        if new_rayleigh > 0 and abs(new_rayleigh - rayleigh) <= rtol * new_rayleigh:
            rayleigh = new_rayleigh
            break
        rayleigh = new_rayleigh
    return float(np.sqrt(max(rayleigh, 0.0)))


class GramSum:
    """linops.GramSumMap restated (linops.py:172-212)."""

    def __init__(self, blocks):
        self.blocks = blocks
        self.domain_shape = self.range_shape = blocks[0].domain_shape

    def apply(self, x):
        out = 0.0 * np.asarray(x, dtype=np.float64)
        for b in self.blocks:
            out += 1.0 * b.adjoint_apply(b.apply(x))
        return out

    adjoint_apply = apply


def stacked_norm_sq(blocks, iterations=100, seed=0):
    return power_method(GramSum(blocks), iterations=iterations, seed=seed)
