"""PDHG / SPDHG solvers on sm_100a (mirror of mctomo.solvers, solvers.py:1-498).

Same API surface and semantics as the reference: ``Problem``, ``SolverConfig``
(admissibility checks), ``default_config`` (strong-convexity-balanced step
sizes), ``SolverState``, ``SaddlePoint``, ``sample_gates``, ``step``, ``run``,
``DivergenceError``, ``RHO``.  One iteration is

    (i)   x <- prox_{tau g}(x - tau*zbar)
    (ii)  for i in S: y_i <- prox_{sigma_i f_i*}(y_i + sigma_i A_i x)
    (iii) z <- z + sum_i A_i^T dy_i;  zbar <- z + sum_i (theta/p_i) A_i^T dy_i

executed as four fused sm_100a kernels (engine.py).  ``run`` pre-draws the
SPDHG gate sequence with the *same* numpy generator calls as the reference
(``default_rng(seed)`` then one ``rng.choice(N, p=p/p.sum())`` per iteration,
solvers.py:312, :392), uploads it once, and replays one CUDA graph per epoch.
Solver state lives on the device in fp32; ``SolverState`` exposes it as
float64 numpy arrays like the reference.

Extensions beyond the reference (the BASELINE workloads need them):
``run_batch`` (independent slices in one launch per kernel, per-slice seeds)
and ``distributed.run_pdhg_sharded`` (PDHG gate-sharded over GPUs).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .engine import U64_MAX_AS_I64, Engine, split_operator
from .experiment_io import ConvergenceRecord, rmse
from .functionals import fit_value, g_value, moduli, prox_fstar, prox_g
from .linops import LinearMap

__all__ = [
    "RHO",
    "DivergenceError",
    "Problem",
    "SolverConfig",
    "SolverState",
    "SaddlePoint",
    "default_config",
    "sample_gates",
    "draw_sequence",
    "step",
    "run",
    "run_batch",
    "cg_reference",
    "optimality_residual",
]

RHO = 0.99  # solvers.py:63
MODES = ("pdhg", "spdhg")


class DivergenceError(RuntimeError):
    """Raised when a solver run leaves the finite/bounded regime."""


@dataclass(frozen=True)
class Problem:
    """Saddle point problem data: operators, data blocks, penalty weight."""

    alpha: float
    operators: tuple
    data: tuple

    def __post_init__(self):
        if not self.alpha > 0:
            raise ValueError("alpha must be positive")
        if not self.operators:
            raise ValueError("at least one gate required")
        if len(self.operators) != len(self.data):
            raise ValueError("one data block per operator required")
        dom = tuple(self.operators[0].domain_shape)
        for k, (op, d) in enumerate(zip(self.operators, self.data)):
            if tuple(op.domain_shape) != dom:
                raise ValueError(f"gate {k} domain mismatch")
            if d.shape != tuple(op.range_shape):
                raise ValueError(
                    f"gate {k} data shape {d.shape} != operator range {tuple(op.range_shape)}")

    @classmethod
    def from_parts(cls, alpha: float, operators: Sequence[LinearMap], data) -> "Problem":
        return cls(alpha=float(alpha), operators=tuple(operators),
                   data=tuple(np.asarray(d, dtype=np.float64) for d in data))

    @property
    def num_gates(self) -> int:
        return len(self.operators)

    @property
    def image_shape(self) -> tuple:
        return tuple(self.operators[0].domain_shape)

    def objective(self, x) -> float:
        """Full objective; applies every gated operator once (on the device)."""
        n = self.num_gates
        total = g_value(self.alpha, x)
        for op, d in zip(self.operators, self.data):
            total += fit_value(n, d, op.apply(np.asarray(x, dtype=np.float64)))
        return total

    def data_objective(self) -> float:
        cache = self.__dict__.setdefault("_cache", {})
        if "data_objective" not in cache:
            n = self.num_gates
            cache["data_objective"] = sum(fit_value(n, d, np.zeros_like(d)) for d in self.data)
        return cache["data_objective"]

    ENGINE_CACHE = 2  # device engines kept per problem (LRU)

    def _engine(self, keep_projections: bool) -> Engine:
        """The device engine run() uses for this (immutable) problem: data, warps and
        workspace uploaded once and reused by later runs (state is reset per run).
        One engine per (device, stream), so runs issued concurrently on different
        streams never share state; at most ``ENGINE_CACHE`` engines stay cached
        (least recently used evicted; a run in flight keeps its own reference).

        The data blocks are uploaded when the engine is built: like the operators,
        ``Problem.data`` must not be modified in place after the first run()
        (build a new Problem instead, or call ``release()``)."""
        torch = _lib.require_cuda()
        cache = self.__dict__.setdefault("_engines", {})
        stream = torch.cuda.current_stream()
        key = (bool(keep_projections), stream.device.index, stream.cuda_stream)
        eng = cache.pop(key, None)
        if eng is None:
            while len(cache) >= self.ENGINE_CACHE:
                cache.pop(next(iter(cache)))
            eng = Engine([self.operators], [self.data], keep_projections=keep_projections)
        cache[key] = eng  # most recently used last
        return eng

    def release(self) -> None:
        """Drop the cached device engines (data, duals, workspace) of this problem."""
        self.__dict__.pop("_engines", None)


@dataclass(frozen=True)
class SolverConfig:
    """Step sizes, sampling law and budget of one run (solvers.py:127-195)."""

    mode: str
    sigmas: tuple
    tau: float
    theta: float
    probs: tuple
    epochs: int
    seed: int
    gate_norms: tuple
    stacked_norm_sq: float | None = None

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        n = len(self.sigmas)
        if n == 0 or len(self.probs) != n or len(self.gate_norms) != n:
            raise ValueError("sigmas, probs, gate_norms must share one length >= 1")
        if not all(s > 0 and math.isfinite(s) for s in self.sigmas):
            raise ValueError("all sigmas must be positive and finite")
        if not (self.tau > 0 and math.isfinite(self.tau)):
            raise ValueError("tau must be positive and finite")
        if not (0 < self.theta <= 1):
            raise ValueError("theta must lie in (0, 1]")
        if not all(0 < p <= 1 for p in self.probs):
            raise ValueError("probabilities must lie in (0, 1]")
        if self.mode == "pdhg" and any(p != 1.0 for p in self.probs):
            raise ValueError("pdhg mode requires all probabilities equal to 1")
        if self.epochs < 0:
            raise ValueError("epochs must be >= 0")
        if not all(v > 0 for v in self.gate_norms):
            raise ValueError("gate norms must be positive")
        slack = 1.0 + 1e-9
        if self.mode == "spdhg":
            for s, p, v in zip(self.sigmas, self.probs, self.gate_norms):
                if s * self.tau * v * v > RHO ** 2 * p * slack:
                    raise ValueError("inadmissible step sizes: sigma*tau*||A_i||^2 exceeds "
                                     f"RHO^2*p_i for a gate with norm {v:.6g}")
        else:
            s2 = (self.stacked_norm_sq if self.stacked_norm_sq is not None
                  else sum(v * v for v in self.gate_norms))
            for s in self.sigmas:
                if s * self.tau * s2 > RHO ** 2 * slack:
                    raise ValueError("inadmissible step sizes: sigma*tau*||stack||^2 exceeds RHO^2")

    @property
    def num_gates(self) -> int:
        return len(self.sigmas)

    @property
    def iterations_per_epoch(self) -> int:
        return 1 if self.mode == "pdhg" else self.num_gates


def default_config(mode: str, gate_norms: Sequence[float], alpha: float, epochs: int,
                   seed: int = 0, stacked_norm_sq: float | None = None) -> SolverConfig:
    """Strong-convexity-balanced step sizes (solvers.py:198-247, the code's rule)."""
    gate_norms = tuple(float(v) for v in gate_norms)
    if not gate_norms:
        raise ValueError("at least one gate norm required")
    if not all(v > 0 for v in gate_norms):
        raise ValueError("gate norms must be positive")
    n = len(gate_norms)
    mu_g, mu_fstar = moduli(alpha, n)
    gamma = math.sqrt(mu_g / mu_fstar)
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
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    return SolverConfig(mode=mode, sigmas=sigmas, tau=tau, theta=1.0, probs=probs,
                        epochs=int(epochs), seed=int(seed), gate_norms=gate_norms,
                        stacked_norm_sq=stacked_norm_sq)


@dataclass
class SaddlePoint:
    """Primal-dual optimum used as the distance reference (solvers.py:279-295)."""

    x_star: np.ndarray
    y_star: list
    source: str
    converged: bool
    residual: float

    def distance_sq(self, x, y) -> float:
        total = float(np.vdot(x - self.x_star, x - self.x_star))
        for yk, ystar in zip(y, self.y_star):
            diff = yk - ystar
            total += float(np.vdot(diff, diff))
        return total


def sample_gates(rng: np.random.Generator, probs: Sequence[float], mode: str) -> tuple:
    """Draw the gate subset for one iteration (solvers.py:298-313)."""
    if mode == "pdhg":
        return tuple(range(len(probs)))
    if mode == "spdhg":
        p = np.asarray(probs, dtype=np.float64)
        return (int(rng.choice(len(probs), p=p / p.sum())),)
    raise ValueError(f"mode must be one of {MODES}, got {mode!r}")


def draw_sequence(config: SolverConfig, iterations: int | None = None,
                  seed: int | None = None) -> np.ndarray:
    """The reference's SPDHG gate sequence, drawn up front on the host.

    Makes exactly the generator calls ``run`` makes (solvers.py:392, :395-396),
    so the sequence is bit-identical to the reference's per-iteration draws.
    """
    if config.mode != "spdhg":
        raise ValueError("only spdhg draws gates at random")
    if iterations is None:
        iterations = config.epochs * config.iterations_per_epoch
    rng = np.random.default_rng(config.seed if seed is None else seed)
    return np.array([sample_gates(rng, config.probs, "spdhg")[0] for _ in range(iterations)],
                    dtype=np.int32)


# ---------------------------------------------------------------------------
class SolverState:
    """Iterate of a run: primal x, duals y_i, aggregates z, zbar, counters.

    Before the first ``step`` the arrays are held on the host; once bound to a
    problem the device buffers are authoritative and the ``x``, ``y``, ``z``,
    ``zbar`` attributes read / write float64 numpy copies (solvers.py:250-276).
    """

    def __init__(self, x, y, z, zbar, iteration: int = 0, epoch: float = 0.0,
                 fwd_calls: int = 0, adj_calls: int = 0, last_projections=None):
        self._engine = None
        self._problem = None
        self._host = {
            "x": np.array(x, dtype=np.float64),
            "y": [np.array(v, dtype=np.float64) for v in y],
            "z": np.array(z, dtype=np.float64),
            "zbar": np.array(zbar, dtype=np.float64),
        }
        self.iteration = iteration
        self.epoch = epoch
        self.fwd_calls = fwd_calls
        self.adj_calls = adj_calls
        self._last = dict(last_projections or {})

    @classmethod
    def _device_zero(cls) -> "SolverState":
        """A zero-counter state whose arrays live on a device engine (bound by run()
        to its engine after reset): no host copies of the N dual blocks."""
        st = cls.__new__(cls)
        st._engine = st._problem = st._host = None
        st.iteration, st.epoch, st.fwd_calls, st.adj_calls = 0, 0.0, 0, 0
        st._last = {}
        return st

    @classmethod
    def zeros(cls, problem: Problem) -> "SolverState":
        shape = problem.image_shape
        return cls(x=np.zeros(shape), y=[np.zeros(d.shape) for d in problem.data],
                   z=np.zeros(shape), zbar=np.zeros(shape))

    # -- device binding ------------------------------------------------------
    def _bind(self, problem: Problem, keep_projections: bool = True) -> Engine:
        if self._engine is not None and self._problem is problem:
            return self._engine
        torch = _lib.require_cuda()
        host = self._host if self._engine is None else self._snapshot_host()
        eng = Engine([problem.operators], [problem.data], keep_projections=keep_projections)
        eng.x[0].copy_(torch.from_numpy(host["x"].astype(np.float32)))
        eng.z[0].copy_(torch.from_numpy(host["z"].astype(np.float32)))
        eng.zbar[0].copy_(torch.from_numpy(host["zbar"].astype(np.float32)))
        if len(host["y"]) != problem.num_gates:
            raise ValueError("state has a different number of dual blocks than the problem")
        for i, v in enumerate(host["y"]):
            eng.y[0, i].copy_(torch.from_numpy(np.asarray(v, dtype=np.float32)))
        self._engine, self._problem, self._host = eng, problem, None
        return eng

    def _snapshot_host(self):
        return {"x": self.x, "y": self.y, "z": self.z, "zbar": self.zbar}

    def _get(self, name):
        if self._engine is None:
            v = self._host[name]
            return [a for a in v] if name == "y" else v
        t = getattr(self._engine, name)
        if name == "y":
            return [t[0, i].double().cpu().numpy() for i in range(t.shape[1])]
        return t[0].double().cpu().numpy()

    def _set(self, name, value):
        if self._engine is None:
            if name == "y":
                self._host["y"] = [np.array(v, dtype=np.float64) for v in value]
            else:
                self._host[name] = np.array(value, dtype=np.float64)
            return
        torch = _lib.require_cuda()
        t = getattr(self._engine, name)
        if name == "y":
            for i, v in enumerate(value):
                t[0, i].copy_(torch.from_numpy(np.asarray(v, dtype=np.float32)))
        else:
            t[0].copy_(torch.from_numpy(np.asarray(value, dtype=np.float32)))

    x = property(lambda s: s._get("x"), lambda s, v: s._set("x", v))
    y = property(lambda s: s._get("y"), lambda s, v: s._set("y", v))
    z = property(lambda s: s._get("z"), lambda s, v: s._set("z", v))
    zbar = property(lambda s: s._get("zbar"), lambda s, v: s._set("zbar", v))

    @property
    def last_projections(self) -> dict:
        if self._engine is None or self._engine.proj is None:
            return dict(self._last)
        return {i: self._engine.proj[0, i].double().cpu().numpy() for i in self._last}

    @last_projections.setter
    def last_projections(self, value):
        self._last = dict(value)


def _raise_status(eng: Engine):
    primal, dual = eng.read_status()
    if primal is not None and (dual is None or primal <= dual[0]):
        raise DivergenceError(f"non-finite primal iterate at iteration {primal}")
    if dual is not None:
        raise DivergenceError(f"non-finite dual iterate (gate {dual[1]}) at iteration {dual[0]}")


def fused(problem: Problem) -> bool:
    """True when every operator of ``problem`` is a gated operator of this package
    (RayTransform, or a ray transform composed with a warp): ``step`` / ``run`` then
    execute the fused sm_100a iteration.  Any other map honouring the reference's
    LinearMap contract (linops.py:39-73) runs through ``_operator_step``."""
    try:
        for op in problem.operators:
            split_operator(op)
    except TypeError:
        return False
    return True


def _operator_step(state: SolverState, config: SolverConfig, problem: Problem,
                   draw: Callable[[], tuple]) -> SolverState:
    """One iteration over operators the fused engine does not know (solvers.py:316-366):
    the maps' own ``apply`` / ``adjoint_apply`` (wherever those compute) sequenced
    on float64 arrays, in the reference's order -- primal check before the draw,
    y_i assigned gate by gate, z / zbar / x only after every gate passed."""
    if state._engine is not None:  # a state last advanced by the fused engine
        state._host, state._engine, state._problem = state._snapshot_host(), None, None
    h = state._host
    n = problem.num_gates
    x_next = prox_g(problem.alpha, config.tau, h["x"] - config.tau * h["zbar"])
    if not np.isfinite(x_next).all():
        raise DivergenceError(f"non-finite primal iterate at iteration {state.iteration + 1}")
    subset = draw()
    while len(subset) == 0:
        subset = draw()
    state._last = {}
    updates = []
    for i in subset:
        op, sigma = problem.operators[i], config.sigmas[i]
        ax = np.asarray(op.apply(x_next), dtype=np.float64)
        state.fwd_calls += 1
        state._last[i] = ax
        y_next = prox_fstar(n, problem.data[i], sigma, h["y"][i] + sigma * ax)
        if not np.isfinite(y_next).all():
            raise DivergenceError(
                f"non-finite dual iterate (gate {i}) at iteration {state.iteration + 1}")
        updates.append((i, np.asarray(op.adjoint_apply(y_next - h["y"][i]), dtype=np.float64)))
        state.adj_calls += 1
        h["y"][i] = y_next
    for _, dz in updates:
        h["z"] += dz
    h["zbar"] = h["z"].copy()
    for i, dz in updates:
        h["zbar"] += (config.theta / config.probs[i]) * dz
    h["x"] = x_next
    state.iteration += 1
    state.epoch += len(subset) / n
    return state


def _operator_run(config: SolverConfig, problem: Problem, saddle, truth, on_epoch):
    """run() over operators the fused engine does not know (solvers.py:369-432)."""
    state = SolverState.zeros(problem)
    record = ConvergenceRecord()
    rng = np.random.default_rng(config.seed)
    guard = _guard(problem.data_objective())
    n = problem.num_gates
    for epoch_index in range(1, config.epochs + 1):
        for _ in range(config.iterations_per_epoch):
            _operator_step(state, config, problem,
                           lambda: sample_gates(rng, config.probs, config.mode))
        last = state.last_projections
        if config.mode == "pdhg" and len(last) == n:  # reuse this epoch's projections
            value = g_value(problem.alpha, state.x) + sum(
                fit_value(n, problem.data[i], last[i]) for i in range(n))
        else:
            value = problem.objective(state.x)
        if not math.isfinite(value) or value > guard:
            raise DivergenceError(
                f"objective {value:.3e} exceeded the divergence guard "
                f"at epoch {epoch_index} (iteration {state.iteration})")
        record.append(epoch=float(epoch_index),
                      dist_sq=saddle.distance_sq(state.x, state.y) if saddle is not None
                      else math.nan,
                      objective=value,
                      rmse_to_truth=rmse(state.x, truth) if truth is not None else math.nan,
                      fwd_calls=state.fwd_calls, adj_calls=state.adj_calls)
        if on_epoch is not None:
            on_epoch(epoch_index, state)
    return state.x.copy(), record


def step(state: SolverState, config: SolverConfig, problem: Problem,
         draw: Callable[[], tuple]) -> SolverState:
    """Advance the state by one iteration in place (solvers.py:316-366).

    ``draw`` supplies the gate subset; an empty draw is retried.  Raises
    :class:`DivergenceError` on the first non-finite iterate.
    """
    n = problem.num_gates
    if config.num_gates != n:
        raise ValueError("config and problem disagree on the gate count")
    if not fused(problem):
        return _operator_step(state, config, problem, draw)
    torch = _lib.require_cuda()
    eng = state._bind(problem)
    eng.set_params(config)
    subset = draw()
    while len(subset) == 0:
        subset = draw()
    subset = tuple(int(i) for i in subset)
    if any(i < 0 or i >= n for i in subset):
        raise ValueError("drawn gate out of range")
    if len(set(subset)) != len(subset):
        raise ValueError("a draw may not repeat a gate within one iteration")
    gates = torch.tensor(subset, dtype=torch.int32, device=eng.device)
    # the fused iteration updates x, z, zbar and the drawn y_i in place: keep the
    # pre-step values so that a DivergenceError leaves the state where the
    # reference's would be (it raises before assigning x, z and the failing y_i)
    saved = [t.clone() for t in (eng.x, eng.z, eng.zbar)] + [eng.y[0, i].clone() for i in subset]
    eng.iteration(eng.items_subset(gates, len(subset), state.iteration + 1), problem.alpha)
    primal, dual = eng.read_status()
    if primal is not None or dual is not None:
        for t, v in zip((eng.x, eng.z, eng.zbar), saved[:3]):
            t.copy_(v)
        # a dual failure at subset position k: gates before k keep their new y_i
        # (solvers.py:341-358 assigns y_i gate by gate); the primal check fails first
        k = 0 if primal is not None else subset.index(dual[1])
        for pos in range(k, len(subset)):
            eng.y[0, subset[pos]].copy_(saved[3 + pos])
        if primal is None:
            state.fwd_calls += k + 1
            state.adj_calls += k
            state.last_projections = {i: None for i in subset[:k + 1]}
        try:
            _raise_status(eng)
        finally:
            eng.status.fill_(U64_MAX_AS_I64)
    state.fwd_calls += len(subset)
    state.adj_calls += len(subset)
    state.last_projections = {i: None for i in subset}
    state.iteration += 1
    state.epoch += len(subset) / n
    return state


SYNC_EPOCHS = 32  # run(): epochs between host reads of the device diagnostics table


def _guard(problem_data_objective: float) -> float:
    return 1e6 * max(problem_data_objective, np.finfo(np.float64).tiny)


def run(config: SolverConfig, problem: Problem, saddle: SaddlePoint | None = None,
        truth=None, on_epoch: Callable | None = None, *, graph: bool = True,
        diagnostics: bool = True):
    """Run ``config.epochs`` full data passes (solvers.py:369-419).

    Returns ``(x, ConvergenceRecord)`` with x a float64 numpy array.  Per-epoch
    diagnostics (objective, distance to ``saddle``, rmse to ``truth``) are
    computed on the device and are not counted as solver work.  With
    ``diagnostics=False`` the objective column is NaN and only the non-finite
    iterate checks guard the run (the timed benchmark configuration).
    """
    if config.num_gates != problem.num_gates:
        raise ValueError("config and problem disagree on the gate count")
    if not fused(problem):
        return _operator_run(config, problem, saddle, truth, on_epoch)
    record = ConvergenceRecord()
    if config.epochs == 0:
        return np.zeros(problem.image_shape), record
    state = SolverState._device_zero()  # bound to the engine below (no host arrays)
    torch = _lib.require_cuda()
    keep = diagnostics and config.mode == "pdhg"
    eng = problem._engine(keep)  # zero state below == SolverState.zeros(problem)
    state._engine, state._problem, state._host = eng, problem, None
    eng.set_params(config)
    eng.reset()
    n = problem.num_gates
    if config.mode == "spdhg":
        eng.set_sequences(draw_sequence(config)[None, :])
    guard = _guard(problem.data_objective())
    ipe = config.iterations_per_epoch
    g = eng.epoch_graph(config.mode, problem.alpha) if graph else None
    xs = ys = tr = None
    if saddle is not None:
        xs = torch.from_numpy(np.asarray(saddle.x_star, dtype=np.float32)).to(eng.device)
        ys = torch.from_numpy(np.stack([np.asarray(v, dtype=np.float32)
                                        for v in saddle.y_star])).to(eng.device)
    if truth is not None:
        tr = torch.from_numpy(np.asarray(truth, dtype=np.float32)).to(eng.device)
    # Per-epoch diagnostics are written into a device table (no host sync) and
    # read back every SYNC_EPOCHS epochs (every epoch with an on_epoch callback).
    # Rows are then checked in order exactly as the reference does after each
    # epoch: the first non-finite iterate (device status words) raises first,
    # then the objective guard, so the error message names the same epoch /
    # iteration; nothing later than the raising epoch reaches the record.
    cols = n + 4  # ||A_i x - d_i||^2 (n), ||x||^2, ||x - x*||^2, ||y - y*||^2, ||x - truth||^2
    table = torch.full((config.epochs, cols), math.nan, dtype=torch.float64, device=eng.device)
    sync_every = 1 if on_epoch is not None else SYNC_EPOCHS
    pending = []
    st = _lib.stream_handle()  # one stream per run: query it once
    table_ptr = _lib.ptr(table)

    def flush():
        if not pending:
            return
        rows = table[pending[0] - 1:pending[-1]].cpu().numpy()
        primal, dual = eng.read_status()
        bad = [v for v in (primal, dual[0] if dual is not None else None) if v is not None]
        bad_epoch = (min(bad) + ipe - 1) // ipe if bad else None
        for k, e in enumerate(pending):
            if bad_epoch is not None and e >= bad_epoch:
                _raise_status(eng)
            row = rows[k]
            objective_value = math.nan
            if diagnostics:
                objective_value = float(problem.alpha * row[n] + sum(row[i] / n for i in range(n)))
                if not math.isfinite(objective_value) or objective_value > guard:
                    raise DivergenceError(
                        f"objective {objective_value:.3e} exceeded the divergence guard "
                        f"at epoch {e} (iteration {e * ipe})")
            dist = float(row[n + 1] + row[n + 2]) if xs is not None else math.nan
            err = math.sqrt(float(row[n + 3]) / eng.n_img) if tr is not None else math.nan
            record.append(epoch=float(e), dist_sq=dist, objective=objective_value,
                          rmse_to_truth=err, fwd_calls=e * n, adj_calls=e * n)
        pending.clear()

    for epoch_index in range(1, config.epochs + 1):
        if g is not None:
            g.replay()
        else:
            eng.epoch(config.mode, problem.alpha)
        state.iteration += ipe
        state.epoch += 1.0
        state.fwd_calls += n
        state.adj_calls += n
        if config.mode == "pdhg":
            state.last_projections = {i: None for i in range(n)}
        fit_row = table_ptr + 8 * cols * (epoch_index - 1)  # raw fp64 addresses of the row
        xx_row, xd_row, yd_row, tr_row = (fit_row + 8 * (n + k) for k in range(4))
        if diagnostics:
            eng.objective_parts(config.mode == "pdhg", fit_out=fit_row, xx_out=xx_row, st=st)
        if xs is not None:
            eng.reduce(eng.x[0], xs, 1, eng.n_img, _lib.REDUCE_SQDIFF, out=xd_row, st=st)
            eng.reduce(eng.y[0], ys, 1, eng.N * eng.n_sino, _lib.REDUCE_SQDIFF, out=yd_row,
                       st=st)
        if tr is not None:
            eng.reduce(eng.x[0], tr, 1, eng.n_img, _lib.REDUCE_SQDIFF, out=tr_row, st=st)
        pending.append(epoch_index)
        if len(pending) >= sync_every or epoch_index == config.epochs:
            flush()
        if on_epoch is not None:
            on_epoch(epoch_index, state)
    return state.x, record


def run_batch(configs: Sequence[SolverConfig], problems: Sequence[Problem], *,
              graph: bool = True, diagnostics: bool = False):
    """Independent slices solved together (BASELINE C5).

    All problems share one geometry, gate count, mode, step-size rule and
    alpha per slice is honoured only if equal; each slice keeps its own warps,
    data and sampling seed.  Returns a list of ``(x, ConvergenceRecord)``.
    """
    if len(configs) != len(problems) or not problems:
        raise ValueError("one config per problem required")
    c0, p0 = configs[0], problems[0]
    for c, p in zip(configs, problems):
        if c.num_gates != p.num_gates or p.num_gates != p0.num_gates:
            raise ValueError("all slices need the same gate count")
        if (c.mode, c.sigmas, c.tau, c.theta, c.probs, c.epochs) != \
                (c0.mode, c0.sigmas, c0.tau, c0.theta, c0.probs, c0.epochs):
            raise ValueError("batched slices must share step sizes and budget (seeds may differ)")
        if p.alpha != p0.alpha:
            raise ValueError("batched slices must share alpha")
    eng = BatchRunner(configs, problems, keep_projections=diagnostics and c0.mode == "pdhg")
    return eng.run(graph=graph, diagnostics=diagnostics)


class BatchRunner:
    """Engine wrapper for S independent slices (used by run_batch and bench)."""

    def __init__(self, configs, problems, keep_projections=False):
        self.configs = list(configs)
        self.problems = list(problems)
        c0 = self.configs[0]
        self.engine = Engine([p.operators for p in problems], [p.data for p in problems],
                             keep_projections=keep_projections,
                             max_items=len(problems) if c0.mode == "spdhg" else None)
        self.engine.set_params(c0)
        self.mode = c0.mode
        self.alpha = problems[0].alpha
        if self.mode == "spdhg":
            self.engine.set_sequences(np.stack([draw_sequence(c) for c in configs]))

    def run(self, graph=True, diagnostics=False):
        eng = self.engine
        c0 = self.configs[0]
        S = len(self.problems)
        records = [ConvergenceRecord() for _ in range(S)]
        eng.reset()
        g = eng.epoch_graph(self.mode, self.alpha) if graph else None
        n = c0.num_gates
        for e in range(1, c0.epochs + 1):
            if g is not None:
                g.replay()
            else:
                eng.epoch(self.mode, self.alpha)
            objs = [math.nan] * S
            if diagnostics:
                _raise_status(eng)
                objs = eng.objectives(self.alpha, self.mode == "pdhg")
            for s in range(S):
                records[s].append(epoch=float(e), dist_sq=math.nan, objective=objs[s],
                                  rmse_to_truth=math.nan, fwd_calls=e * n, adj_calls=e * n)
        _raise_status(eng)
        xs = eng.x.double().cpu().numpy()
        return [(xs[s], records[s]) for s in range(S)]


# ---------------------------------------------------------------------------
class _DeviceGram:
    """x -> alpha*x + (1/N) sum_i A_i^T A_i x on the device (GramSumMap, linops.py:172-212).

    fp64 vectors, fp32 operator applications (the sm_100a kernels), fp64
    accumulation with the library's mixed-precision axpby / fixed-order dots.
    """

    def __init__(self, problem: Problem):
        torch = _lib.require_cuda()
        self.torch = torch
        self.eng = Engine([problem.operators], [problem.data], max_items=1)
        self.n = problem.num_gates
        self.alpha = float(problem.alpha)
        self.shape = problem.image_shape
        self.size = int(np.prod(self.shape))
        dev = self.eng.device
        self.p32 = torch.empty(self.shape, dtype=torch.float32, device=dev)
        self.s32 = torch.empty(problem.operators[0].range_shape, dtype=torch.float32, device=dev)
        self.g32 = torch.empty(self.shape, dtype=torch.float32, device=dev)
        self.dot_out = torch.empty(1, dtype=torch.float64, device=dev)

    def axpby(self, alpha, x, beta, y):
        _lib.check(_lib.load().mct_axpby_mixed(
            x.numel(), float(alpha), _lib.ptr(x), int(x.dtype == self.torch.float64), float(beta),
            _lib.ptr(y), int(y.dtype == self.torch.float64), _lib.stream_handle()))

    def dot(self, a, b) -> float:
        _lib.check(_lib.load().mct_dot_f64(_lib.ptr(a), _lib.ptr(b), a.numel(),
                                            _lib.ptr(self.dot_out),
                                            _lib.ptr(_lib.scratch(a.device)),
                                            _lib.stream_handle()))
        return float(self.dot_out.item())

    def rhs(self, out):
        """out = (1/N) sum_i A_i^T d_i (fp64)."""
        out.zero_()
        for i in range(self.n):
            self.eng.gated_adjoint(0, i, self.eng.d[0, i], self.g32)
            self.axpby(1.0 / self.n, self.g32, 1.0, out)

    def apply(self, p, out):
        self.axpby(1.0, p, 0.0, self.p32)              # fp64 -> fp32 operand
        self.axpby(self.alpha, p, 0.0, out)            # out = alpha p
        for i in range(self.n):
            self.eng.gated_forward(0, i, self.p32, self.s32)
            self.eng.gated_adjoint(0, i, self.s32, self.g32)
            self.axpby(1.0 / self.n, self.g32, 1.0, out)


def cg_reference(problem: Problem, tol: float = 1e-12, max_iter: int = 500) -> SaddlePoint:
    """Saddle point by CG on the normal equations, on the device (solvers.py:435-490).

    Solves (alpha I + (1/N) sum_i A_i^T A_i) x = (1/N) sum_i A_i^T d_i from zero
    and recovers y_i = (2/N)(A_i x - d_i).  Vectors and reductions are fp64, the
    operator applications fp32 (the sm_100a kernels), so the attainable relative
    residual is ~1e-7; ``converged`` reports honestly whether ``tol`` was met
    and ``residual`` is the true relative residual recomputed at the end.
    """
    if not (tol > 0):
        raise ValueError("tol must be positive")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    torch = _lib.require_cuda()
    G = _DeviceGram(problem)
    f64 = dict(dtype=torch.float64, device=G.eng.device)
    b = torch.empty(G.shape, **f64)
    G.rhs(b)
    b_norm = math.sqrt(G.dot(b, b))
    x = torch.zeros(G.shape, **f64)
    converged = True
    mp = torch.empty(G.shape, **f64)
    if b_norm > 0:
        r = b.clone()
        p = r.clone()
        rs = G.dot(r, r)
        converged = False
        for _ in range(max_iter):
            if math.sqrt(rs) <= tol * b_norm:
                converged = True
                break
            G.apply(p, mp)
            alpha_cg = rs / G.dot(p, mp)
            G.axpby(alpha_cg, p, 1.0, x)
            G.axpby(-alpha_cg, mp, 1.0, r)
            rs_new = G.dot(r, r)
            G.axpby(1.0, r, rs_new / rs, p)   # p = r + beta p
            rs = rs_new
        else:
            converged = math.sqrt(rs) <= tol * b_norm
    G.apply(x, mp)
    G.axpby(1.0, b, -1.0, mp)                 # mp = b - normal(x)
    true_residual = math.sqrt(G.dot(mp, mp))
    residual = true_residual / b_norm if b_norm > 0 else 0.0
    x_star = x.cpu().numpy()
    n = problem.num_gates
    y_star = [(2.0 / n) * (op.apply(x_star) - d) for op, d in zip(problem.operators, problem.data)]
    return SaddlePoint(x_star=x_star, y_star=y_star, source="cg_reference", converged=converged,
                       residual=residual)


def optimality_residual(problem: Problem, saddle: SaddlePoint) -> float:
    """Norm of 2 alpha x* + sum_i A_i^T y*_i (solvers.py:493-498), A_i^T on the device."""
    defect = 2.0 * problem.alpha * np.asarray(saddle.x_star, dtype=np.float64)
    for op, y in zip(problem.operators, saddle.y_star):
        defect = defect + op.adjoint_apply(y)
    return float(np.linalg.norm(defect))
