"""CPU tier: the product's ``step`` / ``run`` / ``power_method`` on operators that are
not this package's gated operators (reference LinearMap contract, linops.py:39-73).

The reference's solver known-answer tests (test_solvers.py:285-483: toy one- and
two-step iterates, theta scaling, empty draws, zero data, saddle fixed points,
aggregate invariant, full-sampling equivalence, run columns and counters,
divergence guard) run here against the product API with host numpy maps -- the
foreign operators compute, the solver sequences them.  The package's own gated
operators always take the fused sm_100a engine (tests/test_gpu_solver.py).
"""

import math

import numpy as np
import pytest

import paper_2410_10503_b200 as m
from paper_2410_10503_b200.solvers import fused


class HostMatrix:
    """A foreign map: dense matrix on flattened grids (numpy, not a package class)."""

    def __init__(self, mat, dom, rng):
        self.mat = np.asarray(mat, dtype=np.float64)
        self.domain_shape, self.range_shape = tuple(dom), tuple(rng)

    def apply(self, x):
        return (self.mat @ np.ravel(x)).reshape(self.range_shape)

    def adjoint_apply(self, y):
        return (self.mat.T @ np.ravel(y)).reshape(self.domain_shape)


class HostDiagonal(HostMatrix):
    def __init__(self, diag):
        d = np.asarray(diag, dtype=np.float64)
        super().__init__(np.diag(d.ravel()), d.shape, d.shape)


def toy():
    return m.Problem.from_parts(0.25, [HostDiagonal(np.ones((1, 1)))], [np.array([[3.5]])])


def toy_cfg(epochs=1, theta=1.0):
    return m.SolverConfig(mode="pdhg", sigmas=(1.5,), tau=0.5, theta=theta, probs=(1.0,),
                          epochs=epochs, seed=0, gate_norms=(1.0,))


def dense(gates=3, dom=(4, 4), rng_shape=(3, 4), alpha=0.05, seed=0):
    r = np.random.default_rng(seed)
    rows, cols = int(np.prod(rng_shape)), int(np.prod(dom))
    mats = [r.standard_normal((rows, cols)) / 4.0 for _ in range(gates)]
    ops = [HostMatrix(a, dom, rng_shape) for a in mats]
    data = [r.standard_normal(rng_shape) for _ in range(gates)]
    norms = [float(np.linalg.svd(a, compute_uv=False)[0]) for a in mats]
    stacked = float(np.linalg.svd(np.vstack(mats), compute_uv=False)[0]) ** 2
    return m.Problem.from_parts(alpha, ops, data), norms, stacked, mats


def saddle_of(problem, mats):
    n = problem.num_gates
    lhs = problem.alpha * np.eye(mats[0].shape[1]) + sum(a.T @ a for a in mats) / n
    rhs = sum(a.T @ np.ravel(d) for a, d in zip(mats, problem.data)) / n
    x = np.linalg.solve(lhs, rhs).reshape(problem.image_shape)
    y = [(2.0 / n) * (op.apply(x) - d) for op, d in zip(problem.operators, problem.data)]
    return x, y


def test_foreign_operators_take_the_generic_path():
    assert not fused(toy())
    geom = m.Geometry(8, 8, 4, 13, 1.0)
    gated = m.Problem.from_parts(0.1, [m.RayTransform(geom)], [np.zeros((4, 13))])
    assert fused(gated)


def test_one_step_toy_exact():
    problem, st = toy(), None
    st = m.SolverState.zeros(problem)
    m.step(st, toy_cfg(), problem, lambda: (0,))
    # x stays 0 (prox at zero); y = (0 - 1.5*3.5)/(1 + 0.75) = -3; zbar = z + dz
    assert st.x[0, 0] == 0.0 and st.y[0][0, 0] == -3.0
    assert st.z[0, 0] == -3.0 and st.zbar[0, 0] == -6.0
    assert (st.iteration, st.epoch, st.fwd_calls, st.adj_calls) == (1, 1.0, 1, 1)


def test_two_step_toy_fractions():
    problem = toy()
    st = m.SolverState.zeros(problem)
    for _ in range(2):
        m.step(st, toy_cfg(), problem, lambda: (0,))
    assert st.x[0, 0] == pytest.approx(12 / 5, rel=1e-14)
    assert st.y[0][0, 0] == pytest.approx(-93 / 35, rel=1e-14)
    assert st.z[0, 0] == pytest.approx(-93 / 35, rel=1e-14)
    assert st.zbar[0, 0] == pytest.approx(-81 / 35, rel=1e-14)


def test_theta_scales_extrapolation():
    problem = toy()
    st = m.SolverState.zeros(problem)
    m.step(st, toy_cfg(theta=0.5), problem, lambda: (0,))
    assert st.zbar[0, 0] == -4.5


def test_empty_draws_are_retried():
    problem = toy()
    st = m.SolverState.zeros(problem)
    draws = iter([(), (), (0,)])
    m.step(st, toy_cfg(), problem, lambda: next(draws))
    assert (st.fwd_calls, st.iteration, st.epoch) == (1, 1, 1.0)


def test_zero_data_stays_zero():
    problem = m.Problem.from_parts(0.25, [HostDiagonal(np.ones((2, 2)))], [np.zeros((2, 2))])
    x, rec = m.run(toy_cfg(epochs=4), problem)
    assert np.array_equal(x, np.zeros((2, 2))) and rec.objective == [0.0] * 4


@pytest.mark.parametrize("mode,draws", [("pdhg", [(0, 1, 2)]), ("spdhg", [(1,), (0,), (2,), (2,)])])
def test_saddle_is_a_fixed_point(mode, draws):
    problem, norms, stacked, mats = dense()
    xs, ys = saddle_of(problem, mats)
    cfg = m.default_config(mode, norms, problem.alpha, 1,
                           stacked_norm_sq=stacked if mode == "pdhg" else None)
    z = sum(op.adjoint_apply(y) for op, y in zip(problem.operators, ys))
    st = m.SolverState(x=xs, y=[y.copy() for y in ys], z=z, zbar=z)
    for d in draws:
        m.step(st, cfg, problem, lambda d=d: d)
    assert np.linalg.norm(st.x - xs) <= 1e-10 * float(np.linalg.norm(xs))
    if mode == "pdhg":
        for a, b in zip(st.y, ys):
            assert np.linalg.norm(a - b) <= 1e-10 * max(1.0, float(np.linalg.norm(b)))


def test_aggregate_tracks_duals():
    problem, norms, _, _ = dense(gates=4, seed=3)
    cfg = m.default_config("spdhg", norms, problem.alpha, 1, seed=5)
    st = m.SolverState.zeros(problem)
    rng = np.random.default_rng(cfg.seed)
    for _ in range(25):
        before = [y.copy() for y in st.y]
        m.step(st, cfg, problem, lambda: m.sample_gates(rng, cfg.probs, "spdhg"))
        agg = sum(op.adjoint_apply(y) for op, y in zip(problem.operators, st.y))
        scale = max(1.0, float(np.linalg.norm(agg)))
        assert np.linalg.norm(st.z - agg) <= 1e-10 * scale
        moved = [i for i, (a, b) in enumerate(zip(st.y, before)) if not np.array_equal(a, b)]
        assert len(moved) <= 1
        for i in moved:
            dz = problem.operators[i].adjoint_apply(st.y[i] - before[i])
            assert np.linalg.norm(st.zbar - (st.z + dz / cfg.probs[i])) <= 1e-10 * scale


def test_full_draw_spdhg_equals_pdhg_bitwise():
    problem, norms, stacked, _ = dense(gates=3, rng_shape=(5, 3), seed=11)
    pcfg = m.default_config("pdhg", norms, problem.alpha, 10, stacked_norm_sq=stacked)
    x_pdhg, _ = m.run(pcfg, problem)
    full = m.SolverConfig(mode="spdhg", sigmas=pcfg.sigmas, tau=pcfg.tau, theta=1.0,
                          probs=(1.0,) * 3, epochs=10, seed=0, gate_norms=tuple(norms))
    st = m.SolverState.zeros(problem)
    for _ in range(10):
        m.step(st, full, problem, lambda: (0, 1, 2))
    assert np.array_equal(st.x, x_pdhg)


def test_run_columns_counters_and_determinism():
    problem, norms, stacked, mats = dense()
    cfg = m.default_config("pdhg", norms, problem.alpha, 3, stacked_norm_sq=stacked)
    _, bare = m.run(cfg, problem)
    assert all(math.isnan(v) for v in bare.dist_sq + bare.rmse_to_truth)
    xs, ys = saddle_of(problem, mats)
    sp = m.SaddlePoint(x_star=xs, y_star=ys, source="dense solve", converged=True, residual=0.0)
    _, full = m.run(cfg, problem, saddle=sp, truth=np.zeros(problem.image_shape))
    assert full.dist_sq == sorted(full.dist_sq, reverse=True) and min(full.dist_sq) > 0
    assert full.epochs == [1.0, 2.0, 3.0] and full.fwd_calls == [3, 6, 9] == full.adj_calls
    p4, n4, _, _ = dense(gates=4, seed=2)
    scfg = m.default_config("spdhg", n4, p4.alpha, 6, seed=9)
    x1, r1 = m.run(scfg, p4)
    x2, r2 = m.run(scfg, p4)
    assert np.array_equal(x1, x2) and r1.objective == r2.objective
    assert r1.fwd_calls == [4, 8, 12, 16, 20, 24]
    seen = []
    m.run(toy_cfg(epochs=3), toy(), on_epoch=lambda e, s: seen.append((e, s.iteration)))
    assert seen == [(1, 1), (2, 2), (3, 3)]
    with pytest.raises(ValueError, match="gate count"):
        m.run(m.default_config("spdhg", norms[:2], problem.alpha, 1), problem)


def test_divergence_guard_fires():
    problem = m.Problem.from_parts(0.25, [HostDiagonal(np.full((2, 2), 60.0))], [np.ones((2, 2))])
    with pytest.raises(m.DivergenceError):
        m.run(m.default_config("pdhg", (0.01,), problem.alpha, 500), problem)


def test_power_method_on_foreign_maps():
    """linops.py:215-289 for maps outside the package: seeded start, early stop."""
    problem, norms, stacked, mats = dense(seed=4)
    for op, nrm in zip(problem.operators, norms):
        assert m.power_method(op, iterations=500) == pytest.approx(nrm, rel=1e-6)
    assert m.stacked_norm_sq(problem.operators, iterations=500) == pytest.approx(stacked, rel=1e-6)
    with pytest.warns(RuntimeWarning):
        assert m.power_method(HostDiagonal(np.zeros((2, 2)))) == 0.0
