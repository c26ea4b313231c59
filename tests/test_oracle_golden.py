"""CPU tier: pin the oracle against golden vectors produced by the reference itself.

The oracle (oracle/, test infrastructure) is the checker for every GPU parity
test, so it is pinned first: against the reference's own outputs
(tests/golden/make_golden.py) and against the reference test-suite's
known-answer cases (test_solvers.py:285-327, test_projector.py:62-104,
test_motion.py:47-89).
"""

import math

import numpy as np
import pytest

import oracle
from oracle import solver as osolver
from conftest import rel_l2

GEOMS = ["fast", "rect_spacing", "tiny", "many_angles", "axis_exact", "half_spacing", "lin",
         "c1", "odd_rect"]


def _geom(g):
    r, c, a, b, sp = g
    return oracle.Geometry(int(r), int(c), int(a), int(b), float(sp))


@pytest.mark.parametrize("name", GEOMS)
def test_oracle_ray_forward_matches_reference(golden_projector, name):
    G = golden_projector
    op = oracle.RayTransform(_geom(G[f"{name}__geom"]))
    out = op.apply(G[f"{name}__x"])
    assert np.max(np.abs(out - G[f"{name}__Ax"])) <= 1e-13 * max(1.0, np.abs(G[f"{name}__Ax"]).max())


@pytest.mark.parametrize("name", GEOMS)
def test_oracle_ray_adjoint_bitwise_reference_order(golden_projector, name):
    # single-threaded, the oracle scatters in the reference's bincount order
    G = golden_projector
    op = oracle.RayTransform(_geom(G[f"{name}__geom"]), threads=1)
    assert np.array_equal(op.adjoint_apply(G[f"{name}__y"]), G[f"{name}__ATy"])


@pytest.mark.parametrize("name", ["fast", "c1"])
def test_oracle_threaded_equals_serial(golden_projector, name):
    G = golden_projector
    geom = _geom(G[f"{name}__geom"])
    a1 = oracle.RayTransform(geom, threads=1)
    a4 = oracle.RayTransform(geom, threads=4)
    x, y = G[f"{name}__x"], G[f"{name}__y"]
    assert np.array_equal(a1.apply(x), a4.apply(x))
    assert rel_l2(a4.adjoint_apply(y), a1.adjoint_apply(y)) <= 1e-14


def test_oracle_adjoint_identity(golden_projector):
    G = golden_projector
    for name in GEOMS:
        x, y = G[f"{name}__x"], G[f"{name}__y"]
        lhs = float(np.vdot(G[f"{name}__Ax"], y))
        rhs = float(np.vdot(x, G[f"{name}__ATy"]))
        assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), abs(rhs))


WARPS = ["rigid_a", "rigid_b", "dilatation", "quarter", "half", "shift", "out_of_frame",
         "c1_like", "shrink"]


def _owarp(G, name):
    rot, tr, tc, sc = G[f"{name}__params"]
    shape = tuple(int(v) for v in G[f"{name}__shape"])
    kind = oracle.RIGID if int(G[f"{name}__kind"]) == 0 else oracle.DILATATION
    return oracle.Warp(shape, kind, rotation=rot, translation=(tr, tc), scale=sc)


@pytest.mark.parametrize("name", WARPS)
def test_oracle_warps_bitwise(golden_warps, name):
    G = golden_warps
    w = _owarp(G, name)
    assert np.array_equal(w.apply(G[f"{name}__x"]), G[f"{name}__Dx"])
    assert np.array_equal(w.adjoint_apply(G[f"{name}__y"]), G[f"{name}__DTy"])


def rigid_field(shape, rot, tr, tc):
    """Pull-back displacement of a rigid warp (motion.py:139-156 in pixel units)."""
    rows, cols = shape
    cs, sn = math.cos(rot), math.sin(rot)
    if abs(cs) < 1e-15:
        cs = 0.0
    if abs(sn) < 1e-15:
        sn = 0.0
    u = np.arange(rows) - (rows - 1) / 2.0
    v = np.arange(cols) - (cols - 1) / 2.0
    uu, vv = np.meshgrid(u, v, indexing="ij")
    du, dv = uu - tr, vv - tc
    su = cs * du + sn * dv
    sv = -sn * du + cs * dv
    return np.stack([su - uu, sv - vv]).astype(np.float32)


@pytest.mark.parametrize("name", ["quarter", "half", "shift", "out_of_frame"])
def test_dense_oracle_exact_fields_bitwise(golden_warps, name):
    # integer-valued fields are exact in fp32: the dense restatement must
    # reproduce the reference's rigid permutation / shift bit for bit
    G = golden_warps
    rot, tr, tc, _ = G[f"{name}__params"]
    shape = tuple(int(v) for v in G[f"{name}__shape"])
    phi = rigid_field(shape, rot, tr, tc)
    w = oracle.Warp(shape, oracle.DENSE, phi=phi)
    assert np.array_equal(w.apply(G[f"{name}__x"]), G[f"{name}__Dx"])
    assert np.array_equal(w.adjoint_apply(G[f"{name}__y"]), G[f"{name}__DTy"])


@pytest.mark.parametrize("name", ["rigid_a", "rigid_b", "c1_like"])
def test_dense_oracle_cross_pinned_to_rigid(golden_warps, name):
    # a rigid warp expressed as an fp32 displacement field reproduces the
    # reference rigid warp up to the fp32 rounding of the field
    G = golden_warps
    rot, tr, tc, _ = G[f"{name}__params"]
    shape = tuple(int(v) for v in G[f"{name}__shape"])
    w = oracle.Warp(shape, oracle.DENSE, phi=rigid_field(shape, rot, tr, tc))
    assert rel_l2(w.apply(G[f"{name}__x"]), G[f"{name}__Dx"]) <= 2e-6
    assert rel_l2(w.adjoint_apply(G[f"{name}__y"]), G[f"{name}__DTy"]) <= 2e-6


def test_dense_oracle_adjoint_identity(rng):
    shape = (37, 29)
    phi = (3.0 * rng.standard_normal((2,) + shape)).astype(np.float32)
    w = oracle.Warp(shape, oracle.DENSE, phi=phi)
    for _ in range(5):
        x = rng.standard_normal(shape)
        y = rng.standard_normal(shape)
        lhs, rhs = np.vdot(w.apply(x), y), np.vdot(x, w.adjoint_apply(y))
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


# ---------------------------------------------------------------- sampling
def test_oracle_sampling_matches_reference(golden_sampling):
    for n in (4, 10, 20):
        for seed in (0, 5, 42):
            rng = np.random.default_rng(seed)
            seq = [osolver.sample_gates(rng, (1.0 / n,) * n, "spdhg")[0] for _ in range(50 * n)]
            assert np.array_equal(seq, golden_sampling[f"n{n}_s{seed}"])


# ---------------------------------------------------------- solver oracle
class _Toy:
    """1x1 identity operator (the reference toy problem, test_solvers.py:62-66)."""

    domain_shape = range_shape = (1, 1)

    def apply(self, x):
        return np.array(x, dtype=np.float64, copy=True)

    adjoint_apply = apply


def _toy_cfg(theta=1.0):
    return osolver.Config("pdhg", (1.5,), 0.5, theta, (1.0,), 1, 0, (1.0,))


def test_oracle_step_toy_known_answers():
    data = [np.array([[3.5]])]
    st = osolver.State.zeros((1, 1), data)
    osolver.step(st, _toy_cfg(), 0.25, [_Toy()], data, lambda: (0,))
    assert st.x[0, 0] == 0.0 and st.y[0][0, 0] == -3.0
    assert st.z[0, 0] == -3.0 and st.zbar[0, 0] == -6.0
    osolver.step(st, _toy_cfg(), 0.25, [_Toy()], data, lambda: (0,))
    assert st.x[0, 0] == pytest.approx(2.4, rel=1e-14)
    assert st.y[0][0, 0] == pytest.approx(-93 / 35, rel=1e-14)
    assert st.zbar[0, 0] == pytest.approx(-81 / 35, rel=1e-14)
    st = osolver.State.zeros((1, 1), data)
    osolver.step(st, _toy_cfg(theta=0.5), 0.25, [_Toy()], data, lambda: (0,))
    assert st.zbar[0, 0] == -4.5


def _tiny_ops(G, threads=1):
    r, c, a, b, sp = G["geom"]
    geom = oracle.Geometry(int(r), int(c), int(a), int(b), float(sp))
    specs = [{"kind": "rigid", "rotation": m[0], "translation": (m[1], m[2])} for m in G["motion"]]
    return oracle.gate_operators(geom, specs, threads)


@pytest.mark.parametrize("mode,seed", [("pdhg", 0), ("spdhg", 5)])
def test_oracle_solver_matches_reference_trajectory(golden_tiny, mode, seed):
    G = golden_tiny
    ops = _tiny_ops(G)
    alpha = float(G["alpha"])
    cfg = osolver.Config(mode, tuple(G[f"{mode}__sigmas"]), float(G[f"{mode}__tau"]), 1.0,
                         (1.0,) * 4 if mode == "pdhg" else (0.25,) * 4, 10, seed,
                         tuple(G["gate_norms"]))
    st, objs = osolver.run(cfg, alpha, ops, list(G["data"]))
    assert rel_l2(st.x, G[f"{mode}__x"]) <= 1e-11
    assert rel_l2(np.stack(st.y), G[f"{mode}__y"]) <= 1e-11
    assert rel_l2(st.z, G[f"{mode}__z"]) <= 1e-11
    assert np.allclose(objs, G[f"{mode}__objective"], rtol=1e-11)


def test_oracle_default_config_matches_reference(golden_tiny):
    G = golden_tiny
    alpha = float(G["alpha"])
    cfg = osolver.default_config("spdhg", G["gate_norms"], alpha, 10, seed=5)
    assert np.allclose(cfg.sigmas, G["spdhg__sigmas"], rtol=1e-15)
    assert cfg.tau == pytest.approx(float(G["spdhg__tau"]), rel=1e-15)
    cfg = osolver.default_config("pdhg", G["gate_norms"], alpha, 10,
                                 stacked_norm_sq=float(G["stacked_norm_sq"]))
    assert np.allclose(cfg.sigmas, G["pdhg__sigmas"], rtol=1e-15)


def test_oracle_power_method_matches_reference(golden_tiny):
    G = golden_tiny
    ops = _tiny_ops(G)
    norms = [osolver.power_method(op, iterations=40) for op in ops]
    assert np.allclose(norms, G["gate_norms"], rtol=1e-12)
    assert osolver.stacked_norm_sq(ops, iterations=40) == pytest.approx(
        float(G["stacked_norm_sq"]), rel=1e-12)


@pytest.mark.parametrize("mode", ["pdhg", "spdhg"])
def test_oracle_c1_trajectory_matches_reference(golden_c1, mode):
    from paper_2410_10503_b200 import workloads

    G = golden_c1
    cfgw = workloads.CONFIGS["c1"]
    inp = workloads.slice_inputs(cfgw, 0)
    assert np.array_equal(inp.phantom, G["phantom"])
    geom = oracle.Geometry(*cfgw.geometry_args)
    ops = oracle.gate_operators(geom, inp.gates, threads=oracle.default_threads())
    cfg = osolver.default_config(
        mode, G["gate_norms"], cfgw.alpha, cfgw.epochs, seed=cfgw.seed,
        stacked_norm_sq=float(G["stacked_norm_sq"]) if mode == "pdhg" else None)
    st, objs = osolver.run(cfg, cfgw.alpha, ops, list(G["data"].astype(np.float64)))
    assert rel_l2(st.x, G[f"{mode}__x"]) <= 1e-10
    assert np.allclose(objs, G[f"{mode}__objective"], rtol=1e-10)
