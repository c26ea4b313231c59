"""CPU tier: host-side logic mirrored from the reference (no device compute).

Mirrors the reference's own unit tests for the API surface: Geometry
(test_projector.py:21-56), MotionParams / motion_sequence (test_motion.py:22-45,
:125-164), SolverConfig / default_config / sample_gates (test_solvers.py:122-281),
Problem validation (:82-97), ConvergenceRecord CSV round trip, gaussian_field
recipe (test_simulate.py:70-106); plus the seeded workload generators and the
"no CPU fallback" rule.
"""

import math

import numpy as np
import pytest

from paper_2410_10503_b200 import (RHO, ConvergenceRecord, Geometry, MotionParams, Problem,
                                   SolverConfig, default_config, draw_sequence, motion_sequence,
                                   sample_gates, workloads)
from paper_2410_10503_b200.motion import RIGID_TERMINAL_ROTATION


def test_geometry_validation_and_presets():
    with pytest.raises(ValueError):
        Geometry(0, 10, 4, 8, 1.0)
    with pytest.raises(ValueError):
        Geometry(10, 10, 0, 8, 1.0)
    with pytest.raises(ValueError):
        Geometry(10, 10, 4, 8, -1.0)
    d = Geometry.default()
    assert (d.rows, d.cols, d.num_angles, d.num_bins) == (100, 100, 200, 200)
    g = Geometry(16, 16, 8, 11, 0.5)
    assert g.angles[0] == 0.0 and np.all(g.angles < math.pi)
    assert np.allclose(g.bin_centers, -g.bin_centers[::-1])
    cos, sin, rdom = Geometry(1, 1, 200, 3, 1.0).angle_tables()
    # A=200: the 45 degree angle is cols-dominant; A=180: rows
    assert rdom[50] == 0
    assert Geometry(1, 1, 180, 3, 1.0).angle_tables()[2][45] == 1


def test_motion_params():
    with pytest.raises(ValueError):
        MotionParams(kind="affine")
    with pytest.raises(ValueError):
        MotionParams(kind="rigid", scale=1.1)
    with pytest.raises(ValueError):
        MotionParams(kind="dilatation", rotation=0.1, scale=1.1)
    with pytest.raises(ValueError):
        MotionParams(kind="rigid", rotation=math.nan)
    p = MotionParams(kind="rigid", rotation=0.2, translation=(1.5, -2.0))
    assert MotionParams.from_dict(p.to_dict()) == p
    assert MotionParams.identity().is_identity() and not p.is_identity()
    seq = motion_sequence("rigid", 5)
    assert seq[0].is_identity()
    assert seq[-1].rotation == pytest.approx(RIGID_TERMINAL_ROTATION)
    with pytest.raises(ValueError):
        motion_sequence("spline", 4)


def _good(**kw):
    base = dict(mode="spdhg", sigmas=(0.1, 0.1), tau=0.1, theta=1.0, probs=(0.5, 0.5), epochs=1,
                seed=0, gate_norms=(1.0, 1.0))
    base.update(kw)
    return base


@pytest.mark.parametrize("bad", [
    dict(mode="newton"), dict(sigmas=(0.1,)), dict(sigmas=(0.0, 0.1)), dict(tau=-1.0),
    dict(theta=0.0), dict(theta=1.5), dict(probs=(0.0, 1.0)), dict(epochs=-1),
    dict(gate_norms=(0.0, 1.0)), dict(mode="pdhg"), dict(sigmas=(10.0, 10.0)),
])
def test_solver_config_rejects(bad):
    with pytest.raises(ValueError):
        SolverConfig(**_good(**bad))


def test_default_config_pinned_values():
    cfg = default_config("pdhg", (1.0,), alpha=0.25, epochs=5, seed=7)
    assert cfg.sigmas == (0.99,) and cfg.tau == pytest.approx(0.99, rel=1e-15)
    cfg = default_config("spdhg", (1.0,) * 20, alpha=0.25, epochs=1)
    assert cfg.probs == (1.0 / 20,) * 20
    for s, p, v in zip(cfg.sigmas, cfg.probs, cfg.gate_norms):
        assert s * cfg.tau * v * v == pytest.approx(RHO ** 2 * p, rel=1e-12)
    cfg = default_config("pdhg", (1.0, 2.0), alpha=0.5, epochs=1, stacked_norm_sq=4.2)
    assert cfg.sigmas[0] * cfg.tau * 4.2 == pytest.approx(RHO ** 2, rel=1e-12)
    assert cfg.iterations_per_epoch == 1
    assert default_config("spdhg", (1.0,) * 6, 0.25, 1).iterations_per_epoch == 6
    with pytest.raises(ValueError):
        default_config("pdhg", (), alpha=0.25, epochs=1)
    with pytest.raises(ValueError):
        default_config("newton", (1.0,), alpha=0.25, epochs=1)


def test_sample_gates_and_presampled_sequence(golden_sampling):
    rng = np.random.default_rng(0)
    before = rng.bit_generator.state
    assert sample_gates(rng, (1.0, 1.0, 1.0), "pdhg") == (0, 1, 2)
    assert rng.bit_generator.state == before
    with pytest.raises(ValueError):
        sample_gates(rng, (1.0,), "smooth")
    for n in (4, 10, 20):
        for seed in (0, 5, 42):
            cfg = default_config("spdhg", (1.0,) * n, 0.25, 50, seed=seed)
            assert np.array_equal(draw_sequence(cfg), golden_sampling[f"n{n}_s{seed}"])


class _Shape:
    def __init__(self, dom, rng):
        self.domain_shape, self.range_shape = dom, rng


def test_problem_validation():
    op = _Shape((2, 2), (3, 3))
    d = np.zeros((3, 3))
    with pytest.raises(ValueError, match="alpha"):
        Problem.from_parts(0.0, [op], [d])
    with pytest.raises(ValueError, match="gate"):
        Problem.from_parts(1.0, [], [])
    with pytest.raises(ValueError, match="data block"):
        Problem.from_parts(1.0, [op], [d, d])
    with pytest.raises(ValueError, match="data shape"):
        Problem.from_parts(1.0, [op], [np.zeros((2, 2))])
    with pytest.raises(ValueError, match="domain mismatch"):
        Problem.from_parts(1.0, [op, _Shape((3, 3), (3, 3))], [d, d])
    p = Problem.from_parts(0.5, [op, op], [d, d + 1.0])
    assert p.num_gates == 2 and p.image_shape == (2, 2)
    assert p.data_objective() == pytest.approx(9.0 / 2)


def test_convergence_record_csv_roundtrip(tmp_path):
    rec = ConvergenceRecord()
    rec.append(1, 0.5, 2.0, math.nan, 4, 4)
    rec.append(2, 0.25, 1.0 / 3.0, 0.1, 8, 8)
    with pytest.raises(ValueError):
        rec.append(2, 0.1, 0.1, 0.1, 12, 12)
    path = tmp_path / "rec.csv"
    rec.write_csv(path)
    back = ConvergenceRecord.read_csv(path)
    assert back.objective == rec.objective and back.fwd_calls == rec.fwd_calls


def test_gaussian_field_recipe(golden_sampling):
    assert np.array_equal(workloads.gaussian_field((5, 7), 1234, 3),
                          golden_sampling["field_5x7_1234_3"])
    assert np.array_equal(workloads.gaussian_field((180, 183), 0, 2),
                          golden_sampling["field_c1_0_2"])
    with pytest.raises(ValueError):
        workloads.gaussian_field((4, 4), 0, -1)


def test_workload_generators_deterministic():
    a = workloads.ellipse_phantom(64, 8, 3)
    b = workloads.ellipse_phantom(64, 8, 3)
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert a.min() >= 0.0 and a.max() <= 1.0 and a.max() > 0.1
    g = workloads.rigid_gates(4, 0)
    assert all(abs(x["rotation"]) <= math.radians(5) for x in g)
    assert all(abs(t) <= 3 for x in g for t in x["translation"])
    phi = workloads.bump_field(96, 6.0, 0, 3)
    mag = np.sqrt(phi[0] ** 2 + phi[1] ** 2).max()
    assert phi.shape == (2, 96, 96) and 3.0 - 1e-4 <= mag <= 6.0 + 1e-4
    assert not np.array_equal(phi, workloads.bump_field(96, 6.0, 0, 4))
    c5 = workloads.CONFIGS["c5"]
    assert c5.batch == 64 and c5.num_gates == 10
    assert workloads.CONFIGS["c3"].samples == 720 * 729 * 512


def test_no_cpu_fallback():
    """Without a CUDA device every compute entry point raises (no silent CPU path)."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2410_10503_b200 import RayTransform

    with pytest.raises(RuntimeError, match="CUDA"):
        RayTransform(Geometry(8, 8, 4, 12, 1.0)).apply(np.zeros((8, 8)))


def test_helper_maps_validation_and_no_fallback():
    """IdentityMap / DiagonalMap / StackedMap (linops.py:76-169): shape checks on
    the host, compute only on the device."""
    torch = pytest.importorskip("torch")
    from paper_2410_10503_b200 import DiagonalMap, IdentityMap, StackedMap

    a, b = IdentityMap((3, 4)), IdentityMap((3, 5))
    with pytest.raises(ValueError):
        StackedMap([])
    with pytest.raises(ValueError):
        StackedMap([a, b])
    with pytest.raises(ValueError):
        StackedMap([a, DiagonalMap(np.ones((4, 3)))])
    s = StackedMap([a, DiagonalMap(np.full((3, 4), 2.0))])
    assert s.domain_shape == (3, 4) and s.range_shape == (2, 3, 4)
    with pytest.raises(ValueError):
        s.apply(np.zeros((4, 3)))
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError, match="CUDA"):
            s.apply(np.zeros((3, 4)))


def test_chunk_plan_of_the_pair_ring():
    """K1-K3 chunks of a launch through a workspace whose pair ring holds `chunk_items`
    items (engine.chunk_plan): whole gate pairs, the unpaired tail (an odd
    or a half last item) with the last chunk, (0, 0) when everything fits."""
    from paper_2410_10503_b200.engine import chunk_plan

    assert chunk_plan(1, 0, 1) == [(0, 0)]
    assert chunk_plan(20, 0, 20) == [(0, 0)]          # C3: every pair has its region
    assert chunk_plan(7, 0, 7) == [(0, 0)]
    assert chunk_plan(40, 0, 8) == [(0, 8), (8, 8), (16, 8), (24, 8), (32, 0)]  # C4
    assert chunk_plan(64, 0, 32) == [(0, 32), (32, 0)]                            # C5
    assert chunk_plan(7, 0, 2) == [(0, 2), (2, 2), (4, 0)]     # the odd item rides along
    assert chunk_plan(5, 1, 2) == [(0, 2), (2, 0)]             # 2 pairs + a half item
    assert chunk_plan(6, 2, 2) == [(0, 2), (2, 0)]             # 2 pairs + odd + half
    assert chunk_plan(3, 1, 2) == [(0, 0)]
    for n, part, c in [(40, 0, 8), (11, 0, 4), (9, 1, 2), (64, 0, 32)]:
        plan = chunk_plan(n, part, c)
        paired = (n - 1 if part else n) & ~1
        covered = []
        for f, cnt in plan:
            assert f % 2 == 0 and (cnt == 0 or cnt % 2 == 0) and cnt <= c
            end = f + cnt if cnt else n
            covered += list(range(f, end))
            assert min(end, paired) - f <= c
        assert covered == list(range(n))
    with pytest.raises(ValueError):
        chunk_plan(9, 0, 3)
