"""GPU tier: sm_100a operators vs the reference's golden outputs and the oracle.

Bars (BASELINE.json north_star): operator outputs within relative L2 1e-5 of
the fp64 reference on identical (fp32-rounded) inputs; adjoint identity
<A x, y> = <x, A^* y> to 1e-5 with fp64 inner products.  Known-answer cases
follow test_projector.py:62-160 and test_motion.py:47-105 at fp32 tolerances
(exact where the reference is exact).
"""

import math

import numpy as np
import pytest

import oracle
from conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-5  # north_star operator parity (fp32 vs fp64 reference)


@pytest.fixture(scope="module")
def m():
    import paper_2410_10503_b200 as m

    m.build_native()
    return m


def _geom(m, g):
    r, c, a, b, sp = g
    return m.Geometry(int(r), int(c), int(a), int(b), float(sp))


GEOMS = ["fast", "rect_spacing", "tiny", "many_angles", "axis_exact", "half_spacing", "lin",
         "c1", "odd_rect"]


@pytest.mark.parametrize("name", GEOMS)
def test_ray_forward_adjoint_vs_reference(m, golden_projector, name):
    G = golden_projector
    op = m.RayTransform(_geom(m, G[f"{name}__geom"]))
    ax = op.apply(G[f"{name}__x"])
    aty = op.adjoint_apply(G[f"{name}__y"])
    assert ax.dtype == np.float64 and ax.shape == G[f"{name}__Ax"].shape
    assert rel_l2(ax, G[f"{name}__Ax"]) <= TOL
    assert rel_l2(aty, G[f"{name}__ATy"]) <= TOL


@pytest.mark.parametrize("name", GEOMS)
def test_ray_adjoint_identity(m, golden_projector, name):
    op = m.RayTransform(_geom(m, golden_projector[f"{name}__geom"]))
    assert m.adjoint_mismatch(op, pairs=5, seed=0) <= TOL


def test_axis_aligned_one_hot_is_exact(m):
    geom = m.Geometry(65, 65, 48, 95, 1.0)
    x = np.zeros((65, 65))
    x[20, 40] = 1.0
    sino = m.forward(geom, x)
    j = (40 - 32) + 47
    assert sino[0, j] == 1.0
    row = sino[0].copy()
    row[j] = 0.0
    assert np.all(row == 0.0)


def test_row_sums_match_tent_sum(m):
    geom = m.Geometry(65, 65, 48, 95, 1.0)
    x = np.zeros((65, 65))
    x[32, 32] = 1.0
    sino = m.forward(geom, x)
    centers = geom.bin_centers
    for a, th in enumerate(geom.angles):
        mm = max(abs(math.cos(th)), abs(math.sin(th)))
        expected = np.maximum(0.0, 1.0 - np.abs(centers / mm)).sum() / mm
        assert sino[a].sum() == pytest.approx(expected, rel=1e-6)
    assert sino[0].sum() == 1.0


def test_center_bin_of_ones_image(m):
    geom = m.Geometry(64, 64, 36, 95, 64.0 * math.sqrt(2.0) / 95.0)
    sino = m.forward(geom, np.ones((64, 64)))
    for a, th in enumerate(geom.angles):
        mm = max(abs(math.cos(th)), abs(math.sin(th)))
        assert sino[a, 47] == pytest.approx(64.0 / mm, rel=2e-6)


def test_quarter_turn_rotational_consistency(m):
    geom = m.Geometry(33, 33, 24, 49, 1.0)
    img = np.random.default_rng(0).random((33, 33))
    rot = m.WarpOperator(m.MotionParams("rigid", math.pi / 2.0), (33, 33)).apply(img)
    op = m.ray_transform(geom)
    s0, s1 = op.apply(img), op.apply(rot)
    n = geom.num_angles
    for a in range(n):
        exp = s0[a - n // 2] if a >= n // 2 else s0[a + n // 2][::-1]
        assert np.max(np.abs(s1[a] - exp)) <= 1e-5 * np.abs(s0).max()


def test_linearity_and_zero(m):
    geom = m.Geometry(24, 24, 12, 30, 1.2)
    r = np.random.default_rng(5)
    a, b = r.random((24, 24)), r.random((24, 24))
    left = m.forward(geom, 2.0 * a - 3.0 * b)
    right = 2.0 * m.forward(geom, a) - 3.0 * m.forward(geom, b)
    assert rel_l2(left, right) <= 1e-6
    assert np.all(m.forward(geom, np.zeros((24, 24))) == 0.0)
    with pytest.raises(ValueError):
        m.forward(geom, np.zeros((24, 23)))
    with pytest.raises(ValueError):
        m.adjoint(geom, np.zeros((11, 30)))


@pytest.mark.parametrize("batch", [2, 3, 4, 5])
@pytest.mark.parametrize("shape", [(48, 40, 30, 70, 1.0), (33, 64, 31, 80, 0.9)])
def test_batched_forward_equals_single(m, batch, shape):
    """Batches run the gate-pair kernels (items 2p, 2p+1 share one walk / one set
    of tent weights, an odd last item the single-item kernels).  A^*: every
    item's result is bitwise the single-item one (with <= 16 angle pairs the
    angle split is 1 for any launch).  A: single items walk angle A-a through the
    column-mirrored image (rows-dominant interpolation from the other side, the
    cols-dominant samples in reverse order), equal to fp32 rounding."""
    import torch

    geom = m.Geometry(*shape)
    op = m.RayTransform(geom)
    x = torch.randn(batch, geom.rows, geom.cols, device="cuda")
    yb = op.forward_batch(x)
    for i in range(batch):
        assert rel_l2(yb[i].double().cpu().numpy(), op.apply(x[i]).double().cpu().numpy()) <= 1e-6
    assert torch.equal(yb, op.forward_batch(x))
    y = torch.randn(batch, geom.num_angles, geom.num_bins, device="cuda")
    xb = op.adjoint_batch(y)
    for i in range(batch):
        assert torch.equal(xb[i], op.adjoint_apply(y[i]))


def test_forward_adjoint_deterministic(m):
    import torch

    op = m.RayTransform(m.Geometry(96, 96, 90, 137, 1.0))
    x = torch.randn(96, 96, device="cuda")
    y = torch.randn(90, 137, device="cuda")
    assert torch.equal(op.apply(x), op.apply(x))
    assert torch.equal(op.adjoint_apply(y), op.adjoint_apply(y))


# ---------------------------------------------------------------- large sizes
@pytest.mark.parametrize("n,A,B", [(256, 360, 363), (512, 720, 729), (1024, 1440, 1453)])
def test_ray_parity_vs_oracle_large(m, n, A, B):
    r = np.random.default_rng(n)
    x = r.standard_normal((n, n)).astype(np.float32).astype(np.float64)
    y = r.standard_normal((A, B)).astype(np.float32).astype(np.float64)
    geom = m.Geometry(n, n, A, B, 1.0)
    op = m.RayTransform(geom)
    orc = oracle.RayTransform(oracle.Geometry(n, n, A, B, 1.0), threads=oracle.default_threads())
    assert rel_l2(op.apply(x), orc.apply(x)) <= TOL
    assert rel_l2(op.adjoint_apply(y), orc.adjoint_apply(y)) <= TOL


@pytest.mark.parametrize("n,A,B", [(512, 720, 729), (1024, 1440, 1453)])
def test_adjoint_identity_full_size(m, n, A, B):
    import torch

    g = torch.Generator(device="cuda").manual_seed(3)
    op = m.RayTransform(m.Geometry(n, n, A, B, 1.0))
    x = torch.randn(n, n, device="cuda", generator=g)
    y = torch.randn(A, B, device="cuda", generator=g)
    lhs = float((op.apply(x).double() * y.double()).sum())
    rhs = float((x.double() * op.adjoint_apply(y).double()).sum())
    assert abs(lhs - rhs) <= TOL * max(abs(lhs), abs(rhs))


# ---------------------------------------------------------------------- warps
WARPS = ["rigid_a", "rigid_b", "dilatation", "quarter", "half", "shift", "out_of_frame",
         "c1_like", "shrink"]
EXACT = {"quarter", "half", "shift", "out_of_frame"}


def _warp(m, G, name):
    rot, tr, tc, sc = G[f"{name}__params"]
    shape = tuple(int(v) for v in G[f"{name}__shape"])
    kind = "rigid" if int(G[f"{name}__kind"]) == 0 else "dilatation"
    if kind == "rigid":
        p = m.MotionParams("rigid", float(rot), (float(tr), float(tc)))
    else:
        p = m.MotionParams("dilatation", scale=float(sc))
    return m.WarpOperator(p, shape)


@pytest.mark.parametrize("name", WARPS)
def test_warp_vs_reference(m, golden_warps, name):
    G = golden_warps
    w = _warp(m, G, name)
    dx, dty = w.apply(G[f"{name}__x"]), w.adjoint_apply(G[f"{name}__y"])
    if name in EXACT:
        assert np.array_equal(dx, G[f"{name}__Dx"])
        assert np.array_equal(dty, G[f"{name}__DTy"])
    else:
        assert rel_l2(dx, G[f"{name}__Dx"]) <= TOL
        assert rel_l2(dty, G[f"{name}__DTy"]) <= TOL
    assert m.adjoint_mismatch(w, pairs=5, seed=2) <= TOL


def test_identity_warp_copies(m, rng):
    w = m.WarpOperator(m.MotionParams.identity(), (12, 12))
    x = rng.random((12, 12))
    out = w.apply(x)
    assert np.array_equal(out, x)
    out[3, 3] = 99.0
    assert x[3, 3] != 99.0


@pytest.mark.parametrize("shape,peak", [((37, 29), 3.0), ((128, 128), 6.0), ((256, 256), 4.0)])
def test_dense_warp_vs_oracle(m, shape, peak):
    from paper_2410_10503_b200 import workloads

    r = np.random.default_rng(shape[0])
    if shape[0] == shape[1]:
        phi = workloads.bump_field(shape[0], peak, 1, 0)
    else:
        phi = (peak * r.standard_normal((2,) + shape)).astype(np.float32)
    w = m.DenseWarpOperator(phi)
    o = oracle.Warp(shape, oracle.DENSE, phi=phi)
    x = r.standard_normal(shape).astype(np.float32).astype(np.float64)
    y = r.standard_normal(shape).astype(np.float32).astype(np.float64)
    assert rel_l2(w.apply(x), o.apply(x)) <= TOL
    assert rel_l2(w.adjoint_apply(y), o.adjoint_apply(y)) <= TOL
    assert m.adjoint_mismatch(w, pairs=3) <= TOL
    assert 0 < w.nnz <= 4 * shape[0] * shape[1]


def test_gated_operator_is_warp_then_project(m):
    from paper_2410_10503_b200 import workloads

    geom = m.Geometry(128, 128, 90, 183, 1.0)
    phi = workloads.bump_field(128, 5.0, 2, 1)
    dense = m.DenseWarpOperator(phi)
    rigid = m.WarpOperator(m.MotionParams("rigid", 0.05, (1.2, -0.7)), (128, 128))
    x = np.random.default_rng(1).random((128, 128))
    base = m.ray_transform(geom)
    for w in (dense, rigid):
        op = m.compose(base, w)
        assert isinstance(op, m.GatedOperator)
        assert rel_l2(op.apply(x), base.apply(w.apply(x))) <= 1e-6
        y = np.random.default_rng(2).standard_normal(geom.sino_shape)
        assert rel_l2(op.adjoint_apply(y), w.adjoint_apply(base.adjoint_apply(y))) <= 1e-6
        assert m.adjoint_mismatch(op, pairs=3) <= TOL


def test_power_method_matches_reference_norms(m, golden_tiny, golden_c1):
    from paper_2410_10503_b200 import workloads

    G = golden_tiny
    r, c, a, b, sp = G["geom"]
    geom = m.Geometry(int(r), int(c), int(a), int(b), float(sp))
    motion = [m.MotionParams("rigid", float(p[0]), (float(p[1]), float(p[2]))) for p in G["motion"]]
    info = m.estimate_norms(geom, motion, iterations=40)
    assert np.allclose(info["gate_norms"], G["gate_norms"], rtol=1e-4)
    assert info["stacked_norm_sq"] == pytest.approx(float(G["stacked_norm_sq"]), rel=1e-4)
    C = golden_c1
    cfg = workloads.CONFIGS["c1"]
    inp = workloads.slice_inputs(cfg, 0)
    info = m.estimate_norms(m.Geometry(*cfg.geometry_args), inp.gates, iterations=100)
    assert np.allclose(info["gate_norms"], C["gate_norms"], rtol=1e-4)
    assert info["base_norm_sq"] == pytest.approx(float(C["base_norm_sq"]), rel=1e-4)


@pytest.mark.parametrize("n,peak", [(512, 6.0), (1024, 8.0)])
def test_dense_gated_parity_full_size(m, n, peak):
    """A_i and A_i^* with a BASELINE dense field at C3 / C4 size vs the fp64 oracle."""
    from paper_2410_10503_b200 import workloads

    A, B = {512: (720, 729), 1024: (1440, 1453)}[n]
    phi = workloads.bump_field(n, peak, 0, 1)
    geom = m.Geometry(n, n, A, B, 1.0)
    op = m.compose(m.ray_transform(geom), m.DenseWarpOperator(phi))
    orc = oracle.Composed(oracle.RayTransform(oracle.Geometry(n, n, A, B, 1.0),
                                              threads=oracle.default_threads()),
                          oracle.Warp((n, n), oracle.DENSE, phi=phi))
    r = np.random.default_rng(n + 1)
    x = workloads.ellipse_phantom(n, 12, 5).astype(np.float64)
    y = r.standard_normal((A, B)).astype(np.float32).astype(np.float64)
    assert rel_l2(op.apply(x), orc.apply(x)) <= TOL
    assert rel_l2(op.adjoint_apply(y), orc.adjoint_apply(y)) <= TOL


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("g", [
    (1, 1, 1, 1, 1.0),          # single pixel, single ray
    (7, 3, 5, 4, 0.8),          # ragged, few bins
    (50, 20, 13, 9, 2.5),       # detector narrower than the image (rays miss corners)
    (32, 32, 7, 200, 0.3),      # fine bins: wide adjoint footprint (K = 3)
    (19, 41, 64, 61, 1.0),      # non-square, 45-degree tie handled by the host flags
    (1, 40, 6, 45, 1.0),        # one-row image
    (40, 1, 6, 45, 1.0),        # one-column image (centre column = its own mirror)
    (33, 33, 2, 47, 1.0),       # two angles: 0 and pi/2 only, no mirror pairs
    (33, 35, 3, 47, 1.0),       # odd angle count: one mirror pair + angle 0
    (64, 64, 200, 91, 1.0),     # the reference's default angle count (45 deg is cols-dominant)
])
def test_edge_geometries_vs_oracle(m, g):
    """Single items (mirror-angle kernels) and a batch of 3 (one gate pair + an odd
    last item) against the fp64 oracle on every edge geometry."""
    import torch

    r = np.random.default_rng(sum(int(v) for v in g[:4]))
    geom = m.Geometry(*g)
    op = m.RayTransform(geom)
    orc = oracle.RayTransform(oracle.Geometry(*g))
    x = r.standard_normal(geom.image_shape).astype(np.float32).astype(np.float64)
    y = r.standard_normal(geom.sino_shape).astype(np.float32).astype(np.float64)
    assert rel_l2(op.apply(x), orc.apply(x)) <= TOL
    assert rel_l2(op.adjoint_apply(y), orc.adjoint_apply(y)) <= TOL
    xb = r.standard_normal((3,) + tuple(geom.image_shape)).astype(np.float32)
    yb = r.standard_normal((3,) + tuple(geom.sino_shape)).astype(np.float32)
    fb = op.forward_batch(torch.from_numpy(xb).cuda()).double().cpu().numpy()
    ab = op.adjoint_batch(torch.from_numpy(yb).cuda()).double().cpu().numpy()
    for i in range(3):
        assert rel_l2(fb[i], orc.apply(xb[i].astype(np.float64))) <= TOL, i
        assert rel_l2(ab[i], orc.adjoint_apply(yb[i].astype(np.float64))) <= TOL, i


@pytest.mark.parametrize("g", [(32, 32, 8, 400, 0.1), (48, 40, 30, 301, 0.2),
                               (33, 33, 12, 150, 0.24), (64, 64, 9, 2000, 0.05)])
def test_fine_detector_spacing_vs_oracle(m, g):
    """Any positive detector spacing (projector.py:63-68): below 1/4 pixel the A^*
    footprint exceeds the unrolled kernels (K > 3) and the runtime-footprint kernel
    runs; single items, a batch of 3 (gate pair + odd item) and the adjoint
    identity against the fp64 oracle."""
    import torch

    r = np.random.default_rng(int(g[3]))
    geom = m.Geometry(*g)
    op = m.RayTransform(geom)
    orc = oracle.RayTransform(oracle.Geometry(*g))
    x = r.standard_normal(geom.image_shape).astype(np.float32).astype(np.float64)
    y = r.standard_normal(geom.sino_shape).astype(np.float32).astype(np.float64)
    assert rel_l2(op.apply(x), orc.apply(x)) <= TOL
    assert rel_l2(op.adjoint_apply(y), orc.adjoint_apply(y)) <= TOL
    lhs, rhs = float(np.vdot(op.apply(x), y)), float(np.vdot(x, op.adjoint_apply(y)))
    assert abs(lhs - rhs) <= 1e-5 * max(abs(lhs), abs(rhs))
    yb = r.standard_normal((3,) + tuple(geom.sino_shape)).astype(np.float32)
    ab = op.adjoint_batch(torch.from_numpy(yb).cuda()).double().cpu().numpy()
    for i in range(3):
        assert rel_l2(ab[i], orc.adjoint_apply(yb[i].astype(np.float64))) <= TOL, i


def test_dense_zero_field_is_identity_and_out_of_frame(m, rng):
    x = rng.standard_normal((40, 33)).astype(np.float32).astype(np.float64)
    w0 = m.DenseWarpOperator(np.zeros((2, 40, 33), dtype=np.float32))
    assert np.array_equal(w0.apply(x), x)
    assert np.array_equal(w0.adjoint_apply(x), x)
    far = np.full((2, 40, 33), 500.0, dtype=np.float32)
    wf = m.DenseWarpOperator(far)
    assert np.all(wf.apply(x) == 0.0) and np.all(wf.adjoint_apply(x) == 0.0)
    with pytest.raises(ValueError):
        m.DenseWarpOperator(np.full((2, 4, 4), np.nan, dtype=np.float32))
    with pytest.raises(ValueError):
        m.DenseWarpOperator(np.zeros((3, 4, 4)))


def test_helper_maps_on_device(m, rng):
    """IdentityMap, DiagonalMap, StackedMap of gated operators (linops.py:76-169)."""
    geom = m.Geometry(24, 24, 16, 32, 1.1)
    ops = m.gate_operators(geom, [m.MotionParams.identity(),
                                  m.MotionParams(kind="rigid", rotation=0.2, translation=(1.0, -0.5)),
                                  m.MotionParams(kind="dilatation", scale=1.05)])
    x = rng.standard_normal(geom.image_shape).astype(np.float32).astype(np.float64)
    ident = m.IdentityMap(geom.image_shape)
    assert np.array_equal(ident.apply(x), x)
    d = rng.uniform(0.5, 2.0, geom.image_shape).astype(np.float32).astype(np.float64)
    assert np.allclose(m.DiagonalMap(d).apply(x), x * d, rtol=1e-6)
    st = m.StackedMap(ops)
    y = st.apply(x)
    assert y.shape == (3,) + tuple(geom.sino_shape)
    for k, op in enumerate(ops):
        assert np.array_equal(y[k], op.apply(x))
    yy = rng.standard_normal(st.range_shape).astype(np.float32).astype(np.float64)
    want = sum(op.adjoint_apply(yy[k]).astype(np.float64) for k, op in enumerate(ops))
    assert rel_l2(st.adjoint_apply(yy), want) <= 1e-6
    assert m.adjoint_mismatch(st, pairs=3) <= TOL
    # ||stack||^2 == lambda_max(sum_i A_i^* A_i)  (linops.py:275-289)
    nsq = m.power_method(st, iterations=60) ** 2
    assert nsq == pytest.approx(m.stacked_norm_sq(ops, iterations=60), rel=1e-4)


def test_gated_forward_many_matches_single(m, rng):
    """mct_gated_forward_many (all gates of a slice in one pass, used by the
    per-epoch objective) vs one gated forward per gate."""
    import torch

    from paper_2410_10503_b200 import _lib
    from paper_2410_10503_b200.engine import Engine

    geom = m.Geometry(40, 36, 30, 57, 1.0)
    gates = [m.MotionParams.identity(), m.MotionParams(kind="rigid", rotation=0.3),
             rng.uniform(-2, 2, (2, 40, 36)).astype(np.float32)]
    ops = m.gate_operators(geom, gates)
    data = [np.zeros(geom.sino_shape) for _ in ops]
    eng = Engine([ops], [data])
    x = torch.from_numpy(rng.standard_normal(geom.image_shape).astype(np.float32)).cuda()
    out = torch.empty((3,) + tuple(geom.sino_shape), device="cuda")
    _lib.check(_lib.load().mct_gated_forward_many(eng.family.handle, 0, _lib.ptr(eng.all_gates),
                                                  3, _lib.ptr(x), _lib.ptr(out), _lib.ptr(eng.ws),
                                                  _lib.stream_handle()))
    for k, op in enumerate(ops):
        ref = op.apply_device(x)
        assert rel_l2(out[k].double().cpu().numpy(), ref.double().cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("g", [(1, 1, 1, 1, 1.0), (7, 3, 5, 4, 0.8), (40, 1, 6, 45, 1.0),
                               (32, 32, 7, 200, 0.3), (65, 66, 48, 95, 1.0),
                               (24, 24, 6, 400, 0.08)])
def test_no_writes_outside_buffers(m, g):
    """Out-of-bounds write check without a sanitizer: workspace and outputs carry
    canary tails (0xAB) that every launch must leave intact, and a second
    forward / adjoint on the reused workspace reproduces the first bit for bit
    (the zero pads survived)."""
    import torch

    from paper_2410_10503_b200 import _lib

    L = _lib.load()
    geom = m.Geometry(*g)
    op = m.RayTransform(geom)
    plan = op.plan().handle
    batch, tail = 2, 1 << 16
    need = int(L.mct_ray_workspace_bytes(plan, batch))
    ws = torch.full((need + tail,), 0xAB, dtype=torch.uint8, device="cuda")
    ws[:need].zero_()
    A, B = geom.sino_shape
    R, C = geom.image_shape
    x = torch.randn(batch * R * C + tail // 4, device="cuda")
    y = torch.full((batch * A * B + tail // 4,), 7.0, device="cuda")
    img = torch.full((batch * R * C + tail // 4,), 7.0, device="cuda")
    st = _lib.stream_handle()
    outs = []
    for _ in range(2):
        _lib.check(L.mct_ray_forward(plan, _lib.ptr(x), _lib.ptr(y), batch, _lib.ptr(ws), st))
        _lib.check(L.mct_ray_adjoint(plan, _lib.ptr(y), _lib.ptr(img), batch, _lib.ptr(ws), st))
        outs.append((y.clone(), img.clone()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert bool((ws[need:] == 0xAB).all()), "workspace tail overwritten"
    assert bool((y[batch * A * B:] == 7.0).all()), "sinogram tail overwritten"
    assert bool((img[batch * R * C:] == 7.0).all()), "image tail overwritten"
    assert bool(torch.isfinite(img[:batch * R * C]).all())


def test_power_method_contract_on_device(m):
    """The reference's power-method / stacked-norm contract (test_linops.py:115-161)
    on the device maps."""
    assert m.power_method(m.IdentityMap((9,)), iterations=3, seed=0) == 1.0
    op = m.DiagonalMap(np.linspace(0.1, 2.0, 11))
    a = m.power_method(op, iterations=40, seed=5)
    assert a == m.power_method(op, iterations=40, seed=5)
    assert abs(a - 2.0) <= 1e-2
    with pytest.warns(RuntimeWarning):
        assert m.power_method(m.DiagonalMap(np.zeros(4)), iterations=10, seed=0) == 0.0
    n = 7
    blocks = [m.IdentityMap((5,)) for _ in range(n)]
    assert abs(m.stacked_norm_sq(blocks, iterations=50, seed=0) - n) <= 1e-6


def test_mass_conservation_within_sampling_ripple(m):
    """test_projector.py:107-116: integrating each angle's projection over the
    detector recovers the image mass up to the interpolation ripple."""
    geom = m.Geometry.fast()
    x = m.make_phantom("nested_shells", 64, 64)
    sino = m.forward(geom, x)
    mass = x.sum()
    per_angle = sino.sum(axis=1) * geom.detector_spacing
    assert np.max(np.abs(per_angle - mass)) / mass <= 2.5e-3


def test_terminal_warp_norms_stay_near_isometric(m):
    """test_motion.py:108-122: the norm window the step sizes rely on, at the
    largest motion state of each preset family (device power iteration)."""
    rigid = m.MotionParams(kind="rigid", rotation=m.motion.RIGID_TERMINAL_ROTATION,
                           translation=m.motion.RIGID_TERMINAL_TRANSLATION)
    dila = m.MotionParams(kind="dilatation", scale=1.0 + m.motion.DILATATION_TERMINAL_GROWTH)
    for params in (rigid, dila):
        norm = m.power_method(m.WarpOperator(params, (64, 64)), iterations=150, seed=0)
        assert 0.8 <= norm <= 1.2, params.kind


@pytest.mark.parametrize("n,A,B,batch", [(512, 720, 729, 3), (512, 720, 729, 5),
                                         (1024, 1440, 1453, 2)])
def test_large_batches_match_single_items(m, n, A, B, batch):
    """C3-size batches with an odd item (gate pairs + the odd item on the side stream,
    the A^* angle split chosen over both launches, up to the plan's >= 4 slots) and a
    C4-size gate pair agree with single-item calls (fp32 rounding, not bits: the
    single item walks mirror angles and may split A^* differently)."""
    import torch

    geom = m.Geometry(n, n, A, B, 1.0)
    op = m.RayTransform(geom)
    x = torch.randn(batch, n, n, device="cuda")
    y = torch.randn(batch, A, B, device="cuda")
    fb, ab = op.forward_batch(x), op.adjoint_batch(y)
    for i in range(batch):
        assert rel_l2(fb[i].double().cpu().numpy(), op.apply(x[i]).double().cpu().numpy()) <= 1e-6
        assert rel_l2(ab[i].double().cpu().numpy(),
                      op.adjoint_apply(y[i]).double().cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("batch", [16, 17, 20, 33])
@pytest.mark.parametrize("shape", [(48, 40, 30, 70, 1.0), (33, 64, 31, 80, 0.9),
                                   (64, 64, 200, 91, 1.0)])
def test_many_item_batches_match_single_items_and_oracle(m, batch, shape):
    """PDHG-sized launches (16-33 items: gate pairs, plus the mirror kernels for an
    odd last item on the side stream): every item agrees with its single-item call
    and with the fp64 oracle, and the launch is deterministic."""
    import torch

    geom = m.Geometry(*shape)
    op = m.RayTransform(geom)
    orc = oracle.RayTransform(oracle.Geometry(*shape))
    x = torch.randn(batch, geom.rows, geom.cols, device="cuda")
    yb = op.forward_batch(x)
    y = torch.randn(batch, geom.num_angles, geom.num_bins, device="cuda")
    xb = op.adjoint_batch(y)
    for i in range(batch):
        xi = x[i].double().cpu().numpy()
        yi = y[i].double().cpu().numpy()
        assert rel_l2(yb[i].double().cpu().numpy(), op.apply(x[i]).double().cpu().numpy()) <= 1e-6
        assert rel_l2(yb[i].double().cpu().numpy(), orc.apply(xi)) <= TOL, i
        # A^*: bitwise whenever the angle splits agree, else fp32 rounding
        assert rel_l2(xb[i].double().cpu().numpy(),
                      op.adjoint_apply(y[i]).double().cpu().numpy()) <= 1e-6
        assert rel_l2(xb[i].double().cpu().numpy(), orc.adjoint_apply(yi)) <= TOL, i
    assert torch.equal(yb, op.forward_batch(x)) and torch.equal(xb, op.adjoint_batch(y))
