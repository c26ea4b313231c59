"""GPU tier: the workspace's ring of gate-pair regions.

A workspace holds at most `ring` pair regions; launches with more gate pairs run
K1 -> K2 -> K3 chunk by chunk through them (mct_items.first_item / item_count) and K4
once over every item's A^* image.  Chunking changes no arithmetic: iterates are
bitwise equal to the unchunked launches, for PDHG (gate pairs + an odd / half last
item), batched SPDHG slices, the standalone batched A / A^*, and inside the captured
epoch graph.  Reference path: solvers.step (solvers.py:316-366).
"""

import ctypes

import numpy as np
import pytest

import oracle
from oracle import solver as osolver
from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_2410_10503_b200 as m

    m.build_native()
    return m


def fresh_problem(m, cfgw, slice_index, ring, data=None):
    """A problem on a ray plan of its own (so its ring can be set before any workspace
    of that plan exists)."""
    from paper_2410_10503_b200 import projector, workloads

    projector.ray_transform.cache_clear()
    inp = workloads.slice_inputs(cfgw, slice_index)
    geom = m.Geometry(*cfgw.geometry_args)
    ops = m.gate_operators(geom, inp.gates, True)
    if ring is not None:
        ops[0].outer.plan().set_ring_pairs(ring)
    if data is None:
        data = m.simulate.simulate_data(ops, inp.phantom, inp.seed)
    return m.Problem.from_parts(cfgw.alpha, ops, data), inp


@pytest.mark.parametrize("gates,graph", [(7, False), (7, True), (8, True), (5, False), (12, True)])
def test_chunked_pdhg_bitwise_equals_unchunked(m, gates, graph):
    from paper_2410_10503_b200 import workloads
    from paper_2410_10503_b200.engine import Engine

    cfgw = workloads.WorkloadConfig("ring", 48, 40, 71, gates, "dense", 5, 1e-2, 3, peak=3.0)
    base, inp = fresh_problem(m, cfgw, 0, None)
    norms = [m.power_method(op, iterations=20) for op in base.operators]
    cfg = m.default_config("pdhg", norms, cfgw.alpha, cfgw.epochs,
                           stacked_norm_sq=float(sum(v * v for v in norms)))
    x_ref, _ = m.run(cfg, base, graph=graph, diagnostics=False)
    eng_ref = base._engine(False)
    assert eng_ref.chunks(gates) == [(0, 0)]
    y_ref = eng_ref.y.cpu().numpy()
    # the fp64 oracle pins the unchunked run
    ogeom = oracle.Geometry(*cfgw.geometry_args)
    ocfg = osolver.default_config("pdhg", norms, cfgw.alpha, cfgw.epochs,
                                  stacked_norm_sq=float(sum(v * v for v in norms)))
    st, _ = osolver.run(ocfg, cfgw.alpha, oracle.gate_operators(ogeom, inp.gates),
                        list(base.data), diagnostics=False)
    assert np.linalg.norm(st.x) > 0 and rel_l2(x_ref, st.x) <= 1e-3
    for ring in (1, 2):
        prob, _ = fresh_problem(m, cfgw, 0, ring, data=list(base.data))
        x, _ = m.run(cfg, prob, graph=graph, diagnostics=False)
        eng = prob._engine(False)
        nchunks = len(eng.chunks(gates))
        assert nchunks == -(-(gates // 2) // ring)
        assert nchunks == 1 or eng.ws.numel() < eng_ref.ws.numel()
        assert np.array_equal(x, x_ref), ring
        assert np.array_equal(eng.y.cpu().numpy(), y_ref), ring
        # the pads of the ring survived: a second run on the same engine repeats it
        x2, _ = m.run(cfg, prob, graph=graph, diagnostics=False)
        assert np.array_equal(x2, x_ref), ring


def test_chunked_batch_spdhg_equals_unchunked(m):
    """11 slices of one gate per iteration = 5 slice pairs + an odd slice through a
    2-pair ring (3 chunks, the odd slice with the last)."""
    from paper_2410_10503_b200 import workloads

    cfgw = workloads.WorkloadConfig("ring_b", 40, 36, 61, 3, "dense", 4, 1e-2, 2, peak=2.0)
    S = 11
    base = [fresh_problem(m, cfgw, s, None)[0] for s in range(S)]
    norms = [1.1 * m.power_method(op, iterations=20) for op in base[0].operators]
    cfgs = [m.default_config("spdhg", norms, cfgw.alpha, cfgw.epochs, seed=3 + s)
            for s in range(S)]
    ref = m.run_batch(cfgs, base)
    chunked = []
    from paper_2410_10503_b200 import projector

    projector.ray_transform.cache_clear()
    geom = m.Geometry(*cfgw.geometry_args)
    m.ray_transform(geom).plan().set_ring_pairs(2)
    for s in range(S):
        inp = workloads.slice_inputs(cfgw, s)
        chunked.append(m.Problem.from_parts(cfgw.alpha, m.gate_operators(geom, inp.gates, True),
                                            list(base[s].data)))
    out = m.run_batch(cfgs, chunked)
    for s in range(S):
        assert np.array_equal(out[s][0], ref[s][0]), s
    assert np.linalg.norm(ref[0][0]) > 0


def test_chunked_standalone_batch_operators(m):
    """mct_ray_forward / mct_ray_adjoint on a 9-item batch through a 1- and a 3-pair
    ring (the chunk loop lives inside the call) equal the unchunked batch."""
    import torch

    from paper_2410_10503_b200 import projector

    geom = m.Geometry(40, 56, 61, 75, 1.0)
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal((9, 40, 56)).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.standard_normal((9, 61, 75)).astype(np.float32)).cuda()
    projector.ray_transform.cache_clear()
    op = m.ray_transform(geom)
    f_ref, a_ref = op.forward_batch(x).cpu().numpy(), op.adjoint_batch(y).cpu().numpy()
    orc = oracle.RayTransform(oracle.Geometry(40, 56, 61, 75, 1.0))
    assert rel_l2(f_ref[4], orc.apply(x[4].double().cpu().numpy())) <= 1e-5
    assert rel_l2(a_ref[8], orc.adjoint_apply(y[8].double().cpu().numpy())) <= 1e-5
    need_ref = op.plan().workspace_bytes(9)
    for ring in (1, 3):
        projector.ray_transform.cache_clear()
        op = m.ray_transform(geom)
        op.plan().set_ring_pairs(ring)
        assert op.plan().workspace_bytes(9) < need_ref
        for _ in range(2):  # twice: the ring's pads stay zero
            assert np.array_equal(op.forward_batch(x).cpu().numpy(), f_ref)
            assert np.array_equal(op.adjoint_batch(y).cpu().numpy(), a_ref)
    projector.ray_transform.cache_clear()


def test_unchunked_call_past_the_ring_is_refused(m):
    """A K1-K3 call whose gate pairs do not fit the ring returns MCT_ERR_ARG (no launch)
    and names the chunk API; chunk starts off a ring boundary are refused too."""
    from paper_2410_10503_b200 import _lib, workloads
    from paper_2410_10503_b200.engine import Engine

    cfgw = workloads.WorkloadConfig("ring_e", 32, 30, 47, 6, "rigid", 3, 1e-2, 1)
    prob, _ = fresh_problem(m, cfgw, 0, 1)
    eng = Engine([prob.operators], [prob.data])
    cfg = m.default_config("pdhg", [30.0] * 6, cfgw.alpha, 1, stacked_norm_sq=6 * 900.0)
    eng.set_params(cfg)
    L = _lib.load()
    assert L.mct_family_chunk_items(eng.family.handle, 6) == 2
    items = eng.items_pdhg()
    args = (eng.family.handle, ctypes.byref(items), ctypes.byref(eng._st), eng.tau,
            float(cfgw.alpha), _lib.ptr(eng.ws), _lib.stream_handle())
    assert L.mct_iter_prox_warp(*args) == 1
    assert b"chunk" in L.mct_last_error()
    items.first_item, items.item_count = 2, 4  # two pairs into a one-pair ring
    assert L.mct_iter_prox_warp(*args) == 1
    items.first_item, items.item_count = 1, 2  # odd start
    assert L.mct_iter_prox_warp(*args) == 1
    items.first_item, items.item_count = 2, 2
    assert L.mct_iter_prox_warp(*args) == 0
    # K4 takes the whole launch only
    assert L.mct_iter_adjoint_update(eng.family.handle, ctypes.byref(items),
                                     ctypes.byref(eng._st), None, _lib.ptr(eng.ws),
                                     _lib.stream_handle()) == 1


def test_c4_shape_workspace_is_bounded(m):
    """BASELINE C4 geometry (1024^2, 1440 x 1453, 40 gates): the pair ring bounds the
    fused-iteration workspace below 1 GB (one region per pair: 2.2 GB) and the C5
    batch (64 slices of 512^2) below 0.6 GB (one region per pair: 0.88 GB)."""
    from paper_2410_10503_b200 import projector

    projector.ray_transform.cache_clear()
    p4 = m.ray_transform(m.Geometry(1024, 1024, 1440, 1453, 1.0)).plan()
    assert p4.workspace_bytes(40) < 2**30
    p5 = m.ray_transform(m.Geometry(512, 512, 720, 729, 1.0)).plan()
    assert p5.workspace_bytes(64) < 0.6 * 2**30
    assert p5.workspace_bytes(20) > 10 * 16 * 2**20  # C3: every pair keeps its own region
    projector.ray_transform.cache_clear()


@pytest.mark.parametrize("half", [None, (4, 1), (4, 2)])
def test_chunked_gate_shard_rank_with_half_item(m, half):
    """One gate-sharded rank's iteration (4 local gates + a half-gate unit: two pairs
    and an unpaired half item on the side stream) through a 1-pair ring: partial dz, y
    and x equal the unchunked launch bit for bit, for three iterations."""
    import torch

    from paper_2410_10503_b200 import workloads
    from paper_2410_10503_b200.engine import Engine

    cfgw = workloads.WorkloadConfig("ring_h", 48, 40, 71, 6, "dense", 5, 1e-2, 3, peak=3.0)
    base, _ = fresh_problem(m, cfgw, 0, None)
    norms = [m.power_method(op, iterations=20) for op in base.operators]
    cfg = m.default_config("pdhg", norms, cfgw.alpha, 3,
                           stacked_norm_sq=float(sum(v * v for v in norms)))

    def rank_run(problem):
        eng = Engine([problem.operators], [problem.data], gate_range=(0, 4), half=half)
        eng.set_params(cfg)
        eng.reset()
        dz = torch.zeros_like(eng.x)
        outs = []
        for k in range(3):
            eng.iteration(eng.items_pdhg(iteration=k + 1), problem.alpha, dz=dz)
            eng.z_update(dz, cfg.theta)
            outs.append((dz.cpu().numpy().copy(), eng.y.cpu().numpy().copy(),
                         eng.x.cpu().numpy().copy()))
        return eng, outs

    eng_ref, ref = rank_run(base)
    assert np.abs(ref[-1][0]).max() > 0 and np.abs(ref[-1][2]).max() > 0
    prob, _ = fresh_problem(m, cfgw, 0, 1, data=list(base.data))
    eng, out = rank_run(prob)
    assert len(eng.chunks(eng.local, 0 if half is None else half[1])) == 2
    for (dz0, y0, x0), (dz1, y1, x1) in zip(ref, out):
        assert np.array_equal(dz0, dz1) and np.array_equal(y0, y1) and np.array_equal(x0, x1)


def test_ring_setter_validation_and_kernel_timer(m):
    """mct_ray_plan_set_ring_pairs rejects < 1 (ValueError through the binding); the
    KernelTimer marks of a chunked iteration give one K1-K3 mark per chunk, one K4 mark,
    and positive per-kernel times."""
    import torch

    from paper_2410_10503_b200 import projector, workloads
    from paper_2410_10503_b200.engine import Engine, KernelTimer

    projector.ray_transform.cache_clear()
    cfgw = workloads.WorkloadConfig("ring_t", 32, 30, 47, 6, "rigid", 3, 1e-2, 1)
    prob, _ = fresh_problem(m, cfgw, 0, 1)
    plan = prob.operators[0].outer.plan()
    with pytest.raises(ValueError):
        plan.set_ring_pairs(0)
    eng = Engine([prob.operators], [prob.data])
    eng.set_params(m.default_config("pdhg", [30.0] * 6, cfgw.alpha, 1, stacked_norm_sq=5400.0))
    timer = KernelTimer(torch)
    eng.iteration(eng.items_pdhg(), cfgw.alpha, mark=timer)
    torch.cuda.synchronize()
    assert timer.launches() == [3, 3, 3, 1]
    assert all(t > 0 for t in timer.times_ms())
    projector.ray_transform.cache_clear()
