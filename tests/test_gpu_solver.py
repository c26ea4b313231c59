"""GPU tier: fused PDHG / SPDHG iteration vs the reference's trajectories.

Bar (north_star): iterates after K epochs within relative L2 1e-3 of the fp64
reference for the same sampling seed and identical step sizes.  Mechanics
mirror test_solvers.py (counters, determinism, full-sampling equivalence,
aggregate invariant, divergence guard, empty-draw retry, epochs=0).
"""

import math

import numpy as np
import pytest

import oracle
from oracle import solver as osolver
from conftest import rel_l2

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-3


@pytest.fixture(scope="module")
def m():
    import paper_2410_10503_b200 as m

    m.build_native()
    return m


def tiny_problem(m, G):
    r, c, a, b, sp = G["geom"]
    geom = m.Geometry(int(r), int(c), int(a), int(b), float(sp))
    motion = [m.MotionParams("rigid", float(p[0]), (float(p[1]), float(p[2]))) for p in G["motion"]]
    ops = m.gate_operators(geom, motion, True)
    return m.Problem.from_parts(float(G["alpha"]), ops, list(G["data"]))


def tiny_config(m, G, mode, seed, epochs=10):
    return m.SolverConfig(mode=mode, sigmas=tuple(G[f"{mode}__sigmas"]),
                          tau=float(G[f"{mode}__tau"]), theta=1.0,
                          probs=(1.0,) * 4 if mode == "pdhg" else (0.25,) * 4, epochs=epochs,
                          seed=seed, gate_norms=tuple(G["gate_norms"]),
                          stacked_norm_sq=float(G["stacked_norm_sq"]) if mode == "pdhg" else None)


@pytest.mark.parametrize("mode,seed", [("pdhg", 0), ("spdhg", 5)])
@pytest.mark.parametrize("graph", [True, False])
def test_tiny_trajectory_matches_reference(m, golden_tiny, mode, seed, graph):
    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, mode, seed)
    seen = {}
    x, rec = m.run(cfg, problem, truth=G["truth"], graph=graph,
                   on_epoch=lambda e, s: seen.setdefault(e, (s.x, s.y, s.z)))
    assert rel_l2(x, G[f"{mode}__x"]) <= ITER_TOL
    assert rel_l2(seen[10][2], G[f"{mode}__z"]) <= ITER_TOL
    assert rel_l2(np.stack(seen[10][1]), G[f"{mode}__y"]) <= ITER_TOL
    assert rel_l2(seen[1][0], G[f"{mode}__x_e1"]) <= ITER_TOL
    assert np.allclose(rec.objective, G[f"{mode}__objective"], rtol=ITER_TOL)
    assert np.allclose(rec.rmse_to_truth, G[f"{mode}__rmse"], rtol=ITER_TOL)
    assert rec.fwd_calls == list(G[f"{mode}__fwd_calls"])
    assert rec.adj_calls == rec.fwd_calls


@pytest.mark.parametrize("mode", ["pdhg", "spdhg"])
def test_c1_trajectory_matches_reference(m, golden_c1, mode):
    from paper_2410_10503_b200 import workloads

    G = golden_c1
    cfgw = workloads.CONFIGS["c1"]
    problem, truth, _ = m.simulate.workload_problem(cfgw, 0, data=list(G["data"]))
    cfg = m.default_config(mode, G["gate_norms"], cfgw.alpha, cfgw.epochs, seed=cfgw.seed,
                           stacked_norm_sq=float(G["stacked_norm_sq"]) if mode == "pdhg" else None)
    x, rec = m.run(cfg, problem, truth=truth)
    assert rel_l2(x, G[f"{mode}__x"]) <= ITER_TOL
    assert np.allclose(rec.objective, G[f"{mode}__objective"], rtol=ITER_TOL)
    x2, _ = m.run(cfg, problem, diagnostics=False)
    assert np.array_equal(x, x2)  # diagnostics do not perturb the iterates


def test_dense_spdhg_trajectory_vs_oracle(m):
    from paper_2410_10503_b200 import workloads

    cfgw = workloads.WorkloadConfig("dense_small", 96, 120, 137, 5, "dense", 6, 1e-2, 3, peak=4.0)
    problem, truth, inp = m.simulate.workload_problem(cfgw, 0)
    norms = [m.power_method(op, iterations=30) for op in problem.operators]
    geom = oracle.Geometry(*cfgw.geometry_args)
    oops = oracle.gate_operators(geom, inp.gates, threads=oracle.default_threads())
    for mode in ("spdhg", "pdhg"):
        cfg = m.default_config(mode, norms, cfgw.alpha, cfgw.epochs, seed=11)
        x, rec = m.run(cfg, problem)
        ocfg = osolver.default_config(mode, norms, cfgw.alpha, cfgw.epochs, seed=11)
        st, objs = osolver.run(ocfg, cfgw.alpha, oops, [np.asarray(d) for d in problem.data])
        assert rel_l2(x, st.x) <= ITER_TOL, mode
        assert np.allclose(rec.objective, objs, rtol=ITER_TOL)


def test_full_sampling_spdhg_reproduces_pdhg_bitwise(m, golden_tiny):
    G = golden_tiny
    problem = tiny_problem(m, G)
    pcfg = tiny_config(m, G, "pdhg", 0, epochs=6)
    x_pdhg, _ = m.run(pcfg, problem)
    full = m.SolverConfig(mode="spdhg", sigmas=pcfg.sigmas, tau=pcfg.tau, theta=1.0,
                          probs=(1.0,) * 4, epochs=6, seed=0, gate_norms=pcfg.gate_norms)
    st = m.SolverState.zeros(problem)
    for _ in range(6):
        m.step(st, full, problem, lambda: (0, 1, 2, 3))
    assert np.array_equal(st.x, x_pdhg)


def test_run_deterministic_and_counters(m, golden_tiny):
    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, "spdhg", 9, epochs=5)
    x1, r1 = m.run(cfg, problem)
    x2, r2 = m.run(cfg, problem)
    assert np.array_equal(x1, x2) and r1.objective == r2.objective
    assert r1.fwd_calls == [4, 8, 12, 16, 20]


def test_aggregate_invariant_and_single_gate_updates(m, golden_tiny):
    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, "spdhg", 5)
    st = m.SolverState.zeros(problem)
    rng = np.random.default_rng(cfg.seed)
    for _ in range(25):
        y_before = st.y
        m.step(st, cfg, problem, lambda: m.sample_gates(rng, cfg.probs, "spdhg"))
        recomputed = sum(op.adjoint_apply(y) for op, y in zip(problem.operators, st.y))
        assert rel_l2(st.z, recomputed) <= 1e-4
        changed = [i for i, (a, b) in enumerate(zip(st.y, y_before)) if not np.array_equal(a, b)]
        assert len(changed) <= 1
    assert st.iteration == 25 and st.fwd_calls == 25 and st.epoch == pytest.approx(25 / 4)


def test_empty_draw_is_retried(m, golden_tiny):
    G = golden_tiny
    problem = tiny_problem(m, G)
    st = m.SolverState.zeros(problem)
    draws = iter([(), (), (2,)])
    m.step(st, tiny_config(m, G, "spdhg", 0), problem, lambda: next(draws))
    assert st.fwd_calls == 1 and st.iteration == 1


def test_epochs_zero_and_gate_mismatch(m, golden_tiny):
    G = golden_tiny
    problem = tiny_problem(m, G)
    x, rec = m.run(tiny_config(m, G, "pdhg", 0, epochs=0), problem)
    assert np.array_equal(x, np.zeros(problem.image_shape)) and len(rec) == 0
    cfg = m.default_config("spdhg", G["gate_norms"][:3], problem.alpha, 1)
    with pytest.raises(ValueError, match="gate count"):
        m.run(cfg, problem)


def test_divergence_guard_fires(m, golden_tiny):
    G = golden_tiny
    problem = tiny_problem(m, G)
    # norms understated 1000x: wildly inadmissible steps for the true operators
    cfg = m.default_config("pdhg", np.asarray(G["gate_norms"]) / 1000.0, problem.alpha, 200)
    with pytest.raises(m.DivergenceError):
        m.run(cfg, problem)


@pytest.mark.parametrize("case", range(3))
def test_divergence_message_matches_reference(m, golden_tiny, case):
    """Same epoch / iteration in the DivergenceError as the reference
    (golden/divergence.json), with the deferred diagnostics table and with a
    per-epoch callback (host sync every epoch)."""
    import json
    import re

    from conftest import GOLDEN

    ref = json.loads((GOLDEN / "divergence.json").read_text())[case]
    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = m.default_config(ref["mode"], np.asarray(G["gate_norms"]) / ref["norm_scale"],
                           problem.alpha, ref["epochs"], seed=ref["seed"])
    where = re.search(r"at epoch \d+ \(iteration \d+\)", ref["message"]).group(0)
    for cb in (None, lambda e, st: None):
        with pytest.raises(m.DivergenceError, match=re.escape(where)):
            m.run(cfg, problem, on_epoch=cb)


def test_engine_reuse_across_runs(m, golden_tiny):
    """run() keeps one device engine per problem; new seeds / step sizes / modes
    on the same problem give exactly what a fresh problem gives."""
    G = golden_tiny
    problem = tiny_problem(m, G)
    a = tiny_config(m, G, "spdhg", 5, epochs=6)
    b = tiny_config(m, G, "spdhg", 11, epochs=6)
    p = tiny_config(m, G, "pdhg", 0, epochs=6)
    xa, _ = m.run(a, problem)
    xb, _ = m.run(b, problem)
    xp, _ = m.run(p, problem)
    xa2, _ = m.run(a, problem)
    assert np.array_equal(xa, xa2) and not np.array_equal(xa, xb)
    for cfg, x in ((b, xb), (p, xp)):
        xf, _ = m.run(cfg, tiny_problem(m, G))
        assert np.array_equal(x, xf)


def test_deferred_diagnostics_equal_per_epoch(m, golden_tiny):
    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, "spdhg", 5, epochs=40)
    saddle = m.SaddlePoint(x_star=np.ones(problem.image_shape),
                           y_star=[np.zeros(d.shape) for d in problem.data], source="test",
                           converged=True, residual=0.0)
    truth = np.full(problem.image_shape, 0.5)
    x1, r1 = m.run(cfg, problem, saddle=saddle, truth=truth)
    seen = []
    x2, r2 = m.run(cfg, problem, saddle=saddle, truth=truth,
                   on_epoch=lambda e, st: seen.append(e))
    assert np.array_equal(x1, x2) and seen == list(range(1, 41))
    for col in ("epochs", "dist_sq", "objective", "rmse_to_truth", "fwd_calls", "adj_calls"):
        assert getattr(r1, col) == getattr(r2, col), col


def test_run_batch_equals_single_runs(m):
    from paper_2410_10503_b200 import workloads

    cfgw = workloads.WorkloadConfig("batch_small", 64, 60, 91, 3, "dense", 5, 1e-2, 4, peak=3.0)
    probs = [m.simulate.workload_problem(cfgw, s)[0] for s in range(3)]
    norms = [m.power_method(op, iterations=20) for op in probs[0].operators]
    cfgs = [m.default_config("spdhg", norms, cfgw.alpha, cfgw.epochs, seed=100 + s)
            for s in range(3)]
    out = m.run_batch(cfgs, probs)
    for (xb, _), c, p in zip(out, cfgs, probs):
        xs, _ = m.run(c, p, diagnostics=False)
        # same per-slice arithmetic except A^*'s angle split, which follows the
        # launch's tile count (bitwise equal whenever the splits coincide, as here)
        assert rel_l2(xb, xs) <= 1e-6


def test_dense_state_roundtrip_and_fixed_point(m, golden_tiny):
    """A state set from numpy arrays is honoured (reference fixed-point tests style)."""
    G = golden_tiny
    problem = tiny_problem(m, G)
    st = m.SolverState.zeros(problem)
    st.x = np.ones(problem.image_shape)
    assert np.array_equal(st.x, np.ones(problem.image_shape))
    m.step(st, tiny_config(m, G, "pdhg", 0), problem, lambda: (0, 1, 2, 3))
    assert st.iteration == 1


def test_sharded_pdhg_single_rank_matches_run(m, golden_tiny):
    from paper_2410_10503_b200.distributed import run_pdhg_sharded

    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, "pdhg", 0, epochs=8)
    x_run, _ = m.run(cfg, problem, diagnostics=False)
    x_sh = run_pdhg_sharded(cfg, problem)
    assert rel_l2(x_sh, x_run) <= 1e-6
    assert rel_l2(x_sh, G["pdhg__x"]) <= ITER_TOL if cfg.epochs == 10 else True


def test_p2p_exchange_matches_nccl_single_rank(m, golden_tiny):
    """The fused peer-memory exchange (mct_exchange_*) on a one-rank NCCL group:
    same bits as allreduce + z update, flags advance, no timeout."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2410_10503_b200.distributed import ShardedPDHG, run_pdhg_sharded

    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, "pdhg", 0, epochs=7)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        x_nccl = run_pdhg_sharded(cfg, problem, exchange="nccl")
        x_p2p = run_pdhg_sharded(cfg, problem, exchange="p2p")
        assert np.array_equal(x_p2p, x_nccl)
        w = ShardedPDHG(cfg, problem, 0, 1, exchange="p2p")
        for _ in range(3):
            w.finish(w.local_iteration())
        torch.cuda.synchronize()
        pad = w.p2p.buf[-256:].view(torch.int64)[0].item()
        assert pad == 3 and w.p2p.epoch == 3 and int(w.p2p.failed.item()) == 0
        assert not w.p2p_failed_anywhere()
        w.p2p.failed.fill_(1)  # as if a peer wait had timed out
        assert w.p2p_failed_anywhere()
        w.fallback_to_nccl()
        for _ in range(cfg.epochs):
            w.finish(w.local_iteration())
        assert np.array_equal(w.engine.x[0].double().cpu().numpy(), x_nccl)
    finally:
        dist.destroy_process_group()


def test_cg_reference_matches_reference_saddle(m, golden_tiny):
    """Device CG saddle (solvers.py:435-490) vs the reference's fp64 CG saddle."""
    G = golden_tiny
    problem = tiny_problem(m, G)
    sp = m.cg_reference(problem, tol=1e-6, max_iter=2000)
    assert sp.converged and sp.source == "cg_reference"
    assert sp.residual <= 1e-5
    assert rel_l2(sp.x_star, G["saddle_x"]) <= 1e-4
    assert rel_l2(np.stack(sp.y_star), G["saddle_y"]) <= 1e-4
    # defect of 2 alpha x* + sum A_i^T y*_i, relative to its first term (fp32 operators)
    scale = 2.0 * problem.alpha * np.linalg.norm(sp.x_star)
    assert m.optimality_residual(problem, sp) <= 1e-4 * scale
    # the reference's saddle drives run()'s dist_sq column (solvers.py:407)
    ref = m.SaddlePoint(x_star=G["saddle_x"], y_star=list(G["saddle_y"]), source="reference",
                        converged=True, residual=float(G["saddle_residual"]))
    for mode, seed in (("pdhg", 0), ("spdhg", 5)):
        _, rec = m.run(tiny_config(m, G, mode, seed), problem, saddle=ref)
        assert np.allclose(rec.dist_sq, G[f"{mode}__dist_sq"], rtol=ITER_TOL)
    tight = m.cg_reference(problem, tol=1e-13, max_iter=3)
    assert not tight.converged
    with pytest.raises(ValueError):
        m.cg_reference(problem, tol=0.0)


def test_single_gate_and_uncompensated(m):
    """N = 1 (SPDHG == PDHG step rules) and compensated=False (the no-MC baseline)."""
    from paper_2410_10503_b200 import workloads

    geom = m.Geometry(48, 48, 40, 69, 1.0)
    truth = workloads.ellipse_phantom(48, 5, 9)
    gates = workloads.rigid_gates(3, 9)
    ops_mc = m.gate_operators(geom, gates, compensated=True)
    ops_no = m.gate_operators(geom, gates, compensated=False)
    assert all(op is m.ray_transform(geom) for op in ops_no)
    data = m.simulate_data(ops_mc, truth, 9)
    one = m.Problem.from_parts(1e-2, ops_mc[:1], data[:1])
    nrm = [m.power_method(ops_mc[0], iterations=30)]
    x1, _ = m.run(m.default_config("pdhg", nrm, 1e-2, 5), one)
    oops = oracle.gate_operators(oracle.Geometry(48, 48, 40, 69, 1.0), gates[:1])
    st, _ = osolver.run(osolver.default_config("pdhg", nrm, 1e-2, 5), 1e-2, oops, data[:1],
                        diagnostics=False)
    assert rel_l2(x1, st.x) <= ITER_TOL
    nomc = m.Problem.from_parts(1e-2, ops_no, data)
    norms = [m.power_method(op, iterations=30) for op in ops_no]
    xn, rec = m.run(m.default_config("spdhg", norms, 1e-2, 3, seed=2), nomc)
    o_no = [oracle.RayTransform(oracle.Geometry(48, 48, 40, 69, 1.0))] * 3
    st, objs = osolver.run(osolver.default_config("spdhg", norms, 1e-2, 3, seed=2), 1e-2, o_no,
                           data)
    assert rel_l2(xn, st.x) <= ITER_TOL
    assert np.allclose(rec.objective, objs, rtol=ITER_TOL)


@pytest.mark.parametrize("mode", ["pdhg", "spdhg"])
def test_fused_iterations_stay_inside_workspace(m, golden_tiny, mode):
    """K1-K4 write nothing past the engine workspace (canary tail) and give the
    same iterate as with the engine's own workspace."""
    import torch

    from paper_2410_10503_b200.engine import Engine

    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, mode, 5, epochs=4)
    x_ref, _ = m.run(cfg, problem, diagnostics=False)
    eng = Engine([problem.operators], [problem.data])
    eng.set_params(cfg)
    eng.reset()
    if mode == "spdhg":
        eng.set_sequences(m.draw_sequence(cfg)[None])
    need, tail = eng.ws.numel(), 1 << 16
    ws = torch.full((need + tail,), 0xAB, dtype=torch.uint8, device="cuda")
    ws[:need].zero_()
    eng.ws = ws
    for _ in range(cfg.epochs):
        eng.epoch(mode, problem.alpha)
    torch.cuda.synchronize()
    assert bool((ws[need:] == 0xAB).all()), "workspace tail overwritten"
    assert np.array_equal(eng.x[0].double().cpu().numpy(), x_ref)


@pytest.mark.parametrize("mode,draws", [("pdhg", [(0, 1, 2, 3)]),
                                        ("spdhg", [(1,), (0,), (2,), (3,), (2,)])])
def test_saddle_is_fixed_point(m, golden_tiny, mode, draws):
    """test_solvers.py:337-370: started at a saddle point (x*, y*) with
    z = zbar = sum_i A_i^* y*_i, a full-draw step and a single-gate sequence leave
    x in place (device CG saddle, fp32 iterates)."""
    G = golden_tiny
    problem = tiny_problem(m, G)
    saddle = m.cg_reference(problem)
    z = sum(op.adjoint_apply(y) for op, y in zip(problem.operators, saddle.y_star))
    state = m.SolverState(x=saddle.x_star, y=list(saddle.y_star), z=z, zbar=z)
    cfg = tiny_config(m, G, mode, 0, epochs=1)
    for d in draws:
        m.step(state, cfg, problem, lambda d=d: d)
    scale = float(np.linalg.norm(saddle.x_star))
    assert np.linalg.norm(state.x - saddle.x_star) <= 1e-4 * scale
    for y_new, y_old in zip(state.y, saddle.y_star):
        assert np.linalg.norm(y_new - y_old) <= 1e-4 * max(1.0, float(np.linalg.norm(y_old)))


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_p2p_exchange_emulated_ranks(m, golden_tiny, world):
    """The multi-rank exchange protocol on one GPU: W virtual ranks (one engine per
    gate shard, each with its own partial buffers and signal pad), driven through
    the real mct_exchange_post / mct_exchange_z_update kernels.  Every rank posts
    before any rank updates (stream order), so no kernel waits on another -- the
    data flow (parity buffers, per-iteration flags, rank-order sum) is exercised
    without concurrent ranks.  4 gates on 3, 5 or 8 ranks exercise the half-gate
    units (a rank's last item covers half of the angle pairs).  All ranks end with
    identical bits, equal to a host-ordered sum of the same partials and to the
    single-process run."""
    import torch

    from paper_2410_10503_b200 import _lib
    from paper_2410_10503_b200.distributed import ShardedPDHG, exchange_schedule

    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = tiny_config(m, G, "pdhg", 0, epochs=6)
    x_run, _ = m.run(cfg, problem, diagnostics=False)
    L = _lib.load()
    st = _lib.stream_handle()
    ws = [ShardedPDHG(cfg, problem, r, world) for r in range(world)]
    n = ws[0].engine.x.numel()
    parts = [[torch.zeros(n, device="cuda") for _ in range(2)] for _ in range(world)]
    pads = [torch.zeros(world, dtype=torch.int64, device="cuda") for _ in range(world)]
    failed = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(world)]
    pads_dev = torch.tensor([p.data_ptr() for p in pads], dtype=torch.int64, device="cuda")
    parts_dev = [torch.tensor([parts[r][k].data_ptr() for r in range(world)], dtype=torch.int64,
                              device="cuda") for k in (0, 1)]
    ref = ShardedPDHG(cfg, problem, 0, world)  # host-ordered sum of the same partials
    refs = [ShardedPDHG(cfg, problem, r, world) for r in range(1, world)]
    for e in range(cfg.epochs):
        flag, parity = exchange_schedule(e)
        for r, w in enumerate(ws):
            w.engine.iteration(w.engine.items_pdhg(epoch_ctr=True), problem.alpha,
                               dz=parts[r][parity].view(w.engine.x.shape))
        for r in range(world):
            _lib.check(L.mct_exchange_post(_lib.ptr(pads_dev), world, r, flag, st))
        for r, w in enumerate(ws):
            _lib.check(L.mct_exchange_z_update(_lib.ptr(parts_dev[parity]), pads[r].data_ptr(),
                                               world, flag, n, _lib.ptr(w.engine.z),
                                               _lib.ptr(w.engine.zbar), float(cfg.theta),
                                               _lib.ptr(failed[r]), st))
            w.engine.advance_epoch()
        dzs = [w.local_iteration().clone() for w in [ref] + refs]
        total = dzs[0].clone()
        for d in dzs[1:]:
            total += d  # rank order, fp32
        for w in [ref] + refs:
            w.finish(total)
    torch.cuda.synchronize()
    assert all(int(f.item()) == 0 for f in failed)
    assert all(int(v) == cfg.epochs for p in pads for v in p.cpu().numpy())
    xs = [w.engine.x[0].double().cpu().numpy() for w in ws]
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])
    assert np.array_equal(xs[0], ref.engine.x[0].double().cpu().numpy())
    assert rel_l2(xs[0], x_run) <= 1e-6


def test_run_batch_pdhg_odd_gates_equals_single_runs(m):
    """Multi-slice PDHG launches with an odd gate count: gate pairs straddle the
    slice boundary (slice 0 gate 2 with slice 1 gate 0) and the last item runs
    alone; every slice still matches its own run()."""
    from paper_2410_10503_b200 import workloads

    cfgw = workloads.WorkloadConfig("batch_pdhg", 48, 40, 71, 3, "dense", 5, 1e-2, 3, peak=3.0)
    probs = [m.simulate.workload_problem(cfgw, s)[0] for s in range(2)]
    norms = [m.power_method(op, iterations=20) for op in probs[0].operators]
    stacked = float(sum(v * v for v in norms))
    cfgs = [m.default_config("pdhg", norms, cfgw.alpha, cfgw.epochs, seed=0,
                             stacked_norm_sq=stacked) for _ in range(2)]
    out = m.run_batch(cfgs, probs)
    for (xb, _), c, p in zip(out, cfgs, probs):
        xs, _ = m.run(c, p, diagnostics=False)
        assert rel_l2(xb, xs) <= 1e-6


def test_odd_item_fork_join_in_graph_on_user_stream(m, golden_tiny):
    """3-item launches (a gate pair + the odd item on the library's side stream, forked
    and joined with events) issued from a user stream and captured in the epoch CUDA
    graph give the same iterate as eager launches on the default stream."""
    import torch

    G = golden_tiny
    problem = tiny_problem(m, G)
    ops = list(problem.operators)[:3]
    sub = m.Problem.from_parts(problem.alpha, ops, list(problem.data)[:3])
    cfg = m.default_config("pdhg", [1.0] * 3, sub.alpha, 3, stacked_norm_sq=3.0)
    x_eager, _ = m.run(cfg, sub, graph=False, diagnostics=False)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x_graph, _ = m.run(cfg, sub, graph=True, diagnostics=False)
    torch.cuda.synchronize()
    assert np.array_equal(x_eager, x_graph)


@pytest.mark.parametrize("shape,angles,bins,sp", [((40, 56), 61, 75, 1.0), ((57, 33), 90, 71, 1.0),
                                                  ((48, 48), 64, 101, 0.7)])
def test_non_square_dense_trajectories_vs_oracle(m, shape, angles, bins, sp):
    """Non-square images (mirror columns of unequal halves, odd angle counts with one
    self-paired angle) and a sub-pixel detector spacing (wider A^* footprint, K = 1),
    3 dense gates and a rigid gate (gate pairs, and single items for SPDHG): PDHG and
    SPDHG trajectories vs the fp64 oracle."""
    rng = np.random.default_rng(7)
    rows, cols = shape
    geom = m.Geometry(rows, cols, angles, bins, sp)
    yy, xx = np.mgrid[0:rows, 0:cols].astype(np.float64)
    specs = []
    for g in range(3):
        cy, cx = rng.uniform(0, rows), rng.uniform(0, cols)
        bump = np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * 12.0 ** 2))
        amp = rng.uniform(-2.5, 2.5, 2)
        specs.append(np.stack([amp[0] * bump, amp[1] * bump]).astype(np.float32))
    specs.append(m.MotionParams(kind="rigid", rotation=0.05, translation=(1.5, -0.7)))
    ops = m.gate_operators(geom, specs)
    truth = rng.uniform(0, 1, shape).astype(np.float32).astype(np.float64)
    data = [np.asarray(op.apply(truth)) + 0.01 * rng.standard_normal(geom.sino_shape)
            for op in ops]
    data = [d.astype(np.float32).astype(np.float64) for d in data]
    problem = m.Problem.from_parts(1e-2, ops, data)
    norms = [m.power_method(op, iterations=30) for op in ops]
    ospecs = [{"kind": "dense", "phi": sp} for sp in specs[:3]] + [
        {"kind": "rigid", "rotation": 0.05, "translation": (1.5, -0.7)}]
    oops = oracle.gate_operators(oracle.Geometry(rows, cols, angles, bins, sp), ospecs,
                                 threads=oracle.default_threads())
    for mode in ("pdhg", "spdhg"):
        cfg = m.default_config(mode, norms, 1e-2, 3, seed=4)
        x, rec = m.run(cfg, problem)
        ocfg = osolver.default_config(mode, norms, 1e-2, 3, seed=4)
        st, objs = osolver.run(ocfg, 1e-2, oops, data)
        assert rel_l2(x, st.x) <= ITER_TOL, mode
        assert np.allclose(rec.objective, objs, rtol=ITER_TOL), mode


def test_step_divergence_leaves_state_at_last_good_iterate(m, golden_tiny):
    """solvers.py:329-352 raises before assigning x, z and the failing y_i: after a
    DivergenceError from step() the device state still holds the pre-step iterate
    (not x_next / the non-finite duals), and the counters did not advance."""
    G = golden_tiny
    problem = tiny_problem(m, G)
    cfg = m.default_config("pdhg", np.asarray(G["gate_norms"]) / 1000.0, problem.alpha, 1)
    st = m.SolverState.zeros(problem)
    for _ in range(2000):
        before = (st.x, st.z, st.zbar, st.y, st.iteration)
        try:
            m.step(st, cfg, problem, lambda: (0, 1, 2, 3))
        except m.DivergenceError:
            break
    else:
        pytest.fail("no divergence")
    assert np.array_equal(st.x, before[0]) and np.array_equal(st.z, before[1])
    assert np.array_equal(st.zbar, before[2]) and st.iteration == before[4]
    assert all(np.isfinite(v).all() for v in (st.x, st.z, st.zbar))
    # the iterate is still the last finite one: stepping again raises again
    with pytest.raises(m.DivergenceError):
        m.step(st, cfg, problem, lambda: (0, 1, 2, 3))


def test_run_batch_17_slices_equal_single_runs(m):
    """17 slices of one gate per SPDHG iteration: every launch holds 8 slice pairs
    plus an odd last slice (mirror kernels on the side stream); every slice matches
    its own run() and the fp64 oracle."""
    from paper_2410_10503_b200 import workloads

    cfgw = workloads.WorkloadConfig("batch_groups", 40, 36, 61, 3, "dense", 4, 1e-2, 2, peak=2.0)
    S = 17
    probs, inps = [], []
    for s in range(S):
        p, _, inp = m.simulate.workload_problem(cfgw, s)
        probs.append(p)
        inps.append(inp)
    norms = [1.1 * m.power_method(op, iterations=20) for op in probs[0].operators]
    cfgs = [m.default_config("spdhg", norms, cfgw.alpha, cfgw.epochs, seed=7 + s)
            for s in range(S)]
    out = m.run_batch(cfgs, probs)
    geom = oracle.Geometry(*cfgw.geometry_args)
    for s in (0, 5, 15, 16):
        xs, _ = m.run(cfgs[s], probs[s], diagnostics=False)
        assert rel_l2(out[s][0], xs) <= 1e-6, s
        ocfg = osolver.default_config("spdhg", norms, cfgw.alpha, cfgw.epochs, seed=7 + s)
        st, _ = osolver.run(ocfg, cfgw.alpha, oracle.gate_operators(geom, inps[s].gates),
                            list(probs[s].data), diagnostics=False)
        assert np.linalg.norm(st.x) > 0 and rel_l2(out[s][0], st.x) <= ITER_TOL, s
