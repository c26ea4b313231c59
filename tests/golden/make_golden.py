"""Generate golden fixtures from the *imported reference* (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array here is an output of the unmodified reference package ``mctomo``
(/root/reference/pkg/src/mctomo) on seeded inputs; the inputs are fp32-rounded so
the GPU path and the reference consume identical values.  The reference cannot
travel to the GPU box, so its outputs are committed as small .npz fixtures.
Nothing here is copied from the reference tests' data (they hold none on disk).
"""

from __future__ import annotations

import math
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from mctomo.linops import power_method, stacked_norm_sq  # noqa: E402
from mctomo.motion import MotionParams, WarpOperator, motion_sequence  # noqa: E402
from mctomo.projector import Geometry, ray_transform  # noqa: E402
from mctomo.simulate import (estimate_norms, gate_operators, gaussian_field,  # noqa: E402
                             generate, make_phantom)
from mctomo.solvers import (Problem, cg_reference, default_config, optimality_residual,  # noqa: E402
                            run, sample_gates)

from paper_2410_10503_b200 import workloads  # noqa: E402  (numpy-only input generators)

F32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731

PROJECTOR_GEOMS = {
    "fast": (64, 64, 128, 128, 64.0 * math.sqrt(2.0) / 128.0),
    "rect_spacing": (33, 21, 24, 40, 1.1),
    "tiny": (24, 24, 16, 32, math.hypot(24, 24) / 32),
    "many_angles": (17, 17, 180, 25, 1.0),
    "axis_exact": (65, 65, 48, 95, 1.0),
    "half_spacing": (16, 16, 8, 11, 0.5),
    "lin": (24, 24, 12, 30, 1.2),
    "c1": (128, 128, 180, 183, 1.0),
    "odd_rect": (40, 31, 37, 51, 1.0),
}

WARP_CASES = {
    "rigid_a": (("rigid", 0.37, (1.3, -0.8), 1.0), (20, 20)),
    "rigid_b": (("rigid", -0.2, (0.0, 2.7), 1.0), (17, 23)),
    "dilatation": (("dilatation", 0.0, (0.0, 0.0), 1.06), (20, 20)),
    "quarter": (("rigid", math.pi / 2.0, (0.0, 0.0), 1.0), (15, 15)),
    "half": (("rigid", math.pi, (0.0, 0.0), 1.0), (11, 11)),
    "shift": (("rigid", 0.0, (2.0, 3.0), 1.0), (16, 16)),
    "out_of_frame": (("rigid", 0.0, (100.0, 0.0), 1.0), (8, 8)),
    "c1_like": (("rigid", math.radians(4.2), (2.3, -1.7), 1.0), (128, 128)),
    "shrink": (("dilatation", 0.0, (0.0, 0.0), 0.93), (31, 26)),
}


def projector_cases():
    rng = np.random.default_rng(20241014)
    out = {}
    for name, g in PROJECTOR_GEOMS.items():
        geom = Geometry(*g)
        op = ray_transform(geom)
        x = F32(rng.standard_normal(geom.image_shape))
        y = F32(rng.standard_normal(geom.sino_shape))
        out[f"{name}__geom"] = np.array(g, dtype=np.float64)
        out[f"{name}__x"] = x
        out[f"{name}__y"] = y
        out[f"{name}__Ax"] = op.apply(x)
        out[f"{name}__ATy"] = op.adjoint_apply(y)
    np.savez_compressed(HERE / "projector.npz", **out)


def warp_cases():
    rng = np.random.default_rng(7)
    out = {}
    for name, ((kind, rot, tr, sc), shape) in WARP_CASES.items():
        op = WarpOperator(MotionParams(kind, rot, tr, sc), shape)
        x = F32(rng.standard_normal(shape))
        y = F32(rng.standard_normal(shape))
        out[f"{name}__params"] = np.array([rot, tr[0], tr[1], sc], dtype=np.float64)
        out[f"{name}__shape"] = np.array(shape)
        out[f"{name}__kind"] = np.array(0 if kind == "rigid" else 1)
        out[f"{name}__x"] = x
        out[f"{name}__y"] = y
        out[f"{name}__Dx"] = op.apply(x)
        out[f"{name}__DTy"] = op.adjoint_apply(y)
    np.savez_compressed(HERE / "warps.npz", **out)


def sampling_cases():
    out = {}
    for n in (4, 10, 20):
        for seed in (0, 5, 42):
            rng = np.random.default_rng(seed)
            probs = (1.0 / n,) * n
            out[f"n{n}_s{seed}"] = np.array(
                [sample_gates(rng, probs, "spdhg")[0] for _ in range(50 * n)], dtype=np.int32)
    out["field_5x7_1234_3"] = gaussian_field((5, 7), 1234, 3)
    out["field_c1_0_2"] = gaussian_field((180, 183), 0, 2)
    np.savez_compressed(HERE / "sampling.npz", **out)


def solver_tiny():
    geom = Geometry(24, 24, 16, 32, math.hypot(24, 24) / 32)
    phantom = make_phantom("nested_shells", 24, 24)
    motion = motion_sequence("rigid", 4, magnitude=0.6)
    ds = generate(phantom, motion, geom, master_seed=3)
    data = [F32(s) for s in ds.sinograms]
    norms = estimate_norms(geom, motion, iterations=40)
    alpha = norms["base_norm_sq"] / 70.0
    ops = gate_operators(geom, motion, True)
    problem = Problem.from_parts(alpha, ops, data)
    out = {
        "geom": np.array([24, 24, 16, 32, math.hypot(24, 24) / 32]),
        "motion": np.array([[m.rotation, m.translation[0], m.translation[1]] for m in motion]),
        "data": np.stack(data),
        "truth": phantom,
        "gate_norms": np.array(norms["gate_norms"]),
        "stacked_norm_sq": np.array(norms["stacked_norm_sq"]),
        "base_norm_sq": np.array(norms["base_norm_sq"]),
        "alpha": np.array(alpha),
    }
    saddle = cg_reference(problem, tol=1e-13, max_iter=3000)
    out["saddle_x"] = saddle.x_star
    out["saddle_y"] = np.stack(saddle.y_star)
    out["saddle_residual"] = np.array(saddle.residual)
    out["saddle_optimality"] = np.array(optimality_residual(problem, saddle))
    for mode, seed in (("pdhg", 0), ("spdhg", 5)):
        cfg = default_config(mode, norms["gate_norms"], alpha, epochs=10, seed=seed,
                             stacked_norm_sq=norms["stacked_norm_sq"] if mode == "pdhg" else None)
        states = {}

        def grab(e, s, states=states):
            states[e] = (s.x.copy(), [v.copy() for v in s.y], s.z.copy(), s.zbar.copy())

        x, rec = run(cfg, problem, saddle=saddle, truth=phantom, on_epoch=grab)
        out[f"{mode}__dist_sq"] = np.array(rec.dist_sq)
        out[f"{mode}__x"] = x
        out[f"{mode}__y"] = np.stack(states[10][1])
        out[f"{mode}__z"] = states[10][2]
        out[f"{mode}__zbar"] = states[10][3]
        out[f"{mode}__x_e1"] = states[1][0]
        out[f"{mode}__objective"] = np.array(rec.objective)
        out[f"{mode}__rmse"] = np.array(rec.rmse_to_truth)
        out[f"{mode}__fwd_calls"] = np.array(rec.fwd_calls)
        out[f"{mode}__sigmas"] = np.array(cfg.sigmas)
        out[f"{mode}__tau"] = np.array(cfg.tau)
    np.savez_compressed(HERE / "solver_tiny.npz", **out)


def solver_c1():
    cfg_w = workloads.CONFIGS["c1"]
    inp = workloads.slice_inputs(cfg_w, 0)
    geom = Geometry(*cfg_w.geometry_args)
    motion = [MotionParams("rigid", g["rotation"], tuple(g["translation"])) for g in inp.gates]
    ops = gate_operators(geom, motion, True)
    phantom = inp.phantom.astype(np.float64)
    clean = [op.apply(phantom) for op in ops]
    data = [F32(d) for d in workloads.noisy_data(clean, inp.seed)]
    t0 = time.time()
    norms = estimate_norms(geom, motion, iterations=100)
    print(f"  c1 norms {time.time() - t0:.1f}s", flush=True)
    problem = Problem.from_parts(cfg_w.alpha, ops, data)
    out = {
        "phantom": inp.phantom,
        "data": np.stack(data).astype(np.float32),
        "clean_0": clean[0],
        "gate_norms": np.array(norms["gate_norms"]),
        "stacked_norm_sq": np.array(norms["stacked_norm_sq"]),
        "base_norm_sq": np.array(norms["base_norm_sq"]),
    }
    for mode in ("pdhg", "spdhg"):
        cfg = default_config(mode, norms["gate_norms"], cfg_w.alpha, epochs=cfg_w.epochs,
                             seed=cfg_w.seed,
                             stacked_norm_sq=norms["stacked_norm_sq"] if mode == "pdhg" else None)
        t0 = time.time()
        x, rec = run(cfg, problem, truth=phantom)
        print(f"  c1 {mode} {time.time() - t0:.1f}s", flush=True)
        out[f"{mode}__x"] = x
        out[f"{mode}__objective"] = np.array(rec.objective)
        out[f"{mode}__rmse"] = np.array(rec.rmse_to_truth)
    np.savez_compressed(HERE / "solver_c1.npz", **out)


def divergence_cases():
    """The reference's DivergenceError messages on the tiny preset with
    inadmissible (understated-norm) step sizes (solvers.py:401-419)."""
    import json

    from mctomo.solvers import DivergenceError

    with np.load(HERE / "solver_tiny.npz") as f:
        G = {k: f[k] for k in f.files}
    r, c, a, b, sp = G["geom"]
    geom = Geometry(int(r), int(c), int(a), int(b), float(sp))
    motion = [MotionParams("rigid", float(p[0]), (float(p[1]), float(p[2]))) for p in G["motion"]]
    prob = Problem.from_parts(float(G["alpha"]), gate_operators(geom, motion, True),
                              list(G["data"]))
    out = []
    for mode, scale in (("pdhg", 1000.0), ("spdhg", 1000.0), ("pdhg", 30.0)):
        cfg = default_config(mode, np.asarray(G["gate_norms"]) / scale, prob.alpha, 200, seed=3)
        try:
            run(cfg, prob)
            msg = None
        except DivergenceError as exc:
            msg = str(exc)
        out.append({"mode": mode, "norm_scale": scale, "seed": 3, "epochs": 200, "message": msg})
    (HERE / "divergence.json").write_text(json.dumps(out, indent=1) + "\n")


def dataset_cases():
    """Data generation + file formats (§8f #3/#4): phantoms, the pinned noise
    stream, generate(), and the reference's own on-disk files (dataset and
    saddle directories, convergence CSV, PGM) written by its experiment_io."""
    import shutil

    from mctomo import experiment_io as rio
    from mctomo.simulate import NoiseModel, nonrigid_preset, rigid_preset
    from mctomo.solvers import SaddlePoint

    out = {}
    for kind in ("nested_shells", "thorax"):
        for shape in ((48, 40), (64, 64), (17, 33)):
            out[f"phantom_{kind}_{shape[0]}x{shape[1]}"] = make_phantom(kind, *shape)
    for name, (shape, seed, gate) in {"f_5x7": ((5, 7), 1234, 3), "f_odd": ((1, 13), 7, 0),
                                      "f_one": ((1, 1), 9, 2),
                                      "f_big": ((128, 129), (1 << 64) + 5, 11)}.items():
        out[name] = gaussian_field(shape, seed, gate)
    tiny = Geometry(24, 24, 16, 32, math.hypot(24, 24) / 32)
    ph = make_phantom("nested_shells", 24, 24)
    cases = {"gen_rigid": (ph, motion_sequence("rigid", 4, 0.6), None, 3),
             "gen_rigid_clean": (ph, motion_sequence("rigid", 4, 0.6), NoiseModel(0.0), 0),
             "gen_dil": (make_phantom("thorax", 24, 24), motion_sequence("dilatation", 3, 0.8),
                         NoiseModel(0.4), 5)}
    for name, (phantom, motion, noise, seed) in cases.items():
        ds = generate(phantom, motion, tiny, noise, master_seed=seed)
        out[f"{name}_sinos"] = np.stack(ds.sinograms)
        out[f"{name}_sigma"] = np.float64(ds.sigma)
    for name, fn in (("preset_rigid", rigid_preset), ("preset_nonrigid", nonrigid_preset)):
        ds = fn(size="fast", seed=1, magnitude=0.3)
        out[f"{name}_sinos"] = np.stack(ds.sinograms[:3])  # first gates (fixture size)
        out[f"{name}_sigma"] = np.float64(ds.sigma)
        out[f"{name}_truth"] = ds.truth
    # on-disk formats
    io_dir = HERE / "io"
    shutil.rmtree(io_dir, ignore_errors=True)
    io_dir.mkdir()
    ds = generate(ph, motion_sequence("rigid", 4, 0.6), tiny, None, master_seed=3,
                  phantom_kind="nested_shells", magnitude=0.6)
    rio.save_dataset(ds, io_dir / "dataset", norms={"gate_norms": [1.5, 2.25, 3.0, 3.5],
                                                     "stacked_norm_sq": 12.5})
    rng = np.random.default_rng(5)
    saddle = SaddlePoint(x_star=rng.standard_normal((24, 24)),
                         y_star=[rng.standard_normal((16, 32)) for _ in range(4)],
                         source="cg", converged=True, residual=3.25e-9)
    rio.save_saddle(io_dir / "saddle", saddle, meta={"alpha": 0.01, "iterations": 41})
    rec = rio.ConvergenceRecord()
    for k in range(1, 13):
        rec.append(k, 0.7 ** k * (1.0 + 0.01 * math.sin(k)), 10.0 / k, float("nan") if k == 3
                   else 0.1 / k, 4 * k, 4 * k)
    rec.write_csv(io_dir / "record.csv")
    fit = rio.fit_rate(rec)
    out["fit_rate"] = np.array([fit.rate, fit.log_intercept, fit.r_squared, *fit.epoch_window])
    fit2 = rio.fit_rate(rec, window=(2.0, 9.0))
    out["fit_rate_window"] = np.array([fit2.rate, fit2.log_intercept, fit2.r_squared,
                                       *fit2.epoch_window])
    rio.write_pgm16(io_dir / "image.pgm", rng.standard_normal((7, 5)))
    rio.write_pgm16(io_dir / "flat.pgm", np.full((3, 4), 2.5))
    np.savez_compressed(HERE / "datasets.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["projector", "warps", "sampling", "tiny", "c1", "datasets",
                             "divergence"]
    for w in which:
        t0 = time.time()
        {"projector": projector_cases, "warps": warp_cases, "sampling": sampling_cases,
         "tiny": solver_tiny, "c1": solver_c1, "datasets": dataset_cases,
         "divergence": divergence_cases}[w]()
        print(f"{w}: {time.time() - t0:.1f}s", flush=True)
