"""Data generation and file formats.

CPU tier: phantoms and the host noise stream against the reference's outputs
(golden ``datasets.npz``); the on-disk formats against files the reference's own
experiment_io wrote (``golden/io``): we read them, and what we write is
byte-identical.  GPU tier: the device noise kernel and ``generate`` against the
same goldens (mirrors test_simulate.py / test_experiment_io.py of the reference).
"""

import filecmp
import math

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

from paper_2410_10503_b200 import experiment_io as eio
from paper_2410_10503_b200 import simulate as sim
from paper_2410_10503_b200.motion import MotionParams, motion_sequence
from paper_2410_10503_b200.projector import Geometry

IO = GOLDEN / "io"
TINY = Geometry(24, 24, 16, 32, math.hypot(24, 24) / 32)


@pytest.fixture(scope="module")
def G():
    return load_golden("datasets")


# --------------------------------------------------------------- CPU tier
@pytest.mark.parametrize("kind", sim.PHANTOM_KINDS)
@pytest.mark.parametrize("shape", [(48, 40), (64, 64), (17, 33)])
def test_phantoms_bit_exact(G, kind, shape):
    assert np.array_equal(sim.make_phantom(kind, *shape), G[f"phantom_{kind}_{shape[0]}x{shape[1]}"])


def test_phantom_validation():
    with pytest.raises(ValueError):
        sim.make_phantom("cube", 64, 64)
    with pytest.raises(ValueError):
        sim.make_phantom("thorax", 15, 64)
    with pytest.raises(ValueError):
        sim.make_phantom("thorax", 64, 15)


@pytest.mark.parametrize("name,shape,seed,gate", [
    ("f_5x7", (5, 7), 1234, 3), ("f_odd", (1, 13), 7, 0), ("f_one", (1, 1), 9, 2),
    ("f_big", (128, 129), (1 << 64) + 5, 11)])
def test_host_noise_stream_bit_exact(G, name, shape, seed, gate):
    assert np.array_equal(sim.gaussian_field(shape, seed, gate), G[name])


def test_noise_model_and_dataset_validation():
    with pytest.raises(ValueError):
        sim.NoiseModel(-1.0)
    with pytest.raises(ValueError):
        sim.NoiseModel(float("inf"))
    truth = np.zeros(TINY.image_shape)
    ident = [MotionParams.identity(), MotionParams(kind="rigid", rotation=0.1)]
    sinos = [np.zeros(TINY.sino_shape)] * 2
    ds = sim.GatedDataset(TINY, truth, ident, sinos, 0.0, 0)
    assert ds.num_gates == 2
    with pytest.raises(ValueError):
        sim.GatedDataset(TINY, truth, [], [], 0.0, 0)
    with pytest.raises(ValueError):
        sim.GatedDataset(TINY, truth, ident, sinos[:1], 0.0, 0)
    with pytest.raises(ValueError):
        sim.GatedDataset(TINY, truth, ident[::-1], sinos, 0.0, 0)
    with pytest.raises(ValueError):
        sim.GatedDataset(TINY, truth, ident, [np.zeros((3, 3))] * 2, 0.0, 0)


def test_read_reference_dataset_and_rewrite_byte_identical(tmp_path):
    ds, man = eio.load_dataset(IO / "dataset")
    assert ds.num_gates == 4 and ds.geometry == TINY
    assert ds.phantom_kind == "nested_shells" and ds.magnitude == 0.6
    assert man["norms"]["stacked_norm_sq"] == 12.5
    assert np.array_equal(ds.truth, sim.make_phantom("nested_shells", 24, 24))
    eio.save_dataset(ds, tmp_path / "d", norms=man["norms"])
    names = sorted(p.name for p in (IO / "dataset").iterdir())
    assert sorted(p.name for p in (tmp_path / "d").iterdir()) == names
    match, mismatch, errors = filecmp.cmpfiles(IO / "dataset", tmp_path / "d", names,
                                               shallow=False)
    assert not mismatch and not errors, mismatch


def test_read_reference_saddle_and_rewrite_byte_identical(tmp_path):
    sp = eio.load_saddle(IO / "saddle")
    assert sp.source == "cg" and sp.converged and sp.residual == 3.25e-9
    assert len(sp.y_star) == 4 and sp.x_star.shape == (24, 24)
    eio.save_saddle(tmp_path / "s", sp, meta={"alpha": 0.01, "iterations": 41})
    names = sorted(p.name for p in (IO / "saddle").iterdir())
    _, mismatch, errors = filecmp.cmpfiles(IO / "saddle", tmp_path / "s", names, shallow=False)
    assert not mismatch and not errors, mismatch


def test_convergence_csv_and_fit_rate(G, tmp_path):
    rec = eio.ConvergenceRecord.read_csv(IO / "record.csv")
    assert len(rec) == 12 and math.isnan(rec.rmse_to_truth[2])
    rec.write_csv(tmp_path / "r.csv")
    assert (tmp_path / "r.csv").read_bytes() == (IO / "record.csv").read_bytes()
    for window, key in (((5.0, None), "fit_rate"), ((2.0, 9.0), "fit_rate_window")):
        f = eio.fit_rate(rec, window=window)
        got = np.array([f.rate, f.log_intercept, f.r_squared, *f.epoch_window])
        assert np.array_equal(got, G[key]), key
    with pytest.raises(ValueError):
        eio.fit_rate(rec, window=(10.0, None))
    bad = eio.ConvergenceRecord()
    for k in range(1, 8):
        bad.append(k, 0.0 if k == 6 else 1.0 / k, 1.0, 0.0, k, k)
    with pytest.raises(ValueError):
        eio.fit_rate(bad, window=(1.0, None))


def test_pgm_byte_identical(tmp_path):
    rng = np.random.default_rng(5)  # make_golden's draws: saddle x*, 4 y*, then the image
    rng.standard_normal((24, 24))
    for _ in range(4):
        rng.standard_normal((16, 32))
    eio.write_pgm16(tmp_path / "image.pgm", rng.standard_normal((7, 5)))
    eio.write_pgm16(tmp_path / "flat.pgm", np.full((3, 4), 2.5))
    for name in ("image.pgm", "flat.pgm"):
        assert (tmp_path / name).read_bytes() == (IO / name).read_bytes(), name


def test_raster_roundtrip_and_errors(tmp_path):
    a = np.random.default_rng(0).standard_normal((7, 3))
    eio.write_raster(tmp_path / "a.f64", a)
    assert np.array_equal(eio.read_raster(tmp_path / "a.f64"), a)
    blob = (tmp_path / "a.f64").read_bytes()
    cases = {"bad magic at byte 0": b"XXXX" + blob[4:],
             "bad shape line at byte 11": blob.replace(b"7 3\n", b"7 x\n"),
             "expected 168 payload bytes at byte 15": blob[:-8]}
    for msg, data in cases.items():
        (tmp_path / "b.f64").write_bytes(data)
        with pytest.raises(eio.RasterFormatError, match=msg):
            eio.read_raster(tmp_path / "b.f64")
    with pytest.raises(ValueError):
        eio.write_raster(tmp_path / "c.f64", np.zeros(3))
    geom = Geometry(8, 9, 10, 11, 0.5)
    assert eio.geometry_from_dict(eio.geometry_to_dict(geom)) == geom


# --------------------------------------------------------------- GPU tier
@pytest.mark.gpu
@pytest.mark.parametrize("name,shape,seed,gate", [
    ("f_5x7", (5, 7), 1234, 3), ("f_odd", (1, 13), 7, 0), ("f_one", (1, 1), 9, 2),
    ("f_big", (128, 129), (1 << 64) + 5, 11)])
def test_device_noise_matches_reference_stream(G, name, shape, seed, gate):
    dev = sim.gaussian_field_device(shape, seed, gate).cpu().numpy()
    ref = G[name]
    # uniforms are bit-identical; log1p / sincos are CUDA's fp64 (a few ulp)
    assert np.allclose(dev, ref, rtol=1e-14, atol=1e-14)
    assert np.mean(dev == ref) > 0.5


@pytest.mark.gpu
def test_device_noise_base_scale_and_fp32():
    import torch

    base = torch.randn(40, 50, device="cuda")
    out = sim.gaussian_field_device((40, 50), 3, 1, scale=0.25, base=base)
    ref = base.double().cpu().numpy() + 0.25 * sim.gaussian_field((40, 50), 3, 1)
    assert np.allclose(out.cpu().numpy(), ref, rtol=1e-14, atol=1e-14)
    o32 = sim.gaussian_field_device((40, 50), 3, 1, scale=0.25, base=base, dtype="float32")
    assert o32.dtype == torch.float32
    assert np.allclose(o32.cpu().numpy(), ref.astype(np.float32), rtol=1e-6, atol=1e-6)
    with pytest.raises(ValueError):
        sim.gaussian_field_device((4, 4), 0, -1)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["gen_rigid", "gen_rigid_clean", "gen_dil"])
def test_generate_matches_reference(G, case):
    ph, motion, noise, seed = {
        "gen_rigid": ("nested_shells", motion_sequence("rigid", 4, 0.6), None, 3),
        "gen_rigid_clean": ("nested_shells", motion_sequence("rigid", 4, 0.6),
                            sim.NoiseModel(0.0), 0),
        "gen_dil": ("thorax", motion_sequence("dilatation", 3, 0.8), sim.NoiseModel(0.4), 5),
    }[case]
    ds = sim.generate(sim.make_phantom(ph, 24, 24), motion, TINY, noise, master_seed=seed)
    got, ref = np.stack(ds.sinograms), G[f"{case}_sinos"]
    assert got.dtype == np.float64 and got.shape == ref.shape
    # fp32 device projector on fp32-rounded phantom vs the fp64 reference
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
    assert ds.sigma == pytest.approx(float(G[f"{case}_sigma"]), rel=1e-5)


@pytest.mark.gpu
def test_generate_validation_and_truth_copy():
    ph = sim.make_phantom("nested_shells", 24, 24)
    moved_first = [MotionParams(kind="rigid", translation=(1.0, 0.0)), MotionParams.identity()]
    with pytest.raises(ValueError):
        sim.generate(ph, moved_first, TINY)
    with pytest.raises(ValueError):
        sim.generate(ph, [], TINY)
    with pytest.raises(ValueError):
        sim.generate(np.zeros((8, 8)), motion_sequence("rigid", 2, 0.5), TINY)
    ds = sim.generate(ph, motion_sequence("rigid", 2, 0.5), TINY)
    ph[0, 0] = 123.0
    assert ds.truth[0, 0] != 123.0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["preset_rigid", "preset_nonrigid"])
def test_presets_match_reference(G, name):
    fn = sim.rigid_preset if name == "preset_rigid" else sim.nonrigid_preset
    ds = fn(size="fast", seed=1, magnitude=0.3)
    assert ds.num_gates == (20 if name == "preset_rigid" else 10)
    assert ds.geometry == Geometry.fast() and ds.motion[0].is_identity()
    assert np.array_equal(ds.truth, G[f"{name}_truth"])
    got, ref = np.stack(ds.sinograms[:3]), G[f"{name}_sinos"]
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
    assert ds.sigma == pytest.approx(float(G[f"{name}_sigma"]), rel=1e-5)
    with pytest.raises(ValueError):
        fn(size="huge")


@pytest.mark.gpu
def test_generated_dataset_roundtrips_through_files(tmp_path):
    ds = sim.rigid_preset(size="fast", sigma=0.0, magnitude=0.3)
    eio.save_dataset(ds, tmp_path / "d")
    back, _ = eio.load_dataset(tmp_path / "d")
    assert all(np.array_equal(a, b) for a, b in zip(ds.sinograms, back.sinograms))
    assert back.motion == ds.motion and back.sigma == ds.sigma
