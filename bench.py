#!/usr/bin/env python
"""Benchmark: PDHG / SPDHG epochs/s at 512^2 x 20 gates (BASELINE.json metric, config C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3] [--no-cpu-baseline]

A "step" is one epoch (one PDHG iteration over all gates) of the C3 workload:
512x512 fp32 random-ellipse phantom, 20 dense non-rigid gates, 720 angles x 729
unit-spaced bins, alpha = 5e-3.  ``value`` is PDHG epochs/s (gate-sharded over
the N ranks when N > 1 -- each rank owns 2*gates/N half-gate units -- strong
scaling of one problem); SPDHG epochs/s (an independent replica on every rank --
SPDHG of one problem does not shard -- aggregated over the ranks) is reported
beside it.  ``--gpus N`` with N > 1 starts the N ranks itself (torch.distributed.run,
one rank per visible GPU) unless it already runs under a launcher.

Timing: W warm-up epochs, then exactly K epochs bracketed by a barrier and a
device synchronize, CUDA events on the launching stream, max over ranks.  The
per-epoch working set (data + duals + workspace ~ 0.8 GB) exceeds the 126 MB L2,
so no explicit flush is needed (stated in ``config``).  ``e2e`` repeats the
measurement through the C-ABI with the step's inputs (the 20 gated sinograms)
copied host->device from pinned memory and the result x copied back every step
(uploads double-buffered on a copy stream, the read-back from a device snapshot on a
third stream, the epoch launched as the CUDA graph ``run()`` uses; ``value`` times eager
launches with a CUDA event between the kernels, which is about 1 % slower).

``--impl reference`` times the CPU restatement of the reference (oracle/, fp64 C,
all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SPDHG/PDHG epochs/s at 512²×20 gates; A_i+A_i^* achieved HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the torch.distributed gate-sharded path even for one rank "
                         "(exercises the multi-GPU code path on a single GPU)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="gate-sharded PDHG partial sum: fused NVLink peer-memory exchange "
                         "inside the z update (p2p) or NCCL allreduce + z update")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- clocks
REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------ e2e read-back
class ReadBack:
    """Device -> host read of every step's result x without stalling the next step:
    x is snapshotted on the compute stream (device copy, a few µs) and the D2H of the
    snapshot runs on its own stream into pinned memory, double-buffered; a snapshot
    buffer is rewritten only after its previous D2H finished."""

    def __init__(self, torch, x, stream):
        self.torch, self.stream = torch, stream
        self.stage = [torch.empty_like(x) for _ in range(2)]
        self.host = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for _ in range(2)]
        self.snap = [torch.cuda.Event(), torch.cuda.Event()]
        self.back = [torch.cuda.Event(), torch.cuda.Event()]
        self.s = torch.cuda.Stream()
        self.k = 0
        self.bytes = int(x.numel() * x.element_size())

    def read(self, x):
        b = self.k & 1
        if self.k >= 2:
            self.stream.wait_event(self.back[b])
        self.stage[b].copy_(x, non_blocking=True)
        self.snap[b].record(self.stream)
        with self.torch.cuda.stream(self.s):
            self.s.wait_event(self.snap[b])
            self.host[b].copy_(self.stage[b], non_blocking=True)
            self.back[b].record(self.s)
        self.k += 1

    def finish(self):
        self.stream.wait_stream(self.s)


# ------------------------------------------------------- algorithmic bytes
def alg_bytes(cfg):
    """SURVEY.md §8d SpMV-equivalent fp32 bytes (4 B per nonzero operand / output)."""
    n2 = cfg.n * cfg.n
    ab = cfg.num_angles * cfg.num_bins
    S = cfg.samples
    F = 2 * n2 if cfg.motion == "dense" else 0
    b_fwd_kernel = 4 * (2 * S + ab + 4 * ab)          # K2: 2S taps + out + dual epilogue
    b_adj_kernel = 4 * (2 * S + n2)                   # K3: 2S taps + out
    b_pair = 4 * (4 * n2 + n2 + 2 * S + ab + F) + 4 * (2 * S + n2 + 4 * n2 + n2 + F)
    b_elem = 4 * (7 * n2 + 4 * ab)
    b_min_pair = 4 * (2 * n2 + 2 * ab + 2 * F)
    return {"K2_forward_dual": b_fwd_kernel, "K3_adjoint": b_adj_kernel, "pair": b_pair,
            "elem": b_elem, "min_pair": b_min_pair, "S": S}


def joseph_samples_nz(cfg) -> int:
    """Joseph samples with a nonzero weight in one application of A (projector.py:
    134-166): per ray (a, j), the dominant-axis steps k whose continuous minor index
    cont_k = P*s_j + Q + k*slope lies in (-1, lim), i.e. with at least one tap inside
    the image.  Exact integer count from the reference's own angle / bin formulas."""
    n_r = n_c = cfg.n
    A, B = cfg.num_angles, cfg.num_bins
    ang = np.arange(A) * (math.pi / A)
    cs, sn = np.cos(ang), np.sin(ang)
    rdom = np.abs(cs) >= sn
    s = (np.arange(B) - (B - 1) / 2.0) * 1.0
    hr, hc = 0.5 * (n_r - 1), 0.5 * (n_c - 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        P = np.where(rdom, 1.0 / cs, -1.0 / sn)
        slope = np.where(rdom, sn / cs, cs / sn)
    Q = np.where(rdom, hc - hr * slope, hr - hc * slope)
    lim = np.where(rdom, n_c, n_r)[:, None].astype(np.float64)
    nmaj = np.where(rdom, n_r, n_c)[:, None]
    c0 = P[:, None] * s[None, :] + Q[:, None]
    sl = slope[:, None] * np.ones((1, B))
    flat = sl == 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        ka, kb = (-1.0 - c0) / sl, (lim - c0) / sl
    lo, hi = np.minimum(ka, kb), np.maximum(ka, kb)
    kmin = np.maximum(0, np.floor(lo) + 1)
    kmax = np.minimum(nmaj - 1, np.ceil(hi) - 1)
    cnt = np.where(flat, np.where((c0 > -1.0) & (c0 < lim), nmaj, 0),
                   np.clip(kmax - kmin + 1, 0, None))
    return int(cnt.sum())


def l1_operand_bytes(cfg):
    """Bytes the K2 / K3 gathers must deliver from L1 to registers per item (fp32):
    K2: one (value, forward difference) pair = 8 B per nonzero Joseph sample; K3: the
    (value, difference) pair of the bin under every pixel-angle tent = 8 B per
    pixel-angle (footprint 2 bins, spacing 1).  A gate pair fetches both items' 8 B in
    one 16-byte load: 512 B per warp request, 4 L1 wavefronts at the ideal."""
    return {"K2_forward_dual": 8 * joseph_samples_nz(cfg),
            "K3_adjoint": 8 * cfg.n * cfg.n * cfg.num_angles}


def l1_peak_gbs(sm_mhz):
    """L1 data-pipe peak: one 128-byte wavefront per SM per clock (B200: 148 SMs)
    at the SM clock sampled during the timed region.  tools/micro/l1_peak.cu measures
    the delivered fraction of it for contiguous 16-byte requests
    (profiles/l1_peak.json)."""
    sms = 148
    try:
        import torch

        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    except Exception:
        pass
    return 128.0 * sms * float(sm_mhz) * 1e6 / 1e9


FWD_IL = 2  # K2 lane interleave (paper_2410_10503_b200/csrc/mct_internal.cuh MCT_FWD_IL)


def pattern_cycles(cfg):
    """Mean L1 cost (SM cycles per 32-lane 16-byte request) of each gather's access
    pattern, from the measured cost-vs-lane-spacing curve (tools/micro/l1_pattern.cu,
    profiles/l1_pattern.json: 4 cycles while 8 consecutive lanes stay inside 128 bytes,
    i.e. spacing <= 1 element, rising to 8 cycles at spacing >= 1.2), averaged over the
    geometry's angles (equal weight per angle).  K2: consecutive bins sit sp/|cos|
    (rows-dominant) or sp/sin (cols-dominant) elements apart, FWD_IL lanes per bin;
    K3: the 32 columns of a warp map to bins |cos|/sp apart."""
    p = ROOT / "profiles" / "l1_pattern.json"
    if not p.exists():
        return None
    runs = json.loads(p.read_text())["runs"]
    xs = np.array([r["P"] for r in runs])
    ys = np.array([r["cycles_per_request"] for r in runs])
    th = np.arange(cfg.num_angles) * (np.pi / cfg.num_angles)
    c, s = np.abs(np.cos(th)), np.abs(np.sin(th))
    sp = 1.0  # BASELINE geometries: unit detector spacing
    p2 = np.where(c >= s, sp / np.maximum(c, 1e-12), sp / np.maximum(s, 1e-12))
    # K2 lanes interleave FWD_IL nearly parallel rays per bin (csrc MCT_FWD_IL): 8 lanes
    # span (8 / IL - 1) bin spacings, i.e. the microbenchmark's 8 lanes at spacing
    # (8 / IL - 1) * P / 7
    p2 = p2 * (8 / FWD_IL - 1) / 7
    p3 = c / sp
    f = lambda P: float(np.interp(np.minimum(P, xs[-1]), xs, ys).mean())
    return {"K2_forward_dual": f(p2), "K3_adjoint": f(p3)}


def roofline_line(cfg, kern_ms, items, traffic_all, wave_frac, sm_mhz, hbm_peak, peak_src):
    """The bench line's ``roofline``: the limiter that binds K2 / K3 is the L1 data
    pipe (ncu, profiles/ncu_traffic.json: data-pipe wavefronts 79 % / 90 % of peak on
    the 20-gate C3 launches, DRAM < 4 %), so the headline
    fraction is operand bytes delivered L1 -> registers (l1_operand_bytes, exact
    counts) over the data-pipe peak; the SURVEY §8d SpMV-equivalent HBM figure and
    the compulsory-bytes HBM fraction are kept as labelled secondary fields.
    ``kern_ms``: event time of each kernel summed over one step; ``items``: items
    (gate-slices) one step's launches process."""
    l1b = l1_operand_bytes(cfg)
    peak = l1_peak_gbs(sm_mhz)
    pat = pattern_cycles(cfg) or {}
    per = {}
    for k in ("K2_forward_dual", "K3_adjoint"):
        gbs = l1b[k] * items / (kern_ms[k] * 1e-3) / 1e9
        # the access pattern's own ceiling: 512 B per request every `cycles` SM clocks
        ppk = peak * 4.0 / pat[k] if k in pat else None
        per[k] = {"ms": kern_ms[k], "operand_bytes": l1b[k] * items, "achieved": gbs,
                  "frac": gbs / peak,
                  "pattern_cycles_per_request": pat.get(k),
                  "pattern_peak": ppk, "frac_of_pattern_peak": gbs / ppk if ppk else None,
                  "l1_wavefront_frac_ncu": (wave_frac or {}).get(k),
                  "dram_bytes_ncu": (traffic_all or {}).get(k)}
    dominant = max(per, key=lambda k: per[k]["ms"])
    ab = alg_bytes(cfg)
    spmv = ab[dominant] * items / (kern_ms[dominant] * 1e-3) / 1e9
    step_ms = sum(kern_ms.values())
    return {
        "bound": "l1_data_pipe", "kernel": dominant, "achieved": per[dominant]["achieved"],
        "peak": peak, "unit": "GB/s", "frac": per[dominant]["frac"],
        "traffic": per[dominant]["dram_bytes_ncu"],
        "peak_source": f"128 B/clk/SM L1 data pipe x SMs x {sm_mhz:.0f} MHz (sampled SM clock); "
                       "delivered fraction measured by tools/micro/l1_peak.cu "
                       "(profiles/l1_peak.json)",
        "bytes_model": "operand bytes L1 -> registers: 8 B (value, difference) per nonzero "
                       "Joseph sample (K2) / per pixel-angle tent (K3) per item",
        "kernels": per,
        "hbm": {"peak": hbm_peak, "peak_source": peak_src,
                "spmv_equivalent_gbs": spmv, "spmv_equivalent_frac": spmv / hbm_peak,
                "spmv_note": "SURVEY §8d algorithmic bytes (4 B per nonzero); taps are "
                             "served from L1, so this exceeds the HBM peak",
                "compulsory_frac": ab["min_pair"] * items / (step_ms * 1e-3) / 1e9 / hbm_peak,
                "dram_frac_ncu": (per[dominant]["dram_bytes_ncu"] / (kern_ms[dominant] * 1e-3)
                                  / 1e9 / hbm_peak) if per[dominant]["dram_bytes_ncu"] else None},
    }


TRAFFIC_ITEMS = 20  # items of the launch profiles/ncu_traffic.json was captured on


def load_traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return {}
    return {}


# ------------------------------------------------------------ reference arm
class CpuPort:
    """The reference algorithm's PDHG iteration restated in fp64 C (oracle/, all host
    threads): per gate A_i x, the dual prox, A_i^T dy; the primal prox once per epoch."""

    def __init__(self, cfg, threads):
        import oracle
        from oracle import solver as osolver
        from paper_2410_10503_b200 import workloads

        self.osolver = osolver
        inp = workloads.slice_inputs(cfg, 0)
        geom = oracle.Geometry(*cfg.geometry_args)
        self.ops = oracle.gate_operators(geom, inp.gates, threads=threads)
        rng = np.random.default_rng(0)
        self.data = [rng.standard_normal(geom.sino_shape) for _ in range(cfg.num_gates)]
        self.y = [np.zeros(geom.sino_shape) for _ in range(cfg.num_gates)]
        self.x = inp.phantom.astype(np.float64)
        self.z = np.zeros_like(self.x)
        self.cfg = cfg
        self.k = 0

    def gate_step(self):
        """One gate of a PDHG iteration (1/N of an epoch)."""
        o, n, i = self.osolver, self.cfg.num_gates, self.k % self.cfg.num_gates
        if i == 0:
            self.xn = o.prox_g(self.cfg.alpha, 1e-3, self.x - 1e-3 * self.z)
        proj = self.ops[i].apply(self.xn)
        y_new = o.prox_fstar(n, self.data[i], 1e-3, self.y[i] + 1e-3 * proj)
        self.z = self.z + self.ops[i].adjoint_apply(y_new - self.y[i])
        self.y[i] = y_new
        self.k += 1


def cpu_epoch_sample(cfg, threads, gates_sampled=None, cache={}):
    """Seconds per epoch of the CPU port: one whole PDHG epoch (every gate's A_i x,
    dual prox, A_i^T dy) timed, unless ``gates_sampled`` bounds the sample."""
    if gates_sampled is None:
        gates_sampled = cfg.num_gates
    port = cache.get((cfg.name, threads))
    if port is None:
        port = cache[(cfg.name, threads)] = CpuPort(cfg, threads)
        port.gate_step()  # warm
    t0 = time.perf_counter()
    for _ in range(gates_sampled):
        port.gate_step()
    return (time.perf_counter() - t0) / gates_sampled * cfg.num_gates


def run_reference(args, cfg):
    """The reference arm: the CPU port timed on this host, one gate-iteration per step."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    port = CpuPort(cfg, threads)
    steps = max(1, min(args.steps, 400))
    for _ in range(args.warmup):
        port.gate_step()
    t0 = time.perf_counter()
    for _ in range(steps):
        port.gate_step()
    t = time.perf_counter() - t0
    per_epoch = cfg.num_gates * cfg.batch  # gate-iterations in one (batch) epoch
    v = (steps / per_epoch) / t
    sample = (f"{steps} gate-iterations (A_i x, dual prox, A_i^T dy; = {steps / per_epoch:g} "
              f"epochs of {cfg.batch} slice(s)) of the fp64 C oracle port on {threads} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "epochs/s",
        "n_gpus": max(args.gpus, world), "steps": steps, "warmup": args.warmup,
        "ms_per_step": t / steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE C3 shapes)",
        "config": {"workload": f"{cfg.name}: {cfg.batch}x {cfg.n}^2, N={cfg.num_gates} "
                               f"{cfg.motion} gates, {cfg.num_angles}x{cfg.num_bins}, "
                               f"{'SPDHG batch' if cfg.batch > 1 else 'PDHG'}",
                   "step": "one gate-iteration (1/N epoch)"},
        "cpu_baseline": {"value": v, "unit": "epochs/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "epochs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def build_problem(cfg, torch):
    import paper_2410_10503_b200 as m
    from paper_2410_10503_b200 import workloads

    problem, truth, inp = m.simulate.workload_problem(cfg, 0)
    # step sizes: device power iterations feed the reference's default_config rule
    norms = [m.power_method(op, iterations=20, seed=0) for op in problem.operators]
    stacked = m.stacked_norm_sq(problem.operators, iterations=20, seed=0)
    return problem, norms, stacked


def event_time(torch, fn, stream):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    fn()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2410_10503_b200 as m
    from paper_2410_10503_b200 import _lib
    from paper_2410_10503_b200.distributed import ShardedPDHG
    from paper_2410_10503_b200.engine import Engine, KernelTimer

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    m.build_native()
    problem, norms, stacked = build_problem(cfg, torch)
    pcfg = m.default_config("pdhg", norms, cfg.alpha, args.steps, stacked_norm_sq=stacked)
    scfg = m.default_config("spdhg", norms, cfg.alpha, args.steps, seed=0)
    stream = torch.cuda.current_stream()

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if not use_dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- PDHG (gate-sharded across ranks) -------------------
    # The timed region launches the four fused kernels of every epoch eagerly
    # with a CUDA event between consecutive kernels on the launching stream, so
    # the per-kernel durations used by the roofline come from the timed region
    # itself (at C3 the GPU runs ~3 ms behind the host: launches never starve it).
    import ctypes

    L = _lib.load()
    exchange = None
    if not use_dist:
        eng = Engine([problem.operators], [problem.data])
        worker = None
    else:
        exchange = args.exchange
        try:
            worker = ShardedPDHG(pcfg, problem, rank, world, exchange=exchange)
        except Exception as exc:  # no symmetric-memory / P2P support on this box
            if exchange != "p2p":
                raise
            print(json.dumps({"warning": f"p2p exchange unavailable ({exc}); using nccl"}),
                  file=sys.stderr)
            exchange = "nccl"
            worker = ShardedPDHG(pcfg, problem, rank, world, exchange=exchange)
        eng = worker.engine
    eng.set_params(pcfg)
    eng.reset()
    items = eng.items_pdhg(epoch_ctr=True)
    names = ["K1_prox_warp", "K2_forward_dual", "K3_adjoint", "K4_adjoint_update"]
    chunks = eng.chunks(eng.local * eng.S, items.last_part)

    def step_fn(timer=None):
        # K1 -> K2 -> K3 per chunk of the workspace's pair ring (one chunk up to ~256 MB
        # of pair regions: C3 runs unchunked), then K4 over every item
        dz = worker.partial_buffer() if use_dist else None
        eng.iteration(items, problem.alpha, dz=dz, mark=timer)
        if use_dist:
            worker.reduce_update(dz)
        eng.advance_epoch()

    n_items = eng.local * eng.S
    # K2 / K3 run one launch for each chunk's gate pairs and one for an odd last item
    n_pairs = (n_items - (1 if eng.half is not None else 0)) // 2 * 2  # a half item is unpaired
    tail = int(n_items > n_pairs)
    n_chunks = len(chunks) if n_pairs > 0 else 0
    launches_per_step = (max(n_chunks, 1) + 2 * (n_chunks + tail) + 2 +
                         ((2 if exchange == "p2p" else 1) if use_dist else 0))
    for _ in range(args.warmup):
        step_fn()
    if use_dist and exchange == "p2p" and worker.p2p_failed_anywhere():
        # a peer wait timed out on some rank during warm-up: every rank switches
        print(json.dumps({"warning": "p2p exchange timed out in warm-up; using nccl"}),
              file=sys.stderr)
        worker.fallback_to_nccl()
        exchange = "nccl"
        for _ in range(args.warmup):
            step_fn()
    hbm_peak, peak_src = peaks()
    step_timers = [KernelTimer(torch, stream) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clocks:
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" selects it
        start.record(stream)
        for k in range(args.steps):
            step_fn(step_timers[k])
        end.record(stream)
        torch.cuda.nvtx.range_pop()
        barrier()
    ms_total = max_over_ranks(start.elapsed_time(end))
    if use_dist:
        worker.check()  # a timed-out peer wait raises instead of reporting a number
    primal, dual = eng.read_status()
    if primal is not None or dual is not None:
        print(json.dumps({"warning": "non-finite iterate during the timed run",
                          "primal": primal, "dual": dual}), file=sys.stderr)
    ms_step = ms_total / args.steps
    value = 1000.0 / ms_step
    # per kernel, summed over the chunks of a step (engine.KernelTimer)
    per_step = np.array([t.times_ms() for t in step_timers])
    kern = {n: float(per_step[:, i].mean()) for i, n in enumerate(names)}
    items_per_launch = eng.local * eng.S
    ab = alg_bytes(cfg)
    iter_ms = sum(kern.values())
    dominant = max(("K2_forward_dual", "K3_adjoint"), key=lambda k: kern[k])
    tr = load_traffic()
    # ncu DRAM bytes / wavefront fractions were captured on the 20-item C3 launch
    traffic_all = ({k: v * items_per_launch / TRAFFIC_ITEMS for k, v in tr.items()
                    if k.startswith("K")} if cfg.name == "c3" else None)
    wave_frac = tr.get("l1_data_pipe_frac") if cfg.name == "c3" else None
    traffic = tr.get(dominant) if cfg.name == "c3" else None
    l1_frac = (tr.get("l1_data_pipe_frac") or {}).get(dominant) if cfg.name == "c3" else None
    clk_mhz = clocks.summary()["sm_mhz"] or clocks.max_mhz or 1965.0
    if traffic is not None:  # captured on the 20-item C3 launch: scale to this launch
        traffic = traffic * items_per_launch / TRAFFIC_ITEMS
    ws_mb = (eng.ws.numel() + 4 * (eng.y.numel() + eng.d.numel() + 4 * eng.x.numel())) / 1e6
    achieved = ab[dominant] * items_per_launch / (kern[dominant] * 1e-3) / 1e9
    pair_gbs = ab["pair"] * items_per_launch / (iter_ms * 1e-3) / 1e9
    min_gbs = ab["min_pair"] * items_per_launch / (iter_ms * 1e-3) / 1e9

    # ---------------- SPDHG (replica per rank) -----------------------------
    # SPDHG of one problem does not shard (one gate per iteration): every rank runs
    # an independent replica of the whole problem; whole-job throughput is
    # world * K epochs over the slowest rank's device time.
    seng = Engine([problem.operators], [problem.data])
    seng.set_params(scfg)
    seng.reset()
    seng.set_sequences(m.draw_sequence(scfg, (args.steps + args.warmup) * cfg.num_gates)[None])
    sgraph = seng.epoch_graph("spdhg", problem.alpha)
    for _ in range(args.warmup):
        sgraph.replay()
    barrier()
    s_ms = max_over_ranks(event_time(torch, lambda: [sgraph.replay() for _ in range(args.steps)],
                                     stream))
    spdhg = {"value": 1000.0 * args.steps * world / s_ms, "unit": "epochs/s",
             "replicas": world, "per_replica": 1000.0 * args.steps / s_ms,
             "ms_per_epoch": s_ms / args.steps,
             "gpu_launches_per_epoch": 4 * cfg.num_gates + 1}
    del seng, sgraph

    # ---------------- e2e through the C-ABI with host buffers ---------------
    e2e = None
    if not args.no_e2e:
        # Every step streams that step's 20 gated sinograms host -> device (pinned)
        # and reads x back.  The H2D of step k+1 runs on a copy stream into the
        # second of two device data buffers while step k computes on the first.
        # (gate-sharded: each rank uploads only its own gates' sinograms)
        glo, ghi = (worker.data_lo, worker.data_hi) if use_dist else (0, cfg.num_gates)
        host_d = torch.from_numpy(np.stack([np.asarray(d, dtype=np.float32)
                                            for d in problem.data[glo:ghi]])[None]).pin_memory()
        back = ReadBack(torch, eng.x, stream)
        d_bufs = [eng.d, torch.empty_like(eng.d)]
        runners = []
        for b in range(2):
            eng.set_data_buffer(d_bufs[b])
            if not use_dist:
                runners.append(eng.epoch_graph("pdhg", problem.alpha).replay)
            else:
                runners.append(step_fn)
        eng.set_data_buffer(d_bufs[0])
        eng.set_data_buffer(d_bufs[0])
        copy_s = torch.cuda.Stream()
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        ev_copied = [torch.cuda.Event(), torch.cuda.Event()]

        def e2e_run(K):
            with torch.cuda.stream(copy_s):
                copy_s.wait_stream(stream)
                d_bufs[0][:, glo:ghi].copy_(host_d, non_blocking=True)
                ev_copied[0].record(copy_s)
            for k in range(K):
                b = k & 1
                stream.wait_event(ev_copied[b])
                if use_dist:
                    eng.set_data_buffer(d_bufs[b])
                runners[b]()
                ev_done[b].record(stream)
                back.read(eng.x)                          # the step's result, D2H
                if k + 1 < K:
                    nb = 1 - b
                    with torch.cuda.stream(copy_s):
                        if k >= 1:
                            copy_s.wait_event(ev_done[nb])  # step k-1 has read buffer nb
                        d_bufs[nb][:, glo:ghi].copy_(host_d, non_blocking=True)
                        ev_copied[nb].record(copy_s)
            stream.wait_stream(copy_s)
            back.finish()

        e2e_run(2)
        barrier()
        e_ms = max_over_ranks(event_time(torch, lambda: e2e_run(args.steps), stream)) / args.steps
        eng.set_data_buffer(d_bufs[0])
        e2e = {"value": 1000.0 / e_ms, "unit": "epochs/s",
               # whole job: every gate's sinogram once, x read back on every rank
               "h2d_bytes_per_step": int(cfg.num_gates * cfg.num_angles * cfg.num_bins * 4),
               "d2h_bytes_per_step": back.bytes * world,
               "overlap": "H2D of step k+1 (copy stream, double-buffered) overlaps step k; the "
                          "D2H of x reads a device snapshot on a third stream",
               "launch": ("one CUDA graph per epoch, as run() launches it (`value` times eager "
                          "launches with a CUDA event between the kernels, about 1 % slower)"
                          if not use_dist else "eager launches (gate-sharded step)")}

    # ---------------- CPU baseline (rank 0, N=1) ----------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        t = cpu_epoch_sample(cfg, threads)
        cpu = {"value": 1.0 / t, "unit": "epochs/s", "cores": threads, "kind": "port",
               "sample": f"one whole PDHG epoch ({cfg.num_gates} gate-iterations) of the fp64 "
                         f"C oracle port on {threads} threads (after one warm gate-iteration)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "epochs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded ellipse phantom, Gaussian-bump dense fields, Philox noise)",
            "config": {"workload": f"{cfg.name}: {cfg.n}^2 fp32, N={cfg.num_gates} dense gates "
                                   f"(peak {cfg.peak} px), {cfg.num_angles}x{cfg.num_bins} bins, "
                                   f"alpha={cfg.alpha}, PDHG gate-sharded over {world} GPU(s)",
                       "mode": "pdhg", "parallelism": f"gate-shard x{world}",
                       "exchange": (exchange if use_dist else "none (single process)"),
                       "l2": f"per-epoch working set {ws_mb:.0f} MB (workspace + state) > "
                             f"126 MB L2: no flush needed"},
            "roofline": roofline_line(cfg, kern, items_per_launch, traffic_all, wave_frac,
                                      clk_mhz, hbm_peak, peak_src),
            "roofline_pair": {"achieved_alg_gbs": pair_gbs, "frac_alg": pair_gbs / hbm_peak,
                              "achieved_min_gbs": min_gbs, "frac_min": min_gbs / hbm_peak,
                              "joseph_samples_per_s": 2 * ab["S"] * items_per_launch /
                              (iter_ms * 1e-3)},
            "kernel_ms": kern,
            "spdhg": spdhg,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches_per_step * args.steps,
            "device_memory": device_memory(torch),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def device_memory(torch):
    """Peak device memory of this process (torch's allocator: the engine's data,
    duals, state and workspace all live there)."""
    return {"peak_allocated_bytes": int(torch.cuda.max_memory_allocated()),
            "peak_reserved_bytes": int(torch.cuda.max_memory_reserved())}


def run_batch_ours(args, cfg):
    """C5: a batch of independent slices, SPDHG, slices partitioned over the ranks
    (distributed.slice_shard, no data-path collective).  A step is
    one epoch of the whole batch; value = batch epochs/s (max over ranks)."""
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2410_10503_b200 as m
    from paper_2410_10503_b200 import _lib
    from paper_2410_10503_b200.distributed import slice_shard
    from paper_2410_10503_b200.engine import Engine, KernelTimer

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    m.build_native()
    lo, hi = slice_shard(cfg.batch, world, rank)
    if hi <= lo:
        raise SystemExit("more ranks than slices")
    probs = [m.simulate.workload_problem(cfg, s)[0] for s in range(lo, hi)]
    # one step-size rule for every slice: slice 0's norms x 1.1 (admissible for all)
    base = probs[0] if lo == 0 else m.simulate.workload_problem(cfg, 0)[0]
    norms = [1.1 * m.power_method(op, iterations=20, seed=0) for op in base.operators]
    cfgs = [m.default_config("spdhg", norms, cfg.alpha, args.steps, seed=cfg.seed + s)
            for s in range(lo, hi)]
    S = hi - lo
    eng = Engine([p.operators for p in probs], [p.data for p in probs], max_items=S)
    eng.set_params(cfgs[0])
    eng.reset()
    eng.set_sequences(np.stack([m.draw_sequence(c, (args.steps + args.warmup + 2) *
                                                c.num_gates) for c in cfgs]))
    stream = torch.cuda.current_stream()

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if not use_dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # per-kernel share: one eager epoch with events between the launches
    names = ["K1_prox_warp", "K2_forward_dual", "K3_adjoint", "K4_adjoint_update"]
    timers = [KernelTimer(torch, stream) for _ in range(cfg.num_gates)]
    for k in range(cfg.num_gates):
        eng.iteration(eng.items_spdhg(k), cfg.alpha, mark=timers[k])
    eng.advance_epoch()
    torch.cuda.synchronize()
    per_iter = np.array([t.times_ms() for t in timers])
    kern = {n_: float(per_iter[:, i].sum()) for i, n_ in enumerate(names)}
    chunks = eng.chunks(S, 0)
    eng.reset()
    g = eng.epoch_graph("spdhg", cfg.alpha)
    for _ in range(args.warmup):
        g.replay()
    hbm_peak, peak_src = peaks()
    barrier()
    with ClockSampler(local) as clocks:
        ms = event_time(torch, lambda: [g.replay() for _ in range(args.steps)], stream)
        barrier()
    ms_total = max_over_ranks(ms)
    primal, dual = eng.read_status()
    if primal is not None or dual is not None:
        print(json.dumps({"warning": "non-finite iterate during the timed run",
                          "primal": primal, "dual": dual}), file=sys.stderr)
    ms_step = ms_total / args.steps
    value = 1000.0 / ms_step
    ab = alg_bytes(cfg)
    dominant = max(("K2_forward_dual", "K3_adjoint"), key=lambda k: kern[k])
    # kern[*] sums one epoch: num_gates launches, each over the S local slices
    achieved = ab[dominant] * S * cfg.num_gates / (kern[dominant] * 1e-3) / 1e9
    traffic = None  # the committed ncu traffic capture is of the C3 20-gate launch
    l1_frac = None
    clk_mhz = clocks.summary()["sm_mhz"] or clocks.max_mhz or 1965.0
    pair_gbs = ab["pair"] * cfg.batch * cfg.num_gates / (ms_step * 1e-3) / 1e9

    # e2e: every step uploads the local slices' sinograms from pinned host memory
    # and reads x back; the upload of step k+1 runs on a copy stream into the
    # second of two device data buffers while step k computes on the first
    e2e = None
    if not args.no_e2e:
        host_d = eng.d.cpu().pin_memory()
        back = ReadBack(torch, eng.x, stream)
        d_bufs = [eng.d, torch.empty_like(eng.d)]
        graphs = []
        for b in range(2):
            eng.set_data_buffer(d_bufs[b])
            graphs.append(eng.epoch_graph("spdhg", cfg.alpha))
        copy_s = torch.cuda.Stream()
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        ev_copied = [torch.cuda.Event(), torch.cuda.Event()]

        def e2e_run(K):
            with torch.cuda.stream(copy_s):
                copy_s.wait_stream(stream)
                d_bufs[0].copy_(host_d, non_blocking=True)
                ev_copied[0].record(copy_s)
            for k in range(K):
                b = k & 1
                stream.wait_event(ev_copied[b])
                graphs[b].replay()
                ev_done[b].record(stream)
                back.read(eng.x)
                if k + 1 < K:
                    nb = 1 - b
                    with torch.cuda.stream(copy_s):
                        if k >= 1:
                            copy_s.wait_event(ev_done[nb])  # step k-1 has read buffer nb
                        d_bufs[nb].copy_(host_d, non_blocking=True)
                        ev_copied[nb].record(copy_s)
            stream.wait_stream(copy_s)
            back.finish()

        eng.reset()  # epoch counter back to 0: the drawn gate sequences cover warmup + steps
        e2e_run(1)
        eng.reset()
        barrier()
        e_ms = max_over_ranks(event_time(torch, lambda: e2e_run(args.steps), stream)) / args.steps
        eng.set_data_buffer(d_bufs[0])
        e2e = {"value": 1000.0 / e_ms, "unit": "epochs/s",
               "h2d_bytes_per_step": int(host_d.numel() * 4) * world,
               "d2h_bytes_per_step": back.bytes * world,
               "overlap": "H2D of step k+1 (copy stream, double-buffered) overlaps step k; the "
                          "D2H of x reads a device snapshot on a third stream"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        t = cpu_epoch_sample(cfg, threads) * cfg.batch
        cpu = {"value": 1.0 / t, "unit": "epochs/s", "cores": threads, "kind": "port",
               "sample": f"one whole epoch of one slice ({cfg.num_gates} gate-iterations, fp64 "
                         f"C oracle port, {threads} threads), scaled x{cfg.batch} slices"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "epochs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded ellipse phantoms, Gaussian-bump dense fields, Philox noise)",
            "config": {"workload": f"{cfg.name}: batch of {cfg.batch} slices {cfg.n}^2 fp32, "
                                   f"N={cfg.num_gates} dense gates (peak {cfg.peak} px), "
                                   f"{cfg.num_angles}x{cfg.num_bins} bins, alpha={cfg.alpha}, "
                                   f"SPDHG per-slice seeds, slices partitioned over {world} "
                                   f"GPU(s)", "mode": "spdhg-batch",
                       "parallelism": f"slice-shard x{world} (no collective)",
                       "l2": "per-epoch working set > 1 GB > 126 MB L2 (no flush needed)"},
            "roofline": roofline_line(cfg, kern, S * cfg.num_gates, None, None, clk_mhz,
                                      hbm_peak, peak_src),
            "roofline_pair": {"achieved_alg_gbs": pair_gbs, "frac_alg": pair_gbs / hbm_peak},
            "kernel_ms_per_epoch_rank0": kern,
            "e2e": e2e,
            "cpu_baseline": cpu,
            # per iteration: K1, K4 and K2 / K3 for the slice pairs (+ an odd last slice)
            # per iteration: K1 per chunk of the pair ring, K2 / K3 per chunk + an odd
            # slice's single-item launch, K4; plus one counter bump per epoch
            "gpu_launches": ((len(chunks) + 2 * ((len(chunks) if S >= 2 else 0) + S % 2) + 1)
                             * cfg.num_gates + 1) * args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args) -> int | None:
    """``--gpus N`` (N > 1) without a torch.distributed environment: start the N
    ranks here, one process per visible GPU, through torch.distributed.run (the same
    launch the driver uses), and return the launcher's exit code.  Returns None when
    this process is already a rank (WORLD_SIZE set) or N == 1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if args.gpus > have:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, "
                                   f"found {have}", "n_gpus": args.gpus}), flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    from paper_2410_10503_b200 import workloads

    if args.impl != "reference":
        rc = launch_ranks(args)
        if rc is not None:
            return rc

    cfg = workloads.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg.batch > 1:
        return run_batch_ours(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
