"""Device execution engine of the fused PDHG / SPDHG iteration.

One ``Engine`` owns, for S slices x N gates of one geometry:

* the C ``mct_family`` (ray plan + per-(slice, gate) warp descriptors + per-gate
  step parameters),
* the device state (x, x_next, z, zbar: (S, rows, cols); y, d, proj:
  (S, N, A, B); the divergence status words),
* the per-item workspace (padded warped image X / XT, padded dual increment
  DY, backprojection image), zeroed once so the kernels' pad regions read 0,
* the epoch counter and pre-drawn gate sequences, and the CUDA graphs that
  replay one epoch without host involvement.

An iteration is four launches (solvers.step, solvers.py:316-366):
K1 prox+warp+pack, K2 Joseph forward + dual prox, K3 transpose-gather A^*,
K4 warp adjoint + z / zbar / x update.  PDHG processes every (local) gate as
one batch of items; SPDHG processes one drawn gate per slice.
"""

from __future__ import annotations

import ctypes
import math
from typing import Sequence

import numpy as np

from . import _lib
from .linops import ComposedMap, LinearMap
from .motion import WarpBase
from .projector import GatedOperator, RayTransform

U64_MAX_AS_I64 = -1  # 0xFFFF_FFFF_FFFF_FFFF viewed as int64


def split_operator(op: LinearMap):
    """(RayTransform, warp or None) for a gated operator of this package."""
    if isinstance(op, RayTransform):
        return op, None
    if isinstance(op, (GatedOperator, ComposedMap)) and isinstance(op.outer, RayTransform) \
            and isinstance(op.inner, WarpBase):
        w = op.inner
        return op.outer, (None if w.is_identity_warp else w)
    raise TypeError(
        "the fused solver needs gated operators of this package: RayTransform or "
        f"compose(RayTransform, WarpOperator/DenseWarpOperator); got {type(op).__name__}")


class Family:
    """Owner of a C ``mct_family`` (ray plan + S x N warp plans)."""

    def __init__(self, ray: RayTransform, warps: Sequence[Sequence[WarpBase | None]]):
        _lib.require_cuda()
        L = _lib.load()
        self.ray = ray
        self.S = len(warps)
        self.N = len(warps[0])
        self._warps = [list(w) for w in warps]
        arr = (ctypes.c_void_p * (self.S * self.N))()
        for s, row in enumerate(self._warps):
            if len(row) != self.N:
                raise ValueError("every slice needs the same number of gates")
            for g, w in enumerate(row):
                if w is not None and not w.is_identity_warp:
                    if tuple(w.domain_shape) != tuple(ray.domain_shape):
                        raise ValueError("warp shape does not match the ray geometry")
                    arr[s * self.N + g] = w.plan().handle.value
        h = ctypes.c_void_p()
        _lib.check(L.mct_family_create(ctypes.byref(h), ray.plan().handle, self.S, self.N, arr))
        self.handle = h
        self.item_bytes = ray.plan().item_bytes

    def set_params(self, sigmas, probs, theta):
        s = np.ascontiguousarray(sigmas, dtype=np.float64)
        p = np.ascontiguousarray(probs, dtype=np.float64)
        if s.shape != (self.N,) or p.shape != (self.N,):
            raise ValueError("one sigma and one probability per gate required")
        _lib.check(_lib.load().mct_family_set_params(self.handle, s.ctypes.data, p.ctypes.data,
                                                     float(theta)))

    def __del__(self):
        try:
            if self.handle:
                _lib.load().mct_family_destroy(self.handle)
        except Exception:
            pass


def chunk_plan(n: int, last_part: int, chunk_items: int):
    """(first_item, item_count) of the K1-K3 chunks of an n-item launch through a
    workspace whose pair ring holds ``chunk_items`` items (mct_family_chunk_items):
    whole gate pairs, at most ``chunk_items`` per chunk; the unpaired tail (an odd or
    half last item) rides with the last chunk (item_count 0 = to the end)."""
    paired = (n - 1 if last_part else n) & ~1
    c = int(chunk_items)
    if paired <= c:
        return [(0, 0)]
    if c < 2 or c % 2:
        raise ValueError("a chunk holds whole gate pairs: chunk_items must be even and >= 2")
    return [(f, c if f + c < paired else 0) for f in range(0, paired, c)]


class KernelTimer:
    """CUDA-event marks between the kernels of ``Engine.iteration`` (measurement only):
    ``times_ms()`` sums, per kernel K1..K4, the event time from each of its marks to the
    next mark (a chunked launch marks K1-K3 once per chunk)."""

    def __init__(self, torch, stream=None):
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.marks = []

    def __call__(self, index: int):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        self.marks.append((index, ev))

    def times_ms(self):
        out = [0.0, 0.0, 0.0, 0.0]
        for (i, a), (_, b) in zip(self.marks, self.marks[1:]):
            if i < 4:
                out[i] += a.elapsed_time(b)
        return out

    def launches(self):
        """Marks per kernel (the K1-K3 chunk count shows up here)."""
        return [sum(1 for i, _ in self.marks if i == k) for k in range(4)]


class Engine:
    """Fused-iteration executor for S slices sharing one geometry and gate count."""

    def __init__(self, operators_per_slice: Sequence[Sequence[LinearMap]],
                 data_per_slice: Sequence[Sequence[np.ndarray]], *, keep_projections=False,
                 gate_range: tuple[int, int] | None = None, max_items: int | None = None,
                 half: tuple[int, int] | None = None):
        torch = _lib.require_cuda()
        self.torch = torch
        rays, warps = [], []
        for ops in operators_per_slice:
            row = []
            for op in ops:
                r, w = split_operator(op)
                rays.append(r)
                row.append(w)
            warps.append(row)
        ray = rays[0]
        for r in rays[1:]:
            if r is not ray and r.geom != ray.geom:
                raise ValueError("all gated operators must share one geometry")
        self.ray = ray
        self.geom = ray.geom
        self.family = Family(ray, warps)
        self.S, self.N = self.family.S, self.family.N
        rows, cols = self.geom.image_shape
        A, B = self.geom.sino_shape
        self.n_img = rows * cols
        self.n_sino = A * B
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        f32 = torch.float32
        self.gate_lo, self.gate_hi = gate_range if gate_range is not None else (0, self.N)
        # half: (gate, part) -- one extra item covering the first (part 1) or second
        # (part 2) half of that gate's angle pairs (half-gate units of gate-sharded PDHG)
        self.half = None if half is None else (int(half[0]), int(half[1]))
        if self.half is not None:
            if self.half[1] not in (1, 2) or not 0 <= self.half[0] < self.N:
                raise ValueError("half must be (gate, 1 | 2)")
            if self.gate_lo <= self.half[0] < self.gate_hi:
                raise ValueError("the half gate may not also be a full local gate")
            if self.S != 1:
                raise ValueError("half-gate units need a single slice")
        self.local = self.gate_hi - self.gate_lo + (1 if self.half is not None else 0)
        # state
        self.x = torch.zeros((self.S, rows, cols), dtype=f32, device=dev)
        self.x_next = torch.zeros_like(self.x)
        self.z = torch.zeros_like(self.x)
        self.zbar = torch.zeros_like(self.x)
        self.y = torch.zeros((self.S, self.N, A, B), dtype=f32, device=dev)
        d = np.stack([np.stack([np.asarray(v, dtype=np.float32) for v in dl])
                      for dl in data_per_slice])
        if d.shape != (self.S, self.N, A, B):
            raise ValueError(f"data shape {d.shape} != {(self.S, self.N, A, B)}")
        self.d = torch.from_numpy(np.ascontiguousarray(d)).to(dev)
        self.proj = torch.zeros_like(self.y) if keep_projections else None
        self.status = torch.full((2,), U64_MAX_AS_I64, dtype=torch.int64, device=dev)
        self.dz = None
        items = max_items or max(self.S * self.local, self.S)
        self.max_items = items
        self.ws = torch.zeros(int(_lib.load().mct_family_workspace_bytes(self.family.handle, items)),
                              dtype=torch.uint8, device=dev)
        # launches with more gate pairs than the workspace's ring of pair regions run
        # K1 -> K2 -> K3 in chunks of this many items (mct_family_chunk_items)
        self.chunk_items = int(_lib.load().mct_family_chunk_items(self.family.handle, items))
        self.all_gates = torch.arange(self.N, dtype=torch.int32, device=dev)
        self.local_gates = (None if self.half is None else torch.tensor(
            list(range(self.gate_lo, self.gate_hi)) + [self.half[0]], dtype=torch.int32,
            device=dev))
        self.epoch_ctr = torch.zeros(1, dtype=torch.int32, device=dev)
        self.seq = None
        self._st = _lib.State()
        self._bind()
        self.graphs = {}

    # ------------------------------------------------------------------
    def _bind(self):
        st = self._st
        st.x = _lib.ptr(self.x)
        st.x_next = _lib.ptr(self.x_next)
        st.z = _lib.ptr(self.z)
        st.zbar = _lib.ptr(self.zbar)
        st.y = _lib.ptr(self.y)
        st.d = _lib.ptr(self.d)
        st.proj = _lib.ptr(self.proj) if self.proj is not None else None
        st.status = _lib.ptr(self.status)

    def set_params(self, config):
        self.family.set_params(config.sigmas, config.probs, config.theta)
        self.tau = float(config.tau)
        self.theta = float(config.theta)

    def reset(self):
        for t in (self.x, self.x_next, self.z, self.zbar, self.y):
            t.zero_()
        self.status.fill_(U64_MAX_AS_I64)
        self.epoch_ctr.zero_()

    # ---------------------------------------------------------------- items
    def items_pdhg(self, iteration: int = 1, epoch_ctr: bool = False) -> _lib.Items:
        it = _lib.Items()
        it.gates_dev = _lib.ptr(self.all_gates if self.half is None else self.local_gates)
        it.epoch_ctr_dev = _lib.ptr(self.epoch_ctr) if epoch_ctr else None
        it.slice_stride = 0
        it.epoch_stride = 0
        it.base = self.gate_lo if self.half is None else 0
        it.items_per_slice = self.local
        it.last_part = 0 if self.half is None else self.half[1]
        it.num_slices = self.S
        it.iteration = iteration
        it.iters_per_epoch = 1
        return it

    def items_subset(self, gates_dev, count: int, iteration: int) -> _lib.Items:
        it = _lib.Items()
        it.gates_dev = _lib.ptr(gates_dev)
        it.epoch_ctr_dev = None
        it.slice_stride = 0
        it.epoch_stride = 0
        it.base = 0
        it.items_per_slice = count
        it.num_slices = self.S
        it.iteration = iteration
        it.iters_per_epoch = 1
        return it

    def set_sequences(self, seqs: np.ndarray):
        """Pre-drawn SPDHG gate sequences, shape (S, total_iterations)."""
        seqs = np.ascontiguousarray(seqs, dtype=np.int32)
        if seqs.ndim != 2 or seqs.shape[0] != self.S:
            raise ValueError("one gate sequence per slice required")
        if seqs.size and (seqs.min() < 0 or seqs.max() >= self.N):
            raise ValueError("gate index out of range")
        new = self.torch.from_numpy(seqs).to(self.device)
        if self.seq is not None and tuple(self.seq.shape) == tuple(new.shape):
            self.seq.copy_(new)  # captured epoch graphs read the sequence in place
        else:
            self.seq = new
            self.graphs = {k: g for k, g in self.graphs.items() if k[0] != "spdhg"}
        self.total_iters = seqs.shape[1]

    def items_spdhg(self, k: int) -> _lib.Items:
        it = _lib.Items()
        it.gates_dev = _lib.ptr(self.seq)
        it.epoch_ctr_dev = _lib.ptr(self.epoch_ctr)
        it.slice_stride = self.total_iters
        it.epoch_stride = self.N
        it.base = k
        it.items_per_slice = 1
        it.num_slices = self.S
        it.iteration = k + 1
        it.iters_per_epoch = self.N
        return it

    # ------------------------------------------------------------ iteration
    def iteration(self, items: _lib.Items, alpha: float, dz=None, mark=None):
        """K1..K4 of one iteration on the current stream.  ``mark(i)`` (a
        ``KernelTimer``) is called before kernel i = 0..3 and ``mark(4)`` at the end."""
        L = _lib.load()
        fam = self.family.handle
        ws = _lib.ptr(self.ws)
        st = _lib.stream_handle()
        ip, sp = ctypes.byref(items), ctypes.byref(self._st)
        n = items.items_per_slice * items.num_slices
        for first, count in self.chunks(n, items.last_part):
            items.first_item, items.item_count = first, count
            if mark is not None:
                mark(0)
            _lib.check(L.mct_iter_prox_warp(fam, ip, sp, self.tau, float(alpha), ws, st))
            if mark is not None:
                mark(1)
            _lib.check(L.mct_iter_forward_dual(fam, ip, sp, ws, st))
            if mark is not None:
                mark(2)
            _lib.check(L.mct_iter_adjoint(fam, ip, ws, st))
        items.first_item = items.item_count = 0
        if mark is not None:
            mark(3)
        _lib.check(L.mct_iter_adjoint_update(fam, ip, sp, _lib.ptr(dz) if dz is not None else None,
                                             ws, st))
        if mark is not None:
            mark(4)

    def chunks(self, n: int, last_part: int = 0):
        """(first_item, item_count) of the K1-K3 chunks of an n-item launch."""
        return chunk_plan(n, last_part, self.chunk_items)

    def z_update(self, dz, theta: float):
        _lib.check(_lib.load().mct_iter_z_update(self.family.handle, ctypes.byref(self._st),
                                                 _lib.ptr(dz), float(theta), _lib.stream_handle()))

    def advance_epoch(self, inc: int = 1):
        _lib.check(_lib.load().mct_epoch_advance(_lib.ptr(self.epoch_ctr), inc,
                                                 _lib.stream_handle()))

    def epoch(self, mode: str, alpha: float):
        """One epoch, eagerly: 1 PDHG iteration or N SPDHG iterations."""
        if mode == "pdhg":
            self.iteration(self.items_pdhg(epoch_ctr=True), alpha)
        else:
            for k in range(self.N):
                self.iteration(self.items_spdhg(k), alpha)
        self.advance_epoch()

    def set_data_buffer(self, d):
        """Point the kernels at another (S, N, A, B) fp32 data buffer (double-buffered
        streaming of new sinograms while an epoch computes)."""
        if tuple(d.shape) != tuple(self.d.shape) or d.dtype != self.d.dtype or not d.is_cuda:
            raise ValueError("data buffer must match the engine's (S, N, A, B) fp32 layout")
        self.d = d
        self._bind()

    def epoch_graph(self, mode: str, alpha: float):
        """CUDA graph replaying one epoch (epoch counter advanced inside); one graph per
        (mode, alpha, tau, data buffer)."""
        key = (mode, float(alpha), self.tau, self.d.data_ptr(),
               self.seq.data_ptr() if mode == "spdhg" and self.seq is not None else 0)
        g = self.graphs.get(key)
        if g is None:
            torch = self.torch
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            # warm the kernels once outside capture on a scratch copy of the state
            g = torch.cuda.CUDAGraph()
            saved = self.snapshot()
            with torch.cuda.stream(s):
                self.epoch(mode, alpha)
            torch.cuda.current_stream().wait_stream(s)
            self.restore(saved)
            with torch.cuda.graph(g, stream=s):
                self.epoch(mode, alpha)
            self.graphs[key] = g
        return g

    def snapshot(self):
        ts = [self.x, self.x_next, self.z, self.zbar, self.y, self.status, self.epoch_ctr]
        if self.proj is not None:
            ts.append(self.proj)
        return [t.clone() for t in ts]

    def restore(self, saved):
        ts = [self.x, self.x_next, self.z, self.zbar, self.y, self.status, self.epoch_ctr]
        if self.proj is not None:
            ts.append(self.proj)
        for t, v in zip(ts, saved):
            t.copy_(v)

    # ---------------------------------------------------------- diagnostics
    def reduce(self, a, b, segments: int, length: int, mode: int, out=None, st=None):
        """Fixed-order fp64 reduction of ``segments`` runs of ``length`` (into ``out``).
        ``st``: the current stream's raw handle, when the caller already holds it."""
        if out is None:
            out = self.torch.empty(segments, dtype=self.torch.float64, device=self.device)
        if st is None:
            st = _lib.stream_handle()
        optr = out if isinstance(out, int) else _lib.ptr(out)  # a tensor or a raw device address
        _lib.check(_lib.load().mct_reduce(_lib.ptr(a), _lib.ptr(b) if b is not None else None,
                                          length, segments, length, mode, optr,
                                          _lib.ptr(_lib.scratch(self.device, segments, st)), st))
        return out

    def gated_forward(self, slice_index: int, gate: int, x, out):
        ws = self.ws  # item 0 scratch; callers run between iterations
        _lib.check(_lib.load().mct_gated_forward(self.family.handle, slice_index, gate,
                                                 _lib.ptr(x), _lib.ptr(out), _lib.ptr(ws),
                                                 _lib.stream_handle()))

    def gated_adjoint(self, slice_index: int, gate: int, y, out):
        _lib.check(_lib.load().mct_gated_adjoint(self.family.handle, slice_index, gate,
                                                 _lib.ptr(y), _lib.ptr(out), _lib.ptr(self.ws),
                                                 _lib.stream_handle()))

    def objective_parts(self, reuse_projections: bool, fit_out=None, xx_out=None, st=None):
        """Device fp64 parts of the objective, no host sync: ||A_i x - d_i||^2 per
        (slice, gate) and ||x||^2 per slice (written into ``fit_out`` / ``xx_out``)."""
        torch = self.torch
        if reuse_projections and self.proj is not None:
            proj = self.proj
        else:
            if getattr(self, "_proj_scratch", None) is None:
                self._proj_scratch = torch.empty_like(self.y)
            proj = self._proj_scratch
            if self.max_items >= self.N:  # all gates of a slice in one pass
                h = st if st is not None else _lib.stream_handle()
                for s in range(self.S):
                    _lib.check(_lib.load().mct_gated_forward_many(
                        self.family.handle, s, _lib.ptr(self.all_gates), self.N,
                        _lib.ptr(self.x[s]), _lib.ptr(proj[s]), _lib.ptr(self.ws), h))
            else:
                for s in range(self.S):
                    for g in range(self.N):
                        self.gated_forward(s, g, self.x[s], proj[s, g])
        fit = self.reduce(proj, self.d, self.S * self.N, self.n_sino, _lib.REDUCE_SQDIFF,
                          out=fit_out, st=st)
        xx = self.reduce(self.x, None, self.S, self.n_img, _lib.REDUCE_SQDIFF, out=xx_out, st=st)
        return fit, xx

    def objectives(self, alpha: float, reuse_projections: bool):
        """Per-slice objective alpha||x||^2 + sum_i ||A_i x - d_i||^2 / N (fp64)."""
        fit, xx = self.objective_parts(reuse_projections)
        fit = fit.view(self.S, self.N).cpu().numpy()
        xx = xx.cpu().numpy()
        return [float(alpha * xx[s] + sum(fit[s, g] / self.N for g in range(self.N)))
                for s in range(self.S)]

    def read_status(self):
        st = self.status.cpu().numpy().view(np.uint64)
        primal = int(st[0]) if st[0] != np.uint64(0xFFFFFFFFFFFFFFFF) else None
        dual = None
        if st[1] != np.uint64(0xFFFFFFFFFFFFFFFF):
            v = int(st[1])
            dual = (v >> 20, v & ((1 << 20) - 1))
        return primal, dual
