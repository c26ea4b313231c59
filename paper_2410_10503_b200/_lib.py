"""ctypes binding of the sm_100a C-ABI (include/mctomo_b200.h).

There is no CPU fallback: if the CUDA library is missing or no GPU is visible,
every compute entry point raises.  Loading the library itself does not need a
GPU (it is how the CPU test-suite checks the exported symbols).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .build import LIB_PATH

MCT_OK, MCT_ERR_ARG, MCT_ERR_CUDA, MCT_ERR_STATE = 0, 1, 2, 3
WARP_IDENTITY, WARP_RIGID, WARP_DILATATION, WARP_DENSE = 0, 1, 2, 3
REDUCE_DOT, REDUCE_SQDIFF = 0, 1

c_int, c_int32, c_double, c_void_p = ctypes.c_int, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
c_size_t, c_longlong, c_float = ctypes.c_size_t, ctypes.c_longlong, ctypes.c_float
c_uint64 = ctypes.c_uint64
PP = ctypes.POINTER(c_void_p)


class Items(ctypes.Structure):
    """mct_items (include/mctomo_b200.h)."""

    _fields_ = [
        ("gates_dev", c_void_p),
        ("epoch_ctr_dev", c_void_p),
        ("slice_stride", c_int32),
        ("epoch_stride", c_int32),
        ("base", c_int32),
        ("items_per_slice", c_int32),
        ("num_slices", c_int32),
        ("iteration", c_int32),
        ("iters_per_epoch", c_int32),
        ("last_part", c_int32),
        ("first_item", c_int32),
        ("item_count", c_int32),
    ]


class State(ctypes.Structure):
    """mct_state (include/mctomo_b200.h)."""

    _fields_ = [
        ("x", c_void_p),
        ("x_next", c_void_p),
        ("z", c_void_p),
        ("zbar", c_void_p),
        ("y", c_void_p),
        ("d", c_void_p),
        ("proj", c_void_p),
        ("status", c_void_p),
    ]


# name -> (restype, argtypes); every symbol declared in include/mctomo_b200.h
SIGNATURES = {
    "mct_abi_version": (c_int, []),
    "mct_last_error": (ctypes.c_char_p, []),
    "mct_ray_plan_create": (c_int, [PP, c_int, c_int, c_int, c_int, c_double, c_void_p, c_void_p,
                                    c_void_p]),
    "mct_ray_plan_destroy": (c_int, [c_void_p]),
    "mct_ray_workspace_bytes": (c_size_t, [c_void_p, c_int]),
    "mct_ray_plan_set_ring_pairs": (c_int, [c_void_p, c_int]),
    "mct_ray_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "mct_ray_adjoint": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "mct_warp_plan_create_rigid": (c_int, [PP, c_int, c_int, c_double, c_double, c_double,
                                           c_double]),
    "mct_warp_plan_create_dilatation": (c_int, [PP, c_int, c_int, c_double]),
    "mct_warp_plan_create_identity": (c_int, [PP, c_int, c_int]),
    "mct_warp_plan_create_dense": (c_int, [PP, c_int, c_int, c_void_p, c_void_p]),
    "mct_warp_plan_destroy": (c_int, [c_void_p]),
    "mct_warp_plan_kind": (c_int, [c_void_p]),
    "mct_warp_plan_nnz": (c_longlong, [c_void_p]),
    "mct_warp_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "mct_warp_adjoint": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "mct_family_create": (c_int, [PP, c_void_p, c_int, c_int, c_void_p]),
    "mct_family_destroy": (c_int, [c_void_p]),
    "mct_family_set_params": (c_int, [c_void_p, c_void_p, c_void_p, c_double]),
    "mct_family_workspace_bytes": (c_size_t, [c_void_p, c_int]),
    "mct_family_chunk_items": (c_int, [c_void_p, c_int]),
    "mct_gated_forward": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mct_gated_adjoint": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mct_iter_prox_warp": (c_int, [c_void_p, ctypes.POINTER(Items), ctypes.POINTER(State),
                                   c_double, c_double, c_void_p, c_void_p]),
    "mct_iter_forward_dual": (c_int, [c_void_p, ctypes.POINTER(Items), ctypes.POINTER(State),
                                      c_void_p, c_void_p]),
    "mct_iter_adjoint": (c_int, [c_void_p, ctypes.POINTER(Items), c_void_p, c_void_p]),
    "mct_iter_adjoint_update": (c_int, [c_void_p, ctypes.POINTER(Items), ctypes.POINTER(State),
                                        c_void_p, c_void_p, c_void_p]),
    "mct_iter_z_update": (c_int, [c_void_p, ctypes.POINTER(State), c_void_p, c_double, c_void_p]),
    "mct_epoch_advance": (c_int, [c_void_p, c_int32, c_void_p]),
    "mct_reduce": (c_int, [c_void_p, c_void_p, c_longlong, c_int, c_longlong, c_int, c_void_p,
                           c_void_p, c_void_p]),
    "mct_axpby": (c_int, [c_longlong, c_float, c_void_p, c_float, c_void_p, c_void_p]),
    "mct_axpby_mixed": (c_int, [c_longlong, c_double, c_void_p, c_int, c_double, c_void_p, c_int,
                                c_void_p]),
    "mct_dot_f64": (c_int, [c_void_p, c_void_p, c_longlong, c_void_p, c_void_p, c_void_p]),
    "mct_gaussian_field": (c_int, [c_uint64, c_uint64, c_longlong, c_double, c_void_p, c_void_p,
                                   c_int, c_void_p]),
    "mct_gated_forward_many": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p,
                                       c_void_p, c_void_p]),
    "mct_exchange_post": (c_int, [c_void_p, c_int, c_int, c_uint64, c_void_p]),
    "mct_exchange_z_update": (c_int, [c_void_p, c_void_p, c_int, c_uint64, c_longlong, c_void_p,
                                      c_void_p, c_double, c_void_p, c_void_p]),
}

_LIB = None


def lib_path() -> Path:
    return Path(os.environ.get("MCT_LIB", str(LIB_PATH)))


def load() -> ctypes.CDLL:
    """Load the in-tree sm_100a library (raises loudly if it was not built)."""
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not path.exists():
            raise RuntimeError(
                f"CUDA library {path} is missing: run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.mct_abi_version() != 2:
            raise RuntimeError("unexpected mctomo_b200 ABI version")
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    if rc == MCT_OK:
        return
    msg = load().mct_last_error().decode(errors="replace")
    if rc == MCT_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"mctomo_b200: {msg}")


def require_cuda():
    """Import torch and insist on a CUDA device (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2410_10503_b200 needs a CUDA (sm_100a) device; none is visible")
    load()
    return torch


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr())


REDUCE_PARTS = 128
_SCRATCH = {}


def scratch(device, segments: int = 1, stream: int | None = None):
    """Cached fp64 scratch for the two-pass reductions (per device and stream, so
    reductions issued on different streams never share partials).  ``stream``: the
    raw handle when the caller already has it (saves the torch stream query)."""
    import torch

    key = (str(device), stream_handle() if stream is None else stream)
    need = REDUCE_PARTS * max(1, segments)
    t = _SCRATCH.get(key)
    if t is None or t.numel() < need:
        t = _SCRATCH[key] = torch.empty(need, dtype=torch.float64, device=device)
    return t
