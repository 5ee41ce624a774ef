"""ctypes binding of libuqg.so (include/uqg.h) plus small device helpers.

The product path has no CPU fallback: if the extension or a CUDA device is
missing, every compute entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np

from .errors import DeviceError, EnsembleError, NumericalBreakdownError

LIB_PATH = Path(__file__).resolve().parent / "libuqg.so"

UQG_OK, UQG_EINVAL, UQG_EBREAKDOWN, UQG_ECUDA, UQG_ENOMEM, UQG_ECAPACITY = range(6)

_c_int, _c_double, _c_ll = ctypes.c_int, ctypes.c_double, ctypes.c_longlong
_p = ctypes.c_void_p

# UQG_NKERN (include/uqg.h): length of the per-kernel-class arrays that
# uqg_ctx_profile_read fills
NKERN = 11

# name -> (restype, argtypes); the exact list include/uqg.h declares
SIGNATURES = {
    "uqg_version": (_c_int, []),
    "uqg_last_error": (ctypes.c_char_p, []),
    "uqg_ctx_create": (_c_int, [_c_int, ctypes.POINTER(_p)]),
    "uqg_ctx_destroy": (_c_int, [_p]),
    "uqg_ctx_set_workspace": (_c_int, [_p, _p, _c_ll]),
    "uqg_ctx_set_band_hint": (_c_int, [_p, _c_int, _p, _p, _c_int]),
    "uqg_ctx_profile": (_c_int, [_p, _c_int]),
    "uqg_ctx_profile_read": (_c_int, [_p, _p, _p, _c_int]),
    "uqg_ctx_launch_count": (_c_ll, [_p]),
    "uqg_status_sync": (_c_int, [_p, _p, ctypes.POINTER(_c_int)]),
    "uqg_kl_eval_sep2d": (_c_int, [_p, _c_int, _p, _c_int, _p, _p, _p, _c_int, _p, _p, _c_int,
                                   _c_int, _c_double, _c_int, _c_double, _c_int, _p, _p]),
    "uqg_kl_eval_table": (_c_int, [_p, _p, _c_int, _c_int, _p, _p, _c_int, _c_double, _c_int,
                                   _c_double, _c_int, _p, _p]),
    "uqg_assemble_fv2d": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _c_double, _c_int, _p, _p, _p,
                                   _p]),
    "uqg_kl_eval_sep3d": (_c_int, [_p, _c_int, _p, _c_int, _p, _p, _p, _p, _c_int, _p, _p, _c_int,
                                   _c_int, _c_double, _c_int, _c_double, _c_int, _p, _p]),
    "uqg_assemble_fem3d": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p, _p, _p]),
    "uqg_jacobi_dinv": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p]),
    "uqg_diagonal": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p]),
    "uqg_spmv": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p, _p]),
    "uqg_lane_dot": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _p, _p, _p]),
    "uqg_pcg": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p, _c_double, _p,
                         _c_double, _c_int, _p, _p, _p, _p, _p, _p, _c_int,
                         ctypes.POINTER(_c_int), _p]),
    "uqg_pcg_workspace_bytes": (_c_ll, [_c_int, _c_int, _c_int, _c_int]),
    "uqg_pcg_x_defer": (_c_int, []),
    "uqg_assemble_fv2d_faces": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _c_double, _c_int, _p,
                                         _p, _p, _p]),
    "uqg_spmv_fv2d": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _p, _c_double, _p, _p, _p]),
    "uqg_pcg_fv2d": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _p, _c_double, _p, _c_double, _p,
                              _c_double, _c_int, _p, _p, _p, _p, _p, _p, _c_int,
                              ctypes.POINTER(_c_int), _p]),
    "uqg_group_sort": (_c_int, [_p, _p, _c_int, _c_int, _p, _p, _p, _p]),
    "uqg_group_sort_async": (_c_int, [_p, _p, _c_int, _c_int, _p, _p, _p, _p]),
    "uqg_status_clear": (_c_int, [_p, _p]),
    "uqg_surrogate_eval": (_c_int, [_p, _p, _c_int, _c_int, _p, _p, _p, _c_int, _p, _p]),
    "uqg_anisotropy_indicator": (_c_int, [_p, _p, _c_int, _c_int, _p, _p, _c_int, _c_double,
                                          _c_int, _c_double, _c_int, _c_double, _c_double, _p,
                                          _p]),
}

_lock = threading.Lock()
_lib = None
_ctx: dict[int, int] = {}


def load() -> ctypes.CDLL:
    """Load libuqg.so (no compute; works on a CPU-only host)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() first")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the ensemble solve runs on the GPU only (no CPU fallback)")
    return torch


def device():
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device())


def ctx() -> int:
    """Per-device library context (owns scratch workspace and events)."""
    torch = _torch()
    dev = torch.cuda.current_device()
    lib = load()
    with _lock:
        if dev not in _ctx:
            out = _p()
            check(lib.uqg_ctx_create(dev, ctypes.byref(out)))
            _ctx[dev] = out.value
    return _ctx[dev]


def stream() -> int:
    torch = _torch()
    return torch.cuda.current_stream().cuda_stream


def last_error() -> str:
    msg = load().uqg_last_error()
    return msg.decode() if msg else ""


def check(rc: int, invalid=EnsembleError) -> None:
    if rc == UQG_OK:
        return
    msg = last_error()
    if rc == UQG_EINVAL:
        raise invalid(msg)
    if rc == UQG_EBREAKDOWN:
        raise NumericalBreakdownError(msg)
    raise DeviceError(f"libuqg error {rc}: {msg}")


def call(name: str, *args, invalid=EnsembleError) -> None:
    check(getattr(load(), name)(*args), invalid)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def status_sync() -> int:
    out = _c_int(0)
    check(load().uqg_status_sync(ctx(), stream(), ctypes.byref(out)))
    return out.value


# --- host <-> device layout helpers ------------------------------------------

def to_dev(a, dtype=None):
    """Host array -> contiguous device tensor."""
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False)


def lanes_to_dev(x: np.ndarray):
    """(S, n) lane-major host array -> device [n][S] interleaved (G=1)."""
    return to_dev(np.ascontiguousarray(np.asarray(x, dtype=np.float64).T))


def dev_to_lanes(t, S: int, n: int) -> np.ndarray:
    """Device [n][S] interleaved -> host (S, n) lane-major."""
    return np.ascontiguousarray(t.reshape(n, S).cpu().numpy().T)
