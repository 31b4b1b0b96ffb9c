"""ctypes binding of the C ABI in include/geopairs_b200.h.

The shared library is built in-tree (``paper_2007_16076_b200/libgeopairs_b200.so``,
see ``build.py``).  There is no CPU fallback: loading fails loudly when the
library is missing or no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgeopairs_b200.so")

GP_OK, GP_EINVAL, GP_ENOMEM, GP_ECUDA, GP_EINTERNAL, GP_ECYCLE, GP_EDISAGREE, GP_EFULL = range(8)
DTYPE_I64, DTYPE_F32, DTYPE_U8 = 0, 1, 2
STRATEGY_NAIVE, STRATEGY_FILLING_RATE, STRATEGY_EXTREMA = 0, 1, 2

# every symbol declared in include/geopairs_b200.h
EXPORTS = (
    "gp_last_error", "gp_version", "gp_ctx_create", "gp_ctx_load", "gp_ctx_destroy",
    "gp_ctx_num_pixels",
    "gp_propagate", "gp_propagate_batch", "gp_extrema", "gp_store_create", "gp_store_destroy",
    "gp_store_device_ptrs", "gp_store_fill_tree", "gp_store_fill_source", "gp_store_counts",
    "gp_store_read", "gp_store_apgd_rows", "gp_store_load_rows", "gp_store_recount",
    "gp_commit_source", "gp_run", "gp_run_to_host",
)


class RunStats(ctypes.Structure):
    _fields_ = [
        ("raw_count", ctypes.c_int64), ("adjusted_count", ctypes.c_int64),
        ("centroid", ctypes.c_int64), ("propagations", ctypes.c_int64),
        ("batches", ctypes.c_int64), ("launches", ctypes.c_int64),
        ("kernels", ctypes.c_int64), ("filled_pairs", ctypes.c_int64), ("visits", ctypes.c_int64),
        ("ms_total", ctypes.c_double), ("ms_propagate", ctypes.c_double),
        ("ms_commit", ctypes.c_double), ("ms_setup", ctypes.c_double),
        ("disagreements", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class GeopairsError(RuntimeError):
    """A CUDA / internal failure reported by the native library."""


_lib = None


def load_library(path: str = LIB_PATH, *, require_device: bool = True):
    """Load the native library (cached).  Raises if absent -- no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2007_16076_b200.build` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(path)
    P, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
    L.gp_last_error.restype = ctypes.c_char_p
    L.gp_ctx_create.argtypes = [i32, i32, i32, P, i32, i32, ctypes.POINTER(P)]
    L.gp_ctx_load.argtypes = [P, i32, P]
    L.gp_ctx_destroy.argtypes = [P]
    L.gp_ctx_destroy.restype = None
    L.gp_ctx_num_pixels.argtypes = [P]
    L.gp_propagate.argtypes = [P, P, i32, P, P]
    L.gp_propagate_batch.argtypes = [P, P, i32, P, P, P]
    L.gp_extrema.argtypes = [P, P, P, P]
    L.gp_store_create.argtypes = [i64, ctypes.POINTER(P)]
    L.gp_store_destroy.argtypes = [P]
    L.gp_store_destroy.restype = None
    L.gp_store_device_ptrs.argtypes = [P, P, P, P, P]
    L.gp_store_fill_tree.argtypes = [P, P, P, f32, P]
    L.gp_store_fill_source.argtypes = [P, i64, P, f32, P]
    L.gp_store_counts.argtypes = [P, P, P]
    L.gp_store_read.argtypes = [P, P, P]
    L.gp_store_apgd_rows.argtypes = [P, i32, i64, i64, P]
    L.gp_store_load_rows.argtypes = [P, i32, i64, i64, P]
    L.gp_store_recount.argtypes = [P, P]
    L.gp_commit_source.argtypes = [P, P, i32, f32, P, P]
    L.gp_run.argtypes = [P, P, i32, i32, i32, P, P, ctypes.POINTER(RunStats)]
    L.gp_run_to_host.argtypes = [P, P, i32, i32, i32, P, P, ctypes.POINTER(RunStats), P]
    _lib = L
    if require_device:
        _require_device()
    return L


def _require_device():
    try:
        import torch

        ok = torch.cuda.is_available()
    except Exception:  # pragma: no cover - torch always present in this image
        ok = False
    if not ok:
        raise GeopairsError("no CUDA device visible: the geopairs B200 path has no CPU fallback")


def lib():
    return load_library()


def check(rc: int, *, value_error=ValueError, full_error=None):
    """Map a GP_* status to the reference's exception types."""
    if rc == GP_OK:
        return
    msg = lib().gp_last_error().decode(errors="replace")
    if rc in (GP_EINVAL, GP_ECYCLE, GP_EDISAGREE):
        raise value_error(msg)
    if rc == GP_EFULL and full_error is not None:
        raise full_error(msg)
    if rc == GP_ENOMEM:
        raise MemoryError(msg)
    raise GeopairsError(f"{msg} (status {rc})")


def ptr(a) -> ctypes.c_void_p:
    return a.ctypes.data_as(ctypes.c_void_p)
