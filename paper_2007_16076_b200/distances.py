"""The N x N distances array on the device (reference distances.py).

``DistanceArray`` keeps D (fp32, N x N), the mark matrix (one bit per entry)
and the per-pixel filled counts in device memory (gp_store).  The host views
``dist`` / ``mark`` are materialised on demand with the reference's types and
sentinels: int64 with -1 for unmarked entries when the stored values are
integers (exact: integer distances are < 2^24), float32 otherwise.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib

#: Pixel-count guard for the dense N^2 allocation (distances.py:15).
MAX_PIXELS = 10_000

APGD_MAGIC = b"APGD"
APGD_VERSION = 1
APGD_SENTINEL = 0xFFFF_FFFF_FFFF_FFFF

#: relative agreement tolerance for float-valued fills (integers: exact)
FLOAT_TOL = 1e-4


class SizeGuardError(RuntimeError):
    """Raised when an allocation would exceed the dense-storage pixel guard."""


@dataclass(frozen=True)
class FillStats:
    total_pairs: int
    filled_pairs: int
    rate: Fraction


class DistanceArray:
    """Symmetric all-pairs distance array with mark matrix (distances.py:36-177)."""

    def __init__(self, n: int, *, force: bool = False):
        if n < 2:
            raise ValueError(f"need at least 2 pixels, got {n}")
        if n > MAX_PIXELS and not force:
            raise SizeGuardError(
                f"{n} pixels needs a dense {n}x{n} array (guard is {MAX_PIXELS}); "
                "pass force=True to override"
            )
        self.n = n
        handle = ctypes.c_void_p()
        _lib.check(_lib.lib().gp_store_create(n, ctypes.byref(handle)))
        self._st = handle
        self._filled = 0
        self._integer = True
        self._cache = {}

    def __del__(self):
        st = getattr(self, "_st", None)
        if st is not None and _lib._lib is not None:
            _lib._lib.gp_store_destroy(st)
            self._st = None

    # ---- bookkeeping (distances.py:63-93) ----
    @property
    def total_pairs(self) -> int:
        return (self.n * self.n - self.n) // 2

    @property
    def pairs_filled(self) -> int:
        return self._filled

    @property
    def point_filled_counts(self) -> np.ndarray:
        if "counts" not in self._cache:
            out = np.empty(self.n, dtype=np.int32)
            _lib.check(_lib.lib().gp_store_counts(self._st, _lib.ptr(out), None))
            arr = out.astype(np.int64)
            arr.setflags(write=False)
            self._cache["counts"] = arr
        return self._cache["counts"]

    @property
    def is_complete(self) -> bool:
        return self._filled == self.total_pairs

    def filling_rate(self) -> Fraction:
        return Fraction(self._filled, self.total_pairs)

    def point_filling_rate(self, pixel: int) -> Fraction:
        if not 0 <= pixel < self.n:
            raise ValueError(f"pixel {pixel} out of range for n={self.n}")
        return Fraction(int(self.point_filled_counts[pixel]), self.n - 1)

    def stats(self) -> FillStats:
        return FillStats(self.total_pairs, self._filled, self.filling_rate())

    # ---- fills ----
    def _note_values(self, values: np.ndarray):
        if not np.issubdtype(values.dtype, np.integer):
            self._integer = False
        elif values.size and np.abs(values).max() >= (1 << 24):
            raise ValueError("integer distances must stay below 2^24 on the fp32 device store")

    def _tol(self) -> float:
        return 0.0 if self._integer else FLOAT_TOL

    def fill_from_tree(self, tree) -> int:
        """Mark every ancestor/descendant pair of a tree (distances.py:95-118)."""
        if tree.parent.shape[0] != self.n or tree.dist.shape[0] != self.n:
            raise ValueError(f"tree spans {tree.parent.shape[0]} pixels, array holds {self.n}")
        self._note_values(np.asarray(tree.dist))
        parent = np.ascontiguousarray(tree.parent, dtype=np.int32)
        td = np.ascontiguousarray(tree.dist, dtype=np.float32)
        new = ctypes.c_int64()
        self._cache.clear()
        _lib.check(_lib.lib().gp_store_fill_tree(self._st, _lib.ptr(parent), _lib.ptr(td),
                                                 self._tol(), ctypes.byref(new)))
        self._filled += new.value
        return new.value

    def fill_from_source(self, source: int, dist: np.ndarray) -> int:
        """Mark the source's row and column (distances.py:120-147)."""
        if not 0 <= source < self.n:
            raise ValueError(f"source {source} out of range for n={self.n}")
        if dist.shape[0] != self.n:
            raise ValueError(f"distance map has {dist.shape[0]} entries, need {self.n}")
        if dist[source] != 0:
            raise ValueError("source's distance to itself must be 0")
        self._note_values(np.asarray(dist))
        d32 = np.ascontiguousarray(dist, dtype=np.float32)
        new = ctypes.c_int64()
        self._cache.clear()
        _lib.check(_lib.lib().gp_store_fill_source(self._st, int(source), _lib.ptr(d32),
                                                   self._tol(), ctypes.byref(new)))
        self._filled += new.value
        return new.value

    # ---- host / device views ----
    def _read(self):
        if "D" not in self._cache:
            D = np.empty((self.n, self.n), dtype=np.float32)
            M = np.empty((self.n, self.n), dtype=np.uint8)
            _lib.check(_lib.lib().gp_store_read(self._st, _lib.ptr(D), _lib.ptr(M)))
            M = M.view(np.bool_)
            D = np.where(M, D, np.float32(-1.0))
            if self._integer:
                D = D.astype(np.int64)
            self._cache["D"], self._cache["M"] = D, M
        return self._cache["D"], self._cache["M"]

    @property
    def dist(self) -> np.ndarray:
        return self._read()[0]

    @property
    def mark(self) -> np.ndarray:
        return self._read()[1]

    def device_pointers(self) -> dict:
        """Raw device pointers of D (fp32 n*n), mark (u32 bitmap) and counts (i32)."""
        D, M, C = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        words = ctypes.c_int64()
        _lib.check(_lib.lib().gp_store_device_ptrs(self._st, ctypes.byref(D), ctypes.byref(M),
                                                   ctypes.byref(C), ctypes.byref(words)))
        return {"D": D.value, "mark": M.value, "counts": C.value, "mark_words_per_row": words.value}

    def dist_device(self):
        """Zero-copy torch view (fp32, n x n) of the device D."""
        import torch

        p = self.device_pointers()["D"]
        iface = {"shape": (self.n, self.n), "typestr": "<f4", "data": (p, False), "version": 3,
                 "strides": None}
        holder = type("_DevArr", (), {"__cuda_array_interface__": iface})()
        t = torch.as_tensor(holder, device="cuda")
        return t

    def _after_run(self, filled: int, integer: bool):
        self._filled = int(filled)
        self._integer = bool(integer)
        self._cache.clear()

    def to_bytes(self) -> bytes:
        """APGD dump (distances.py:149-154)."""
        D, M = self._read()
        out = D.astype(np.uint64)
        out[~M] = APGD_SENTINEL
        header = APGD_MAGIC + struct.pack("<BI", APGD_VERSION, self.n)
        return header + out.astype("<u8").tobytes()
