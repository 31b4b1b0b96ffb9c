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
APGD_VERSION_FLOAT = 2  # additive: fp32 stores (binary64 bits per value)
APGD_HEADER = len(APGD_MAGIC) + 5
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

    # ---- one step of a host-selected run (strategies.py:263-271) ----
    def _set_counts(self, counts: np.ndarray):
        arr = counts.astype(np.int64)
        arr.setflags(write=False)
        self._cache = {"counts": arr}

    def _commit_source(self, graph, source: int, counts: np.ndarray) -> int:
        """Propagate from `source`, fill its tree (reference checks) and refresh
        the per-pixel counts: gp_commit_source, one synchronisation."""
        new = ctypes.c_int64()
        self._cache.clear()
        _lib.check(_lib.lib().gp_commit_source(graph.handle, self._st, int(source), self._tol(),
                                               ctypes.byref(new), _lib.ptr(counts)))
        self._filled += new.value
        self._set_counts(counts)
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

    # ---- APGD dump / load (distances.py:149-177) ----
    # Row blocks are converted to u64 on the device (gp_store_apgd_rows /
    # gp_store_load_rows), so no N^2 host temporary is ever built; integer
    # stores write the reference's version 1, float stores version 2
    # (additive: binary64 bits of the fp32 value, same sentinel).
    _TILE_BYTES = 32 << 20

    def _apgd_version(self) -> int:
        return APGD_VERSION if self._integer else APGD_VERSION_FLOAT

    def _tile_rows(self) -> int:
        return max(1, self._TILE_BYTES // (8 * self.n))

    def apgd_header(self) -> bytes:
        return APGD_MAGIC + struct.pack("<BI", self._apgd_version(), self.n)

    def apgd_row_tiles(self):
        """Yield (row0, u64 array [rows, n]) blocks of the APGD payload."""
        n, per, ver = self.n, self._tile_rows(), self._apgd_version()
        buf = np.empty((per, n), dtype="<u8")
        for r0 in range(0, n, per):
            k = min(per, n - r0)
            _lib.check(_lib.lib().gp_store_apgd_rows(self._st, ver, r0, k, _lib.ptr(buf)))
            yield r0, buf[:k]

    def to_bytes(self) -> bytes:
        """Serialize to the APGD binary dump (magic, version, n, u64 grid)."""
        head = self.apgd_header()
        out = bytearray(len(head) + 8 * self.n * self.n)
        out[:len(head)] = head
        view = np.frombuffer(out, dtype=np.uint8)
        for r0, blk in self.apgd_row_tiles():
            o = len(head) + 8 * r0 * self.n
            view[o:o + blk.nbytes] = blk.reshape(-1).view(np.uint8)
        return bytes(out)

    def write_apgd(self, f) -> int:
        """Stream the APGD dump to a binary file object; returns the bytes written."""
        head = self.apgd_header()
        f.write(head)
        total = len(head)
        for _, blk in self.apgd_row_tiles():
            f.write(memoryview(np.ascontiguousarray(blk)).cast("B"))
            total += blk.nbytes
        return total

    @staticmethod
    def _apgd_parse_header(head: bytes):
        if len(head) < APGD_HEADER or head[:4] != APGD_MAGIC:
            raise ValueError("not an APGD dump (bad magic)")
        version, n = struct.unpack("<BI", head[4:APGD_HEADER])
        if version not in (APGD_VERSION, APGD_VERSION_FLOAT):
            raise ValueError(f"unsupported APGD version {version}")
        return version, n

    @classmethod
    def _apgd_store(cls, version: int, n: int, blocks) -> "DistanceArray":
        store = cls(n, force=True)
        for r0, blk in blocks:
            blk = np.ascontiguousarray(blk, dtype="<u8")
            _lib.check(_lib.lib().gp_store_load_rows(store._st, version, r0, blk.shape[0], _lib.ptr(blk)))
        filled = ctypes.c_int64()
        _lib.check(_lib.lib().gp_store_recount(store._st, ctypes.byref(filled)))
        store._filled = filled.value
        store._integer = version == APGD_VERSION
        store._cache.clear()
        return store

    @classmethod
    def from_bytes(cls, data: bytes) -> "DistanceArray":
        """Parse an APGD binary dump back into a DistanceArray."""
        version, n = cls._apgd_parse_header(bytes(data[:APGD_HEADER]))
        expected = APGD_HEADER + 8 * n * n
        if len(data) != expected:
            raise ValueError(f"APGD dump has {len(data)} bytes, expected {expected}")
        grid = np.frombuffer(data, dtype="<u8", offset=APGD_HEADER).reshape(n, n)
        per = max(1, cls._TILE_BYTES // (8 * n))
        return cls._apgd_store(version, n, ((r0, grid[r0:r0 + per]) for r0 in range(0, n, per)))

    @classmethod
    def read_apgd(cls, f) -> "DistanceArray":
        """Stream an APGD dump from a binary file object (no N^2 host buffer)."""
        version, n = cls._apgd_parse_header(f.read(APGD_HEADER))
        per = max(1, cls._TILE_BYTES // (8 * n))

        def blocks():
            for r0 in range(0, n, per):
                k = min(per, n - r0)
                raw = f.read(8 * k * n)
                if len(raw) != 8 * k * n:
                    raise ValueError("APGD dump is truncated")
                yield r0, np.frombuffer(raw, dtype="<u8").reshape(k, n)
            if f.read(1):
                raise ValueError("APGD dump has trailing bytes")

        return cls._apgd_store(version, n, blocks())
