"""ctypes front-end of the CPU oracle (``oracle.c``).

TEST INFRASTRUCTURE ONLY -- see the header of ``oracle.c``.  Imported by
``tests/``, ``__graft_entry__.smoke()`` and the CPU-baseline legs of
``bench.py``; the product package never imports it.

Integer images run the reference's exact int64 arithmetic; float32 images run
the fp32 restatement (``oracle.c`` header).  Parity of this restatement with
the reference itself is pinned by ``tests/test_oracle.py`` against
``tests/golden/*`` (made by ``tests/golden/make_golden.py`` from
/root/reference) and against the reference's known-answer tests.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

METRICS = {"l1": 0, "sum": 1, "mean": 2}
KINDS = {"naive": 0, "filling-rate": 1}

_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.c"))
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int, ctypes.c_int64
        L.or_propagate.argtypes = [i32, i32, i32, i32, i32, P, P, i32, P, P]
        L.or_extrema.argtypes = [i32, i32, i32, i32, i32, P, P, P, P]
        L.or_run.argtypes = [i32, i32, i32, i32, i32, P, i32, i32, i32, P, P, P, P, P, P, i64, P, P]
        L.or_replay_prefix.argtypes = [i32, i32, i32, i32, i32, P, P, i64, i32, i32, P]
        L.or_fill_tree.argtypes = [i64, i32, P, P, P, P, P, P]
        L.or_fill_tree.restype = i64
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _prep(pixels):
    """(pixels array, isf) -- ints become int64 (reference domain), floats fp32."""
    px = np.asarray(pixels)
    if px.ndim != 2:
        raise ValueError("image must be 2-D")
    if np.issubdtype(px.dtype, np.integer):
        return np.ascontiguousarray(px, dtype=np.int64), 0
    return np.ascontiguousarray(px, dtype=np.float32), 1


def _metric(metric) -> int:
    return METRICS[getattr(metric, "value", metric)]


def propagate(pixels, sources, *, conn: int = 8, metric="sum"):
    """dijkstra_csr restated: returns (dist, parent); dist int64 or float32."""
    px, isf = _prep(pixels)
    H, W = px.shape
    src = np.ascontiguousarray(sources, dtype=np.int32)
    dist = np.empty(H * W, dtype=np.float32 if isf else np.int64)
    parent = np.empty(H * W, dtype=np.int32)
    rc = lib().or_propagate(H, W, conn, _metric(metric), isf, _ptr(px), _ptr(src), len(src),
                            _ptr(dist), _ptr(parent))
    if rc:
        raise MemoryError("oracle propagate failed")
    return dist, parent.astype(np.int64)


def extrema(pixels, *, conn: int = 8, metric="sum"):
    """_extrema_context restated: (centroid, dist_from_c, ext)."""
    px, isf = _prep(pixels)
    H, W = px.shape
    dfc = np.empty(H * W, dtype=np.float32 if isf else np.int64)
    ext = np.empty(H * W, dtype=np.int32)
    cen = np.zeros(1, dtype=np.int32)
    lib().or_extrema(H, W, conn, _metric(metric), isf, _ptr(px), _ptr(cen), _ptr(dfc), _ptr(ext))
    return int(cen[0]), dfc, ext.astype(np.int64)


def run(pixels, kind="filling-rate", *, conn: int = 8, metric="sum", naive_with_tree=False,
        nthreads: int = 1, max_steps: int | None = None):
    """run_strategy restated for naive / filling-rate.

    Returns a dict with D (N x N, int64 or float32), seq, new, visits, raw,
    adjusted, centroid, filled.
    """
    px, isf = _prep(pixels)
    H, W = px.shape
    n = H * W
    D = np.empty((n, n), dtype=np.float32 if isf else np.int64)
    seq = np.zeros(n, dtype=np.int32)
    new = np.zeros(n, dtype=np.int64)
    visits = np.zeros(n, dtype=np.int64)
    walked = np.zeros(n, dtype=np.int64)
    stats = np.zeros(8, dtype=np.int64)
    loop_s = np.zeros(1, dtype=np.float64)
    commit_s = np.zeros(n, dtype=np.float64)
    rc = lib().or_run(H, W, conn, _metric(metric), isf, _ptr(px), KINDS[getattr(kind, "value", kind)],
                      int(naive_with_tree), nthreads, _ptr(D), _ptr(seq), _ptr(new), _ptr(visits),
                      _ptr(walked), _ptr(stats), n if max_steps is None else max_steps, _ptr(loop_s),
                      _ptr(commit_s))
    if rc not in (0,) and not (max_steps is not None and rc == 0):
        raise RuntimeError(f"oracle run failed rc={rc}")
    P = int(stats[0])
    return {
        "D": D, "seq": seq[:P].astype(np.int64), "new": new[:P], "visits": visits[:P], "walked": walked[:P],
        "raw": P, "adjusted": int(stats[1]), "centroid": int(stats[3]), "filled": int(stats[4]),
        "loop_seconds": float(loop_s[0]), "commit_seconds": commit_s[:P],
    }


def replay_prefix(pixels, seq, steps: int, *, conn: int = 8, metric="sum", use_tree=True,
                  nthreads: int = 1):
    """Propagate + fill the first ``steps`` sources of a known sequence (CPU baseline)."""
    px, isf = _prep(pixels)
    H, W = px.shape
    s = np.ascontiguousarray(seq[:steps], dtype=np.int32)
    new = np.zeros(steps, dtype=np.int64)
    rc = lib().or_replay_prefix(H, W, conn, _metric(metric), isf, _ptr(px), _ptr(s), steps,
                                int(use_tree), nthreads, _ptr(new))
    if rc:
        raise MemoryError("oracle replay failed")
    return new


def fill_tree(parent, tdist, D, mark, counts):
    """fill_tree_pairs restated on caller arrays; returns (new, bad)."""
    n = len(parent)
    isf = 1 if D.dtype == np.float32 else 0
    par = np.ascontiguousarray(parent, dtype=np.int32)
    td = np.ascontiguousarray(tdist, dtype=np.float32 if isf else np.int64)
    bad = np.zeros(1, dtype=np.int64)
    new = lib().or_fill_tree(n, isf, _ptr(par), _ptr(td), _ptr(D), _ptr(mark), _ptr(counts), _ptr(bad))
    return int(new), int(bad[0])
