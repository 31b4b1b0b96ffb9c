"""Geodesic propagations on the GPU and their trees (reference propagation.py).

``GridGraph`` owns a device context (image + tree store); ``propagate`` runs
the K1 kernel (one CTA) and returns host arrays with the reference's types:
int64 distances/parents for integer images (bit-identical to dijkstra_csr,
reference _kernels.py:33-79), float32 distances for float images.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .grid import METRIC_CODE, Image, Metric, check_pixel

#: Larger than any reachable path time (reference _kernels.py:15).
UNREACHED = np.int64(1) << np.int64(50)


@dataclass(frozen=True)
class PropagationResult:
    """Distances and shortest-path forest of one propagation (propagation.py:16-26)."""

    sources: tuple
    dist: np.ndarray
    parent: np.ndarray


@dataclass(frozen=True)
class GeodesicTree:
    """Shortest-path tree of a single-source propagation (propagation.py:29-42)."""

    root: int
    parent: np.ndarray
    dist: np.ndarray
    children: list
    leaves: list


class GridGraph:
    """Grid graph of an image bound to a device context (propagation.py:45-64).

    ``connectivity`` (additive) selects the 8- (reference) or 4-neighbourhood.
    """

    def __init__(self, image: Image, metric: Metric = Metric.SUM, *, connectivity: int = 8):
        if connectivity not in (4, 8):
            raise ValueError(f"connectivity must be 4 or 8, got {connectivity}")
        self.image = image
        self.metric = metric
        self.connectivity = connectivity
        self.n = image.size
        L = _lib.lib()
        px = np.ascontiguousarray(image.pixels)
        dtype = _lib.DTYPE_I64 if image.is_integer else _lib.DTYPE_F32
        handle = ctypes.c_void_p()
        _lib.check(L.gp_ctx_create(image.height, image.width, dtype, _lib.ptr(px),
                                   METRIC_CODE[metric], connectivity, ctypes.byref(handle)))
        self._ctx = handle

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and _lib._lib is not None:
            _lib._lib.gp_ctx_destroy(ctx)
            self._ctx = None

    @property
    def handle(self):
        return self._ctx

    def propagate(self, sources: Sequence[int]) -> PropagationResult:
        """Geodesic distances from the nearest of ``sources`` to every pixel."""
        srcs = _checked_sources(self.image, sources)
        dist = np.empty(self.n, dtype=np.float32)
        parent = np.empty(self.n, dtype=np.int32)
        s32 = np.ascontiguousarray(srcs, dtype=np.int32)
        _lib.check(_lib.lib().gp_propagate(self._ctx, _lib.ptr(s32), len(s32), _lib.ptr(dist),
                                           _lib.ptr(parent)))
        if self.image.is_integer:
            dist = dist.astype(np.int64)
        return PropagationResult(tuple(int(s) for s in srcs), dist, parent.astype(np.int64))


def _checked_sources(image: Image, sources: Sequence[int]) -> np.ndarray:
    """Validation of propagation.py:92-99."""
    if len(sources) == 0:
        raise ValueError("at least one source pixel is required")
    dims = (image.width, image.height)
    srcs = np.asarray([check_pixel(dims, int(s)) for s in sources], dtype=np.int64)
    if len(set(srcs.tolist())) != len(srcs):
        raise ValueError("duplicate source pixels")
    return srcs


def propagate(image: Image, metric: Metric, sources: Sequence[int], *,
              connectivity: int = 8) -> PropagationResult:
    """One-shot propagation (propagation.py:102-108)."""
    return GridGraph(image, metric, connectivity=connectivity).propagate(sources)


def build_tree(result: PropagationResult, root: int) -> GeodesicTree:
    """Materialise the geodesic tree of a single-source propagation (propagation.py:111-127).

    Children lists are built with one stable argsort instead of a Python loop;
    they are ascending, as in the reference.
    """
    if result.sources != (root,):
        raise ValueError(f"tree root {root} does not match propagation sources {result.sources}")
    n = result.dist.shape[0]
    d = result.dist
    if (np.issubdtype(d.dtype, np.integer) and np.any(d >= UNREACHED)) or (
        np.issubdtype(d.dtype, np.floating) and not np.isfinite(d).all()
    ):
        raise ValueError("propagation did not reach every pixel")
    parent = result.parent
    kids = np.flatnonzero(parent >= 0)
    order = kids[np.argsort(parent[kids], kind="stable")]
    counts = np.bincount(parent[kids], minlength=n)
    splits = np.split(order, np.cumsum(counts)[:-1])
    children = [s.tolist() for s in splits]
    leaves = np.flatnonzero(counts == 0).tolist()
    return GeodesicTree(root, parent, result.dist, children, leaves)


def boundary_pixels(dims: tuple[int, int]) -> list[int]:
    """All border pixels, ascending (propagation.py:130-143)."""
    width, height = dims
    if width < 1 or height < 1:
        raise ValueError(f"invalid dimensions {width}x{height}")
    idx = np.arange(width * height).reshape(height, width)
    mask = np.zeros((height, width), dtype=bool)
    mask[0, :] = mask[-1, :] = True
    mask[:, 0] = mask[:, -1] = True
    return idx[mask].tolist()
