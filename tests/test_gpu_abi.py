"""GPU: the whole C ABI (include/geopairs_b200.h), called directly.

* gp_propagate_batch on a torch stream: distances bit-equal to the oracle /
  the reference, direction codes decoding to the reference's parents --
  every source of the config-2 image and 320 sources of config 4 against
  digests of the UNMODIFIED reference's propagations (tests/golden/trees*.npz,
  reference _kernels.py:33-79: parent set on strict improvement only);
* gp_ctx_load on a reused context = a fresh context;
* status mapping (EINVAL, ENOMEM, ECYCLE, EDISAGREE) and the reference's
  check-before-write of fill_from_source (distances.py:132-136);
* the opt-in device agreement check (GP_VERIFY=1, _kernels.py:110-111);
* the batch-size clamp of k_topk (spec_k > 1024).
"""

from __future__ import annotations

import ctypes
import hashlib

import numpy as np
import pytest
import torch

from conftest import load_golden
from paper_2007_16076_b200.configs import CONFIGS, make_image

pytestmark = pytest.mark.gpu


def _ctx(gp, img, conn=8, metric=1):
    from paper_2007_16076_b200 import _lib

    L = _lib.lib()
    isf = img.dtype == np.float32
    px = np.ascontiguousarray(img.astype(np.float32) if isf else img.astype(np.int64))
    h = ctypes.c_void_p()
    _lib.check(L.gp_ctx_create(img.shape[0], img.shape[1], _lib.DTYPE_F32 if isf else _lib.DTYPE_I64,
                               _lib.ptr(px), metric, conn, ctypes.byref(h)))
    return L, h


def _batch(gp, img, sources, conn=8, stream=None):
    """gp_propagate_batch into torch device buffers on `stream` (dist, parent)."""
    from paper_2007_16076_b200 import _lib

    L, h = _ctx(gp, img, conn)
    H, W = img.shape
    N = H * W
    k = len(sources)
    src = torch.as_tensor(np.asarray(sources, dtype=np.int32), device="cuda")
    td = torch.empty((k, N), dtype=torch.float32, device="cuda")
    dr = torch.empty((k, N), dtype=torch.uint8, device="cuda")
    st = stream or torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        _lib.check(L.gp_propagate_batch(h, ctypes.c_void_p(src.data_ptr()), k,
                                        ctypes.c_void_p(td.data_ptr()), ctypes.c_void_p(dr.data_ptr()),
                                        ctypes.c_void_p(st.cuda_stream)))
    st.synchronize()
    L.gp_ctx_destroy(h)
    codes = dr.cpu().numpy().astype(np.int64)
    v = np.arange(N, dtype=np.int64)[None, :]
    parent = np.where(codes == 255, -1, v + (codes // 3 - 1) * W + (codes % 3 - 1))
    return td.cpu().numpy(), parent


def _digest(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).digest()[:16],
                         dtype=np.uint8)


@pytest.mark.parametrize("index", [2, 4])
def test_batch_trees_match_reference_digests(gp, index):
    """Predecessor identity at config scale: cfg2 every source, cfg4 the first
    64 committed + 256 random sources, against the reference's own
    propagations (dist and parent, int64)."""
    g = load_golden(f"trees{index}.npz")
    img = make_image(index)
    srcs = g["src"].astype(np.int64)
    bad_d, bad_p = [], []
    for c0 in range(0, len(srcs), 1024):
        chunk = srcs[c0:c0 + 1024]
        td, par = _batch(gp, img, chunk)
        for i, s in enumerate(chunk):
            d = td[i]
            assert np.all(d == np.round(d))  # integer image: exact integers
            if not np.array_equal(_digest(d.astype(np.int64)), g["dist_digest"][c0 + i]):
                bad_d.append(int(s))
            if not np.array_equal(_digest(par[i]), g["parent_digest"][c0 + i]):
                bad_p.append(int(s))
    assert not bad_d, f"distances differ from the reference for sources {bad_d[:10]}"
    assert not bad_p, f"parents differ from the reference for sources {bad_p[:10]}"


@pytest.mark.parametrize("conn", [8, 4])
def test_batch_fp32_on_torch_stream_matches_oracle(gp, oracle, conn):
    rng = np.random.default_rng(40 + conn)
    img = rng.random((37, 29), dtype=np.float32)
    srcs = rng.choice(img.size, 50, replace=False)
    td, par = _batch(gp, img, srcs, conn=conn, stream=torch.cuda.Stream())
    for i, s in enumerate(srcs):
        d, p = oracle.propagate(img, [int(s)], conn=conn)
        assert np.array_equal(td[i], d)
        assert np.array_equal(par[i], p)


def test_batch_matches_single_propagate(gp):
    img = np.random.default_rng(3).integers(1, 256, (50, 60))
    graph = gp.GridGraph(gp.Image(img), gp.Metric.SUM)
    srcs = [0, 59, 1234, 2999, 1500]
    td, par = _batch(gp, img, srcs)
    for i, s in enumerate(srcs):
        r = graph.propagate([s])
        assert np.array_equal(td[i].astype(np.int64), r.dist)
        assert np.array_equal(par[i], r.parent)


def test_ctx_load_reuse_equals_fresh_ctx(gp):
    from paper_2007_16076_b200 import _lib

    rng = np.random.default_rng(12)
    a = rng.integers(1, 256, (40, 44)).astype(np.uint8)
    b = rng.integers(1, 256, (40, 44)).astype(np.uint8)
    N = a.size

    def run(L, h):
        st = ctypes.c_void_p()
        _lib.check(L.gp_store_create(N, ctypes.byref(st)))
        seq = np.zeros(N, np.int32)
        new = np.zeros(N, np.int64)
        s = _lib.RunStats()
        _lib.check(L.gp_run(h, st, _lib.STRATEGY_FILLING_RATE, 0, 0, _lib.ptr(seq), _lib.ptr(new),
                            ctypes.byref(s)))
        D = np.empty((N, N), np.float32)
        _lib.check(L.gp_store_read(st, _lib.ptr(D), None))
        L.gp_store_destroy(st)
        P = int(s.raw_count)
        return seq[:P].copy(), new[:P].copy(), D, int(s.centroid)

    L, h = _ctx(gp, a)
    run(L, h)
    _lib.check(L.gp_ctx_load(h, _lib.DTYPE_U8, _lib.ptr(np.ascontiguousarray(b))))
    reused = run(L, h)
    L.gp_ctx_destroy(h)
    L2, h2 = _ctx(gp, b.astype(np.int64))
    fresh = run(L2, h2)
    L2.gp_ctx_destroy(h2)
    for x, y in zip(reused, fresh):
        assert np.array_equal(x, y)
    # a rejected image leaves the context usable and unchanged
    bad = b.copy()
    bad[0, 0] = 0
    assert L.gp_version() >= 1
    L3, h3 = _ctx(gp, b.astype(np.int64))
    rc = L3.gp_ctx_load(h3, _lib.DTYPE_U8, _lib.ptr(np.ascontiguousarray(bad)))
    assert rc == _lib.GP_EINVAL and b"[1, 255]" in L3.gp_last_error()
    assert np.array_equal(run(L3, h3)[2], fresh[2])
    L3.gp_ctx_destroy(h3)


def test_status_codes(gp):
    from paper_2007_16076_b200 import _lib

    L = _lib.lib()
    px = np.ones((4, 4), np.int64)
    h = ctypes.c_void_p()
    assert L.gp_ctx_create(4, 4, _lib.DTYPE_I64, _lib.ptr(px), 1, 5, ctypes.byref(h)) == _lib.GP_EINVAL
    assert L.gp_ctx_create(4, 4, 9, _lib.ptr(px), 1, 8, ctypes.byref(h)) == _lib.GP_EINVAL
    assert L.gp_ctx_create(4, 4, _lib.DTYPE_I64, _lib.ptr(px), 1, 8, ctypes.byref(h)) == _lib.GP_OK
    out_d = np.empty(16, np.float32)
    out_p = np.empty(16, np.int32)
    for srcs in ([16], [-1], [3, 3]):
        s = np.asarray(srcs, np.int32)
        assert L.gp_propagate(h, _lib.ptr(s), len(s), _lib.ptr(out_d), _lib.ptr(out_p)) == _lib.GP_EINVAL
    assert L.gp_propagate(h, None, 0, _lib.ptr(out_d), _lib.ptr(out_p)) == _lib.GP_EINVAL
    L.gp_ctx_destroy(h)
    st = ctypes.c_void_p()
    assert L.gp_store_create(70000, ctypes.byref(st)) == _lib.GP_ENOMEM
    assert L.gp_store_create(1, ctypes.byref(st)) == _lib.GP_EINVAL
    with pytest.raises(MemoryError):
        _lib.check(_lib.GP_ENOMEM)
    with pytest.raises(gp.ArrayFullError):
        _lib.check(_lib.GP_EFULL, full_error=gp.ArrayFullError)
    # ECYCLE / EDISAGREE through the store API
    assert L.gp_store_create(3, ctypes.byref(st)) == _lib.GP_OK
    new = ctypes.c_int64()
    par = np.array([1, 0, -1], np.int32)
    td = np.array([0, 1, 2], np.float32)
    assert L.gp_store_fill_tree(st, _lib.ptr(par), _lib.ptr(td), 0.0, ctypes.byref(new)) == _lib.GP_ECYCLE
    L.gp_store_destroy(st)
    assert L.gp_store_create(3, ctypes.byref(st)) == _lib.GP_OK
    par = np.array([-1, 0, 1], np.int32)
    assert L.gp_store_fill_tree(st, _lib.ptr(par), _lib.ptr(np.array([0, 12, 20], np.float32)), 0.0,
                                ctypes.byref(new)) == _lib.GP_OK and new.value == 3
    assert L.gp_store_fill_tree(st, _lib.ptr(par), _lib.ptr(np.array([0, 13, 20], np.float32)), 0.0,
                                ctypes.byref(new)) == _lib.GP_EDISAGREE
    L.gp_store_destroy(st)


def test_fill_source_disagreement_leaves_store_unchanged(gp):
    """distances.py:132-136: the agreement check precedes every write."""
    img = gp.Image(np.random.default_rng(5).integers(1, 256, (6, 7)))
    n = img.size
    store = gp.DistanceArray(n)
    t = gp.build_tree(gp.propagate(img, gp.Metric.SUM, [3]), 3)
    store.fill_from_tree(t)
    D0, M0 = store.dist.copy(), store.mark.copy()
    c0, f0 = store.point_filled_counts.copy(), store.pairs_filled
    d9 = gp.propagate(img, gp.Metric.SUM, [9]).dist
    with pytest.raises(ValueError):
        store.fill_from_source(9, d9 + 2 * (np.arange(n) != 9))
    assert np.array_equal(store.dist, D0) and np.array_equal(store.mark, M0)
    assert np.array_equal(store.point_filled_counts, c0) and store.pairs_filled == f0
    assert store.fill_from_source(9, d9) > 0  # the good map still fills


@pytest.mark.parametrize("isf", [False, True])
def test_verify_mode(gp, monkeypatch, isf):
    rng = np.random.default_rng(21)
    img = rng.random((20, 23), dtype=np.float32) if isf else rng.integers(1, 256, (20, 23))
    base = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    monkeypatch.setenv("GP_VERIFY", "1")
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    assert run.stats["disagreements"] == 0
    assert [s for _, s, _ in run.trace.samples] == [s for _, s, _ in base.trace.samples]
    assert np.array_equal(run.distances.dist, base.distances.dist)
    monkeypatch.setenv("GP_VERIFY_CORRUPT", "0")  # the first commit's new pairs stored +1
    with pytest.raises(ValueError, match="disagree"):
        gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)


def test_spec_k_above_topk_capacity(gp):
    img = np.random.default_rng(8).integers(1, 256, (48, 50))
    base = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    big = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE, spec_k=2048)
    assert [s for _, s, _ in big.trace.samples] == [s for _, s, _ in base.trace.samples]
    assert np.array_equal(big.distances.dist, base.distances.dist)


def test_extrema_and_small_entry_points(gp, ref_small):
    """gp_extrema (compute_extrema_context, strategies.py:104-116) against the
    reference's centroid / dist_from_c / ext; gp_ctx_num_pixels; counts."""
    from conftest import small_cases
    from paper_2007_16076_b200 import _lib

    for i, c in small_cases(ref_small):
        img, metric = c["img"], str(c["metric"])
        m = {"sum": gp.Metric.SUM, "mean": gp.Metric.MEAN, "l1": gp.Metric.L1}[metric]
        ctx = gp.compute_extrema_context(gp.Image(img), m)
        assert ctx.centroid == int(c["centroid"]), i
        assert np.array_equal(np.asarray(ctx.dist_from_c), c["dfc"]), i
        assert np.array_equal(np.asarray(ctx.ext), c["ext"]), i
        graph = gp.GridGraph(gp.Image(img), m)
        assert _lib.lib().gp_ctx_num_pixels(graph.handle) == img.size
    store = gp.DistanceArray(9)
    counts = np.empty(9, np.int32)
    filled = ctypes.c_int64()
    _lib.check(_lib.lib().gp_store_counts(store._st, _lib.ptr(counts), ctypes.byref(filled)))
    assert counts.tolist() == [0] * 9 and filled.value == 0
