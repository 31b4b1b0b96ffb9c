"""GPU parity: the CUDA path against the reference goldens and the oracle.

Integer images: bit-exact distances, identical predecessors, identical source
sequence and counts.  fp32 images: compared with the fp32 restatement
(oracle/); the expected result is bit-exact as well (same fixpoint, same
first writer), and the asserted bar is the north-star tolerance
rel <= 1e-5 on D with identical sequence/counts.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

from conftest import load_golden, small_cases
from paper_2007_16076_b200.configs import CONFIGS, make_image

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def _metric(gp, name):
    return {"sum": gp.Metric.SUM, "mean": gp.Metric.MEAN, "l1": gp.Metric.L1}[name]


def test_propagation_matches_reference_every_source(gp, ref_small):
    for i, c in small_cases(ref_small):
        img, metric = c["img"], str(c["metric"])
        graph = gp.GridGraph(gp.Image(img), _metric(gp, metric))
        for s in range(img.size):
            r = graph.propagate([s])
            assert np.array_equal(r.dist, c["dist"][s]), (i, s)
            # every metric, L1 plateaus (zero-weight edges) included: the exact
            # heap-order K1 reproduces the reference's pop order there
            assert np.array_equal(r.parent, c["parent"][s]), (i, s)


def test_runs_match_reference_small(gp, ref_small):
    for i, c in small_cases(ref_small):
        img, metric = c["img"], str(c["metric"])
        for tag, kind in (("naive", gp.StrategyKind.NAIVE), ("fr", gp.StrategyKind.FILLING_RATE)):
            run = gp.run_strategy(gp.Image(img), _metric(gp, metric), kind)
            assert run.distances.is_complete
            assert np.array_equal(run.distances.dist, c[tag + "_D"]), (i, tag)
            seq = [s for _, s, _ in run.trace.samples]
            assert seq == c[tag + "_seq"].tolist(), (i, tag)
            assert run.trace.adjusted_count == int(c[tag + "_adj"])
            assert np.array_equal(run.distances.point_filled_counts, c[tag + "_counts"])


@pytest.mark.parametrize("conn", [8, 4])
def test_fp32_propagation_matches_oracle(gp, oracle, conn):
    rng = np.random.default_rng(100 + conn)
    for t in range(6):
        h, w = (int(x) for x in rng.integers(3, 24, 2))
        img = rng.random((h, w), dtype=np.float32)
        if t % 2:
            img = (img * 4).round().astype(np.float32) / 4 + 0.25  # ties
        graph = gp.GridGraph(gp.Image(img), gp.Metric.SUM, connectivity=conn)
        for s in rng.choice(h * w, size=min(12, h * w), replace=False):
            r = graph.propagate([int(s)])
            d, p = oracle.propagate(img, [int(s)], conn=conn)
            assert np.array_equal(r.dist, d)
            assert np.array_equal(r.parent, p)


@pytest.mark.parametrize("conn", [8, 4])
def test_fp32_runs_match_oracle(gp, oracle, conn):
    rng = np.random.default_rng(7 + conn)
    for t in range(4):
        h, w = (int(x) for x in rng.integers(4, 20, 2))
        img = rng.random((h, w), dtype=np.float32)
        for kind in ("filling-rate", "naive"):
            o = oracle.run(img, kind, conn=conn)
            k = gp.StrategyKind.FILLING_RATE if kind == "filling-rate" else gp.StrategyKind.NAIVE
            run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, k, connectivity=conn)
            seq = np.array([s for _, s, _ in run.trace.samples])
            assert np.array_equal(seq, o["seq"])
            D = run.distances.dist
            assert np.allclose(D, o["D"], rtol=RTOL, atol=0)
            assert np.array_equal(D, o["D"])  # expected bit-exact


def test_integer_image_large_run_matches_oracle(gp, oracle):
    img = np.random.default_rng(4).integers(1, 256, (24, 40))
    o = oracle.run(img, "filling-rate", nthreads=4)
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE, spec_k=37)
    assert [s for _, s, _ in run.trace.samples] == o["seq"].tolist()
    assert np.array_equal(run.distances.dist, o["D"])


def _digest(D, isf):
    return hashlib.sha256(np.ascontiguousarray(D).astype("<f4" if isf else "<i4").tobytes()).hexdigest()


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
def test_config_matches_golden(gp, index):
    spec = CONFIGS[index]
    g = load_golden(f"cfg{index}.npz")
    img = make_image(index)
    kind = gp.StrategyKind.FILLING_RATE if spec.strategy == "filling-rate" else gp.StrategyKind.NAIVE
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, kind, connectivity=spec.conn, force=True)
    seq = np.array([s for _, s, _ in run.trace.samples])
    assert run.trace.raw_count == int(g["raw"])
    assert run.trace.adjusted_count == int(g["adjusted"])
    assert np.array_equal(seq, g["seq"])
    # per-commit new pairs (the reference's FillingTrace rates) and the extrema centroid
    filled = np.array([int(f * spec.total_pairs) for _, _, f in run.trace.samples], dtype=np.int64)
    assert np.array_equal(np.diff(np.concatenate([[0], filled])), g["new"])
    assert int(run.stats["centroid"]) == int(g["centroid"])
    assert np.array_equal(run.distances.point_filled_counts, np.full(spec.n, spec.n - 1))
    isf = spec.dtype == "f32"
    Dd = run.distances.dist_device()
    si = torch.as_tensor(g["samp_i"].astype(np.int64), device=Dd.device)
    sj = torch.as_tensor(g["samp_j"].astype(np.int64), device=Dd.device)
    samp = Dd[si, sj].cpu().numpy()
    assert np.allclose(samp, g["samp_v"], rtol=RTOL, atol=0)
    assert np.array_equal(samp, g["samp_v"].astype(np.float32))  # expected bit-exact
    # size-independent properties at full size: symmetry, zero diagonal, row checksums
    assert bool((Dd == Dd.T).all())
    assert bool((torch.diagonal(Dd) == 0).all())
    rows = torch.sum(Dd, dim=1, dtype=torch.float64).cpu().numpy()
    assert np.allclose(rows, g["row_sum"], rtol=1e-9, atol=0)
    if spec.n <= 16384:
        assert _digest(Dd.cpu().numpy(), isf) == str(g["d_sha256"])
    else:  # 16 GiB at 256x256: hashed in row blocks (the same bytes in the same order)
        h = hashlib.sha256()
        for r0 in range(0, spec.n, 2048):
            blk = Dd[r0:r0 + 2048].cpu().numpy()
            h.update(np.ascontiguousarray(blk).astype("<f4" if isf else "<i4").tobytes())
        assert h.hexdigest() == str(g["d_sha256"])


@pytest.mark.parametrize("index", [4, 5])
def test_config_through_run_to_host_matches_golden(gp, index):
    """The e2e path at config scale: gp_run_to_host (one-sided tree fills completed at the
    list switch, rows streamed, early bulk send, patch log) delivers the same bytes as the
    golden array -- cfg4 (1 GiB, reference-pinned) and cfg5 (16 GiB, hashed in row blocks)."""
    import ctypes

    import torch

    from paper_2007_16076_b200 import _lib

    spec = CONFIGS[index]
    g = load_golden(f"cfg{index}.npz")
    img = make_image(index)
    isf = spec.dtype == "f32"
    L = _lib.lib()
    n = spec.n
    px = np.ascontiguousarray(img.astype(np.float32) if isf else img)
    dtype = _lib.DTYPE_F32 if isf else _lib.DTYPE_U8
    ctx, st = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(L.gp_ctx_create(spec.shape[0], spec.shape[1], dtype, _lib.ptr(px), 1, spec.conn, ctypes.byref(ctx)))
    _lib.check(L.gp_store_create(n, ctypes.byref(st)))
    try:
        try:
            host = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        except RuntimeError:  # no room for a pinned array of that size: pageable memory works too
            host = torch.empty((n, n), dtype=torch.float32)
        seq = np.zeros(n, np.int32)
        new = np.zeros(n, np.int64)
        stats = _lib.RunStats()
        _lib.check(L.gp_run_to_host(ctx, st, _lib.STRATEGY_FILLING_RATE, 0, 0, _lib.ptr(seq), _lib.ptr(new),
                                    ctypes.byref(stats), ctypes.c_void_p(host.data_ptr())))
        P = int(stats.raw_count)
        assert P == int(g["raw"]) and np.array_equal(seq[:P], g["seq"]) and np.array_equal(new[:P], g["new"])
        H = host.numpy()
        h = hashlib.sha256()
        for r0 in range(0, n, 2048):
            h.update(np.ascontiguousarray(H[r0:r0 + 2048]).astype("<f4" if isf else "<i4").tobytes())
        assert h.hexdigest() == str(g["d_sha256"])
    finally:
        L.gp_store_destroy(st)
        L.gp_ctx_destroy(ctx)


def test_api_known_answers(gp):
    img = gp.Image.from_flat(3, 1, [1, 2, 3])
    r = gp.propagate(img, gp.Metric.SUM, [0])
    assert r.dist.tolist() == [0, 6, 16] and r.parent.tolist() == [-1, 0, 1]
    cheb = np.array([[max(abs(a - 2), abs(b - 2)) for b in range(5)] for a in range(5)]).ravel()
    assert np.array_equal(gp.propagate(gp.Image(np.full((5, 5), 9)), gp.Metric.SUM, [12]).dist, 36 * cheb)
    with pytest.raises(ValueError):
        gp.propagate(img, gp.Metric.SUM, [])
    with pytest.raises(ValueError):
        gp.propagate(img, gp.Metric.SUM, [0, 0])
    with pytest.raises(ValueError):
        gp.propagate(img, gp.Metric.SUM, [3])


def test_store_fills_and_errors(gp):
    def chain(d):
        n = len(d)
        return gp.GeodesicTree(0, np.array([-1] + list(range(n - 1))), np.array(d), [], [])

    store = gp.DistanceArray(3)
    assert store.fill_from_tree(chain([0, 12, 20])) == 3
    assert store.dist[1, 2] == store.dist[2, 1] == 8
    assert store.is_complete and store.fill_from_tree(chain([0, 12, 20])) == 0
    with pytest.raises(ValueError):
        store.fill_from_tree(chain([0, 13, 20]))
    with pytest.raises(ValueError):
        gp.DistanceArray(3).fill_from_tree(
            gp.GeodesicTree(2, np.array([1, 0, -1]), np.array([0, 1, 2]), [], []))
    with pytest.raises(gp.SizeGuardError):
        gp.DistanceArray(gp.MAX_PIXELS + 1)
    rng = np.random.default_rng(91)
    img = gp.Image(rng.integers(1, 256, (5, 5)))
    s2 = gp.DistanceArray(25)
    for _ in range(6):
        root = int(rng.integers(25))
        s2.fill_from_tree(gp.build_tree(gp.propagate(img, gp.Metric.SUM, [root]), root))
        assert s2.pairs_filled == (int(s2.mark.sum()) - 25) // 2
        assert np.array_equal(s2.point_filled_counts, s2.mark.sum(axis=0) - 1)
    s3 = gp.DistanceArray(25)
    d0 = gp.propagate(img, gp.Metric.SUM, [0]).dist
    assert s3.fill_from_source(0, d0) == 24
    with pytest.raises(ValueError):
        s3.fill_from_source(0, d0 + 2)


def test_host_selected_strategies_complete(gp, ref_small):
    img = gp.Image(np.random.default_rng(42).integers(1, 256, (6, 6)))
    oracle_D = gp.brute_force_oracle(img).dist
    for kind in gp.StrategyKind:
        run = gp.run_strategy(img, gp.Metric.SUM, kind, seed=0)
        assert run.distances.is_complete
        assert np.array_equal(run.distances.dist, oracle_D), kind


def test_other_strategies_match_reference(gp):
    """Spiral, spiral-repulsion and extrema: host selectors
    with device propagation and fills vs runs of the reference itself
    (tests/golden/make_golden.py strategies): sequence, D, counts, adjusted
    count and the exact filling rates."""
    from fractions import Fraction

    g = load_golden("ref_strategies.npz")
    kinds = {"spiral": gp.StrategyKind.SPIRAL, "repulsion": gp.StrategyKind.SPIRAL_REPULSION,
             "extrema": gp.StrategyKind.EXTREMA}
    for i in range(int(g["n_cases"])):
        k = f"c{i}_"
        img = g[k + "img"]
        metric = _metric(gp, str(g[k + "metric"]))
        for tag, kind in kinds.items():
            run = gp.run_strategy(gp.Image(img), metric, kind, int(g[k + "seed"]), repulsion=int(g[k + "rep"]))
            seq = [s for _, s, _ in run.trace.samples]
            assert seq == g[k + tag + "_seq"].tolist(), (i, tag)
            assert np.array_equal(run.distances.dist, g[k + tag + "_D"]), (i, tag)
            assert np.array_equal(run.distances.point_filled_counts, g[k + tag + "_counts"]), (i, tag)
            assert run.trace.adjusted_count == int(g[k + tag + "_adj"]), (i, tag)
            rates = [Fraction(int(a), int(b)) for a, b in g[k + tag + "_rates"]]
            assert [f for _, _, f in run.trace.samples] == rates, (i, tag)


def test_extrema_config2_matches_reference(gp):
    """The device extrema selector (K3 key variant) against the reference's
    own EXTREMA run on the config-2 image (tests/golden/extrema2.npz)."""
    g = load_golden("extrema2.npz")
    spec = CONFIGS[2]
    run = gp.run_strategy(gp.Image(make_image(2)), gp.Metric.SUM, gp.StrategyKind.EXTREMA)
    assert [s for _, s, _ in run.trace.samples] == g["seq"].tolist()
    filled = np.array([int(f * spec.total_pairs) for _, _, f in run.trace.samples], dtype=np.int64)
    assert np.array_equal(np.diff(np.concatenate([[0], filled])), g["new"])
    assert run.trace.adjusted_count == int(g["adjusted"])
    assert _digest(run.distances.dist_device().cpu().numpy(), False) == str(g["d_sha256"])
