"""GPU: edge cases and invariances of the device path (against the oracle)."""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _seq(run):
    return [s for _, s, _ in run.trace.samples]


@pytest.mark.parametrize("shape", [(1, 2), (1, 7), (9, 1), (2, 2), (3, 1), (2, 5), (17, 3)])
def test_degenerate_shapes(gp, oracle, shape):
    img = np.random.default_rng(sum(shape)).integers(1, 256, shape)
    for kind, k in (("filling-rate", gp.StrategyKind.FILLING_RATE), ("naive", gp.StrategyKind.NAIVE)):
        o = oracle.run(img, kind)
        run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, k)
        assert _seq(run) == o["seq"].tolist()
        assert np.array_equal(run.distances.dist, o["D"])
        assert run.trace.adjusted_count == o["adjusted"]


def test_mean_metric_runs(gp, oracle):
    img = np.random.default_rng(3).integers(1, 256, (11, 13))
    o = oracle.run(img, "filling-rate", metric="mean")
    run = gp.run_strategy(gp.Image(img), gp.Metric.MEAN, gp.StrategyKind.FILLING_RATE)
    assert _seq(run) == o["seq"].tolist()
    assert np.array_equal(run.distances.dist, o["D"])


def test_naive_with_tree(gp, oracle):
    img = np.random.default_rng(5).integers(1, 256, (9, 10))
    o = oracle.run(img, "naive", naive_with_tree=True)
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.NAIVE, naive_with_tree=True)
    assert _seq(run) == o["seq"].tolist()
    assert np.array_equal(run.distances.dist, o["D"])
    plain = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.NAIVE)
    assert run.trace.raw_count <= plain.trace.raw_count  # test_strategies.py:335-342


def test_fp32_single_zero_pixel_and_ties(gp, oracle):
    rng = np.random.default_rng(9)
    img = (rng.integers(1, 4, (14, 12)) / 4).astype(np.float32)
    img[5, 5] = 0.0
    for conn in (8, 4):
        o = oracle.run(img, "filling-rate", conn=conn)
        run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE,
                              connectivity=conn)
        assert _seq(run) == o["seq"].tolist()
        assert np.array_equal(run.distances.dist, o["D"])


def test_l1_distances_exact(gp, oracle):
    rng = np.random.default_rng(10)
    img = rng.integers(1, 4, (8, 9))  # many zero-weight edges
    graph = gp.GridGraph(gp.Image(img), gp.Metric.L1)
    for s in range(0, img.size, 7):
        d, p0 = oracle.propagate(img, [s], metric="l1")
        r = graph.propagate([s])
        assert np.array_equal(r.dist, d)
        assert np.array_equal(r.parent, p0)  # heap order on the plateaus
        # and the parents form a valid shortest-path forest
        for v in range(img.size):
            p = int(r.parent[v])
            if p >= 0:
                assert r.dist[v] == r.dist[p] + gp.edge_weight(gp.Image(img), gp.Metric.L1, p, v)
        _check_tree(np.asarray(r.dist, dtype=np.float32), r.parent, img, 8, "l1", [s])


@pytest.mark.parametrize("shape", [(8, 9), (21, 17), (40, 44)])
def test_l1_plateau_runs_match_oracle(gp, oracle, shape):
    """L1 on plateau images (zero-weight edges): the exact heap-order K1 gives
    the reference's trees, so the whole run -- source sequence, counts and the
    array -- equals the oracle's (pinned to the reference on L1 by
    tests/test_oracle.py)."""
    img = np.random.default_rng(12).integers(1, 4, shape) * 5
    for kind in ("filling-rate", "naive"):
        o = oracle.run(img, kind, metric="l1")
        k = gp.StrategyKind.FILLING_RATE if kind == "filling-rate" else gp.StrategyKind.NAIVE
        run = gp.run_strategy(gp.Image(img), gp.Metric.L1, k)
        assert run.distances.is_complete
        assert _seq(run) == o["seq"].tolist()
        assert np.array_equal(run.distances.dist, o["D"])
        assert run.trace.adjusted_count == o["adjusted"]


def test_fp32_zero_pixels_exact_heap(gp, oracle):
    """fp32 image with adjacent zero pixels (SUM weight 0 between them): the
    exact heap-order K1 path, against the oracle's propagations and run."""
    rng = np.random.default_rng(77)
    img = rng.random((13, 15), dtype=np.float32)
    img[3:6, 4:9] = 0.0
    graph = gp.GridGraph(gp.Image(img), gp.Metric.SUM)
    for s in (0, 50, 64, 194):
        r = graph.propagate([s])
        d, p = oracle.propagate(img, [s])
        assert np.array_equal(r.dist, d) and np.array_equal(r.parent, p)
    o = oracle.run(img, "filling-rate")
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    assert _seq(run) == o["seq"].tolist()
    assert np.array_equal(run.distances.dist, o["D"])


@pytest.mark.parametrize("env", [
    {"GP_SPEC_K": "7"}, {"GP_SPEC_K": "1000"}, {"GP_LIST_ALPHA": "0"}, {"GP_LIST_ALPHA": "1000"},
    {"GP_UNITS_PER_WARP": "4"}, {"GP_DELTA_FACTOR": "inf"}, {"GP_DELTA_FACTOR": "0.5"},
    {"GP_PROP_THREADS": "256"}, {"GP_BARRIER": "sw"}, {"GP_PIPELINE": "0"}, {"GP_FILL_QUEUE": "0"},
    {"GP_FILL_UNROLL": "1"}, {"GP_FILL_UNROLL": "8"}, {"GP_PROP_MINB": "2"},
    {"GP_PROP_CLUSTER": "2"}, {"GP_PROP_CLUSTER": "2", "GP_LIST_ALPHA": "1000"}, {"GP_VERIFY": "1"},
    {"GP_CAND": "0"}, {"GP_LPT": "0"}, {"GP_COMMIT_SPLIT": "0"}, {"GP_LIST_CFG": "2"}, {"GP_LIST_CFG": "1"}, {"GP_PROP_LEAN": "0"}, {"GP_PROP_MC": "0"},
    {"GP_COMPACT_DIV": "1"}, {"GP_COMPACT_DIV": "64"}, {"GP_LIST_ALPHA": "1", "GP_COMPACT_DIV": "1"},
    # batched list-mode commits (k_commit_lb): forced on this small map, packed / direct test,
    # record overflow path, longer list phases, one commit per step
    {"GP_LIST_BATCH": "1"}, {"GP_LIST_BATCH": "1", "GP_LB_PACK_MIN": "0"}, {"GP_LIST_BATCH": "1", "GP_LB_PACK": "0"},
    {"GP_LIST_BATCH": "1", "GP_LB_RCAP": "0"}, {"GP_LIST_BATCH": "1", "GP_LB_RCAP": "3", "GP_LB_PACK_MIN": "0"},
    {"GP_LIST_BATCH": "1", "GP_LIST_ALPHA": "6"}, {"GP_LIST_BATCH": "1", "GP_LIST_ALPHA": "6", "GP_LB_PACK_MIN": "0"},
    {"GP_LIST_BATCH": "1", "GP_COMPACT_DIV": "1"}, {"GP_LIST_BATCH": "1", "GP_CAND": "0"},
    {"GP_LIST_BATCH": "0"},
    # two-sided tree fills (no transpose-merge pass)
    {"GP_ONE_SIDED": "0"}, {"GP_ONE_SIDED": "0", "GP_LIST_BATCH": "1"},
])
def test_tuning_knobs_do_not_change_results(gp, oracle, env, monkeypatch):
    img = np.random.default_rng(11).random((24, 20), dtype=np.float32)
    o = oracle.run(img, "filling-rate")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    assert _seq(run) == o["seq"].tolist()
    assert np.array_equal(run.distances.dist, o["D"])
    assert np.array_equal(run.distances.point_filled_counts, np.full(img.size, img.size - 1))


def test_brute_force_oracle_and_apgd(gp):
    img = gp.Image(np.random.default_rng(12).integers(1, 256, (7, 7)))
    bf = gp.brute_force_oracle(img)
    fr = gp.run_strategy(img, gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    assert np.array_equal(bf.dist, fr.distances.dist)
    blob = fr.distances.to_bytes()
    assert blob[:4] == gp.APGD_MAGIC and blob[4] == 1
    n = img.size
    grid = np.frombuffer(blob, dtype="<u8", offset=9).reshape(n, n)
    assert np.array_equal(grid.astype(np.int64), bf.dist)


def test_metric_properties_of_completed_array(gp):
    # test_acceptance.py:519-531: symmetric, zero diagonal, triangle inequality
    img = gp.Image(np.random.default_rng(13).integers(1, 256, (15, 15)))
    D = gp.run_strategy(img, gp.Metric.SUM, gp.StrategyKind.FILLING_RATE).distances.dist
    assert np.array_equal(D, D.T) and (np.diag(D) == 0).all()
    rng = np.random.default_rng(9)
    x, y, z = (rng.integers(0, D.shape[0], 10_000) for _ in range(3))
    assert int((D[x, z] > D[x, y] + D[y, z]).sum()) == 0


@pytest.mark.parametrize("shape,kind,cap,cut", [((40, 37), 1, 0, None), ((64, 64), 1, 0, None), ((23, 30), 0, 0, None),
                                                ((64, 64), 1, 3, None), ((64, 64), 1, 0, 10 ** 9),
                                                ((64, 64), 1, 0, 20000), ((96, 100), 1, 0, 2000000),
                                                ((96, 100), 2, 0, 100000), ((96, 100), 1, 0, -1)])
def test_run_to_host_streams_the_same_array(gp, shape, kind, cap, cut, monkeypatch):
    """gp_run_to_host (rows streamed during the run) == gp_run + gp_store_read;
    cap > 0: GP_E2E_CAP (short commit launches once half the rows are done);
    cut: GP_E2E_CUT with the batched list kernel (open rows sent early once that many
    pairs are left, later fills patched into the host array from the device's log)."""
    import ctypes

    if cap:
        monkeypatch.setenv("GP_E2E_CAP", str(cap))
    if cut is not None:
        monkeypatch.setenv("GP_E2E_CUT", str(cut))
        monkeypatch.setenv("GP_LIST_BATCH", "1")
    if cut == -1:  # also: two-sided fills, one round of lookahead
        monkeypatch.setenv("GP_ONE_SIDED", "0")
        monkeypatch.setenv("GP_E2E_LOOKAHEAD", "1")
    if cut == 20000:  # also: the host-driven round loop (two-sided fills, rows sent at the end)
        monkeypatch.setenv("GP_PIPELINE", "0")

    import torch

    from paper_2007_16076_b200 import _lib

    L = _lib.lib()
    img = np.random.default_rng(shape[0] * 7 + kind).integers(1, 256, shape).astype(np.int64)
    n = img.size
    ctx = ctypes.c_void_p()
    st = ctypes.c_void_p()
    _lib.check(L.gp_ctx_create(shape[0], shape[1], 0, _lib.ptr(img), 1, 8, ctypes.byref(ctx)))
    _lib.check(L.gp_store_create(n, ctypes.byref(st)))
    try:
        seq = np.zeros(n, np.int32)
        new = np.zeros(n, np.int64)
        stats = _lib.RunStats()
        _lib.check(L.gp_run(ctx, st, kind, 0, 0, _lib.ptr(seq), _lib.ptr(new), ctypes.byref(stats)))
        ref = np.empty((n, n), np.float32)
        _lib.check(L.gp_store_read(st, _lib.ptr(ref), None))
        for pinned in (True, False):
            host = torch.full((n, n), -7.0, dtype=torch.float32, pin_memory=pinned)
            seq2 = np.zeros(n, np.int32)
            _lib.check(L.gp_run_to_host(ctx, st, kind, 0, 0, _lib.ptr(seq2), None, ctypes.byref(stats),
                                        ctypes.c_void_p(host.data_ptr())))
            assert np.array_equal(seq2, seq)
            assert np.array_equal(host.numpy(), ref)
    finally:
        L.gp_store_destroy(st)
        L.gp_ctx_destroy(ctx)


@pytest.mark.parametrize("pipeline", ["0", "1"])
def test_run_loops_agree_on_a_larger_image(gp, oracle, pipeline, monkeypatch):
    """Host-driven and device-gated run loops (many misses, a list switch) vs the oracle."""
    img = np.random.default_rng(21).random((48, 40), dtype=np.float32)
    o = oracle.run(img, "filling-rate", nthreads=4)
    monkeypatch.setenv("GP_PIPELINE", pipeline)
    monkeypatch.setenv("GP_SPEC_K", "37")
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    assert _seq(run) == o["seq"].tolist()
    assert np.array_equal(run.distances.dist, o["D"])


@pytest.mark.parametrize("kind", ["filling-rate", "extrema"])
@pytest.mark.parametrize("isint", [True, False])
def test_batched_list_commits_equal_single_commits(gp, kind, isint, monkeypatch):
    """k_commit_lb (several commits per grid step, default above 8192 pixels) against the
    one-commit-per-step list kernel on a 96x100 map: same sequence, same new pairs per
    commit, same array -- for the filling-rate and the extrema keys (the configs' goldens pin
    the filling-rate path to the reference / oracle)."""
    rng = np.random.default_rng(33)
    img = rng.integers(1, 256, (96, 100)) if isint else rng.random((96, 100), dtype=np.float32)
    sk = gp.StrategyKind.FILLING_RATE if kind == "filling-rate" else gp.StrategyKind.EXTREMA
    out = []
    for env in ({"GP_LIST_BATCH": "0"}, {"GP_LIST_BATCH": "1"}, {"GP_LIST_BATCH": "1", "GP_LB_PACK_MIN": "0"},
                {"GP_LIST_BATCH": "1", "GP_LB_RCAP": "2"}):
        for k in ("GP_LIST_BATCH", "GP_LB_PACK_MIN", "GP_LB_RCAP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, sk)
        D = run.distances.dist
        out.append((_seq(run), [c for _, _, c in run.trace.samples], hashlib.sha256(D.tobytes()).hexdigest()))
        assert np.array_equal(D, D.T)
    for o in out[1:]:
        assert o[0] == out[0][0], "committed sequence differs"
        assert o[1] == out[0][1], "per-commit fill counts differ"
        assert o[2] == out[0][2], "distance array differs"


def _check_tree(dist, parent, img, conn, metric, sources):
    """parent is a valid shortest-path forest of dist (zero-weight plateaus)."""
    H, W = img.shape
    f = img.astype(np.float32).ravel()
    N = H * W
    roots = set(int(s) for s in sources)
    for v in range(N):
        p = int(parent[v])
        if v in roots:
            assert p == -1
            continue
        dr, dc = p // W - v // W, p % W - v % W
        assert max(abs(dr), abs(dc)) == 1 and (conn == 8 or abs(dr) + abs(dc) == 1)
        a, b = np.float32(f[p]), np.float32(f[v])
        w = {"sum": np.float32(2) * (a + b), "mean": a + b, "l1": np.float32(2) * abs(a - b)}[metric]
        assert np.float32(dist[p] + w) == dist[v]
    # acyclic: every chain reaches a root within N steps
    done = np.zeros(N, dtype=bool)
    for v in range(N):
        chain, x = [], v
        while not done[x] and parent[x] >= 0:
            chain.append(x)
            x = int(parent[x])
            assert len(chain) <= N, "parent cycle"
        assert parent[x] >= 0 or x in roots or done[x]
        done[chain] = True
        done[x] = True


@pytest.mark.parametrize("shape,conn,metric,isint", [
    ((150, 140), 8, "sum", False),
    ((150, 140), 4, "sum", False),
    ((131, 160), 8, "mean", True),
    ((256, 256), 8, "sum", False),
    ((64, 1024), 8, "sum", True),
    ((160, 120), 8, "l1", True),
])
def test_global_scratch_propagation_matches_oracle(gp, oracle, shape, conn, metric, isint):
    """Maps above the shared-memory limit run K1's global-scratch variant
    (three trees per SM, 4-bit parent codes): distances bit-exact, parents
    identical (positive weights) or a valid shortest-path tree (L1 plateaus)."""
    rng = np.random.default_rng(sum(shape) + conn)
    if isint:
        img = rng.integers(1, 256, shape)
        if metric == "l1":
            img = (img // 64 + 1) * 10  # plateaus: zero-weight edges
    else:
        img = rng.random(shape, dtype=np.float32)
    m = {"sum": gp.Metric.SUM, "mean": gp.Metric.MEAN, "l1": gp.Metric.L1}[metric]
    graph = gp.GridGraph(gp.Image(img), m, connectivity=conn)
    N = shape[0] * shape[1]
    srcs = [0, N - 1, N // 2 + shape[1] // 3] + [int(x) for x in rng.choice(N, 2, replace=False)]
    for s in srcs:
        r = graph.propagate([s])
        d, p = oracle.propagate(img, [s], conn=conn, metric=metric)
        assert np.array_equal(np.asarray(r.dist), d), s
        assert np.array_equal(r.parent, p), s  # L1 plateaus: heap order (exact K1)
        if metric == "l1":
            _check_tree(np.asarray(r.dist, dtype=np.float32), r.parent, img, conn, metric, [s])


@pytest.mark.parametrize("shape,conn,isint", [((64, 1024), 8, True), ((256, 256), 4, False)])
def test_max_size_runs_rows_equal_propagations(gp, oracle, shape, conn, isint):
    """Maximum-size maps (65 536 pixels; a non-square one and a 4-connected
    fp32 one -- shapes no BASELINE config uses): the completed array is
    symmetric with a zero diagonal, every count is N-1, and row s equals the
    oracle's propagation from s (D[s][x] = geodesic distance s -> x): exactly
    for integer images; for fp32 images within rounding, since an entry holds
    the difference of two distances of the tree that filled it."""
    rng = np.random.default_rng(sum(shape) + conn)
    img = rng.integers(1, 256, shape) if isint else rng.random(shape, dtype=np.float32)
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE,
                          connectivity=conn, force=True)
    N = shape[0] * shape[1]
    assert run.distances.is_complete
    assert np.array_equal(run.distances.point_filled_counts, np.full(N, N - 1))
    Dd = run.distances.dist_device()
    assert bool((torch.diagonal(Dd) == 0).all())
    for r0 in range(0, N, 8192):  # symmetry in row blocks (16 GiB array)
        assert bool((Dd[r0:r0 + 8192] == Dd[:, r0:r0 + 8192].T).all())
    for s in [0, N - 1] + [int(x) for x in rng.choice(N, 3, replace=False)]:
        d, _ = oracle.propagate(img, [s], conn=conn)
        row = Dd[s].cpu().numpy()
        if isint:
            assert np.array_equal(row, np.asarray(d, dtype=np.float32)), s
        else:
            assert np.allclose(row, d, rtol=1e-4, atol=1e-6), s


@pytest.mark.parametrize("shape,conn", [((7, 9), 8), ((9, 7), 4), ((1, 13), 8), ((16, 17), 8), ((33, 30), 4)])
@pytest.mark.parametrize("isint", [True, False])
def test_cluster_propagation_small_maps_match_oracle(gp, oracle, monkeypatch, shape, conn, isint):
    """The 2-CTA cluster K1 (GP_PROP_CLUSTER=2 forces it on maps that fit one
    SM) against the oracle: odd pixel counts, single rows, 4/8-connectivity."""
    rng = np.random.default_rng(shape[0] * 100 + shape[1] + conn)
    img = rng.integers(1, 256, shape) if isint else rng.random(shape, dtype=np.float32)
    monkeypatch.setenv("GP_PROP_CLUSTER", "2")
    for kind, k in (("filling-rate", gp.StrategyKind.FILLING_RATE), ("naive", gp.StrategyKind.NAIVE)):
        o = oracle.run(img, kind, conn=conn, naive_with_tree=kind == "naive")
        run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, k, connectivity=conn,
                              naive_with_tree=kind == "naive")
        assert _seq(run) == o["seq"].tolist()
        assert np.array_equal(run.distances.dist, o["D"])


@pytest.mark.parametrize("shape,conn,metric,isint", [
    ((140, 130), 8, "sum", False), ((131, 160), 4, "mean", True), ((133, 137), 8, "sum", True),
])
def test_cluster_and_single_cta_k1_runs_identical(gp, monkeypatch, shape, conn, metric, isint):
    """Maps above one SM's shared memory: the cluster K1 (default) and the
    single-CTA global-scratch K1 (GP_PROP_CLUSTER=0) give the same run --
    source sequence, new pairs per commit, and the whole distance array."""
    rng = np.random.default_rng(sum(shape))
    img = rng.integers(1, 256, shape) if isint else rng.random(shape, dtype=np.float32)
    m = {"sum": gp.Metric.SUM, "mean": gp.Metric.MEAN}[metric]
    out = []
    for knob in ("1", "0"):
        monkeypatch.setenv("GP_PROP_CLUSTER", knob)
        run = gp.run_strategy(gp.Image(img), m, gp.StrategyKind.FILLING_RATE, connectivity=conn, force=True)
        Dd = run.distances.dist_device()
        h = hashlib.sha256(Dd.cpu().numpy().tobytes()).hexdigest()
        out.append(([s for _, s, _ in run.trace.samples], [f for _, _, f in run.trace.samples], h))
        del run, Dd
    assert out[0] == out[1]


@pytest.mark.parametrize("shape,metric,conn", [((300, 300), "sum", 8), ((257, 263), "mean", 4),
                                               ((260, 260), "l1", 8)])
def test_propagation_contexts_above_65536_pixels(gp, oracle, shape, metric, conn):
    """Images above 65 536 pixels serve propagations (the reference's
    GridGraph has no size limit): the whole-GPU K1 against the oracle --
    distances and parents, L1 plateaus through the sequential heap path --
    and the extrema context; stores and runs of that size are refused."""
    rng = np.random.default_rng(sum(shape))
    img = rng.integers(1, 256, shape)
    if metric == "l1":
        img = (img // 64 + 1) * 10  # plateaus
    m = {"sum": gp.Metric.SUM, "mean": gp.Metric.MEAN, "l1": gp.Metric.L1}[metric]
    graph = gp.GridGraph(gp.Image(img), m, connectivity=conn)
    N = img.size
    for srcs in ([0], [N - 1], [N // 2 + 7], [5, N // 3, N - 40]):
        r = graph.propagate(srcs)
        d, p = oracle.propagate(img, srcs, conn=conn, metric=metric)
        assert np.array_equal(r.dist, d), srcs
        assert np.array_equal(r.parent, p), srcs
    if metric != "l1":
        ctx = gp.compute_extrema_context(gp.Image(img), m, connectivity=conn)
        cen, dfc, ext = oracle.extrema(img, conn=conn, metric=metric)
        assert ctx.centroid == cen
        assert np.array_equal(np.asarray(ctx.dist_from_c), dfc) and np.array_equal(np.asarray(ctx.ext), ext)
    with pytest.raises(MemoryError):
        gp.DistanceArray(N, force=True)
