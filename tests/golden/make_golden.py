"""Generate the committed golden fixtures under tests/golden/.

Run in the build container (NOT on the GPU box -- /root/reference does not
exist there):

    python tests/golden/make_golden.py small      # reference, tiny images
    python tests/golden/make_golden.py strategies # reference: spiral / repulsion / extrema runs
    python tests/golden/make_golden.py harness    # reference: test images, experiment CSVs
    python tests/golden/make_golden.py cfg 2      # reference itself (int config)
    python tests/golden/make_golden.py cfg 4      # reference itself, force=True
    python tests/golden/make_golden.py cfg 1|3|5  # fp32 restatement (oracle/)
    python tests/golden/make_golden.py apgd       # reference: APGD dumps (partial + complete)
    python tests/golden/make_golden.py extrema 2  # reference: EXTREMA strategy on the cfg2 image
    python tests/golden/make_golden.py trees 2    # reference: every source of cfg2
    python tests/golden/make_golden.py trees 4    # reference: 256 sampled + first 64 committed

Integer configs (2, 4) and every ``small`` case come from the UNMODIFIED
reference package imported from /root/reference/pkg/src.  The reference
rejects fp32 images and 4-connectivity (grid.py:49-57, propagation.py:13), so
configs 1, 3 and 5 come from the fp32 restatement in oracle/, whose integer
mode is pinned bit-for-bit to the reference by the ``small`` fixtures and
configs 2/4 (tests/test_oracle.py).

Fixture contents per config (kept small enough to commit):
  seq, new (pairs per commit), raw, adjusted, centroid, visits (oracle only),
  d_sha256 (sha256 of D as little-endian int32 for int configs / float32),
  row_sum (float64 per-row sums of D), samp_i/samp_j/samp_v (random entries),
  tree_src/tree_dist/tree_parent (propagations of the first committed sources).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2007_16076_b200.configs import CONFIGS, make_image  # noqa: E402

N_SAMPLES = 100_000
N_TREES = 4


def d_digest(D: np.ndarray, isf: bool) -> str:
    arr = D.astype("<f4" if isf else "<i4")
    return hashlib.sha256(arr.tobytes()).hexdigest()


def _samples(D: np.ndarray, seed: int):
    n = D.shape[0]
    rng = np.random.default_rng(seed)
    i = rng.integers(0, n, N_SAMPLES)
    j = rng.integers(0, n, N_SAMPLES)
    return i.astype(np.int32), j.astype(np.int32), D[i, j]


def _ref():
    sys.path.insert(0, "/root/reference/pkg/src")
    import geopairs  # noqa: F401

    return geopairs


def make_small():
    gp = _ref()
    rng = np.random.default_rng(2007)
    out = {}
    cases = 0
    metrics = [gp.Metric.SUM, gp.Metric.MEAN, gp.Metric.L1]
    for t in range(48):
        h, w = (int(x) for x in rng.integers(1, 11, 2))
        if h * w < 2:
            continue
        img = rng.integers(1, 256, (h, w))
        if t % 4 == 1:  # tie-heavy images: few grey levels
            img = rng.integers(1, 4, (h, w))
        metric = metrics[t % 3] if t % 4 != 3 else gp.Metric.SUM
        image = gp.Image(img)
        graph = gp.GridGraph(image, metric)
        n = h * w
        dist = np.stack([graph.propagate([s]).dist for s in range(n)])
        parent = np.stack([graph.propagate([s]).parent for s in range(n)])
        k = f"c{cases}_"
        out[k + "img"] = img.astype(np.int64)
        out[k + "metric"] = np.array(metric.value)
        out[k + "dist"] = dist
        out[k + "parent"] = parent
        ctx = gp.compute_extrema_context(image, metric)
        out[k + "centroid"] = np.array(ctx.centroid)
        out[k + "dfc"] = ctx.dist_from_c
        out[k + "ext"] = ctx.ext
        for kind in (gp.StrategyKind.NAIVE, gp.StrategyKind.FILLING_RATE):
            run = gp.run_strategy(image, metric, kind)
            tag = "naive" if kind is gp.StrategyKind.NAIVE else "fr"
            out[k + tag + "_D"] = run.distances.dist
            out[k + tag + "_seq"] = np.array([s for _, s, _ in run.trace.samples], dtype=np.int64)
            out[k + tag + "_adj"] = np.array(run.trace.adjusted_count)
            out[k + tag + "_counts"] = np.array(run.distances.point_filled_counts)
        cases += 1
    out["n_cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "ref_small.npz"), **out)
    print("small cases:", cases)


def make_strategies():
    """The other three selectors, run by the reference:
    sequence, D, counts, adjusted count per image, seed and repulsion."""
    gp = _ref()
    rng = np.random.default_rng(16076)
    out = {}
    cases = 0
    kinds = [(gp.StrategyKind.SPIRAL, "spiral"), (gp.StrategyKind.SPIRAL_REPULSION, "repulsion"),
             (gp.StrategyKind.EXTREMA, "extrema")]
    for t in range(16):
        h, w = (int(x) for x in rng.integers(3, 13, 2))
        img = rng.integers(1, 256, (h, w))
        if t % 4 == 1:
            img = rng.integers(1, 4, (h, w))  # tie-heavy
        metric = gp.Metric.SUM if t % 3 else gp.Metric.MEAN
        seed = int(rng.integers(0, 1000))
        rep = 1 + t % 4
        image = gp.Image(img)
        k = f"c{cases}_"
        out[k + "img"] = img.astype(np.int64)
        out[k + "metric"] = np.array(metric.value)
        out[k + "seed"] = np.array(seed)
        out[k + "rep"] = np.array(rep)
        for kind, tag in kinds:
            run = gp.run_strategy(image, metric, kind, seed, repulsion=rep)
            out[k + tag + "_D"] = run.distances.dist
            out[k + tag + "_seq"] = np.array([s for _, s, _ in run.trace.samples], dtype=np.int64)
            out[k + tag + "_adj"] = np.array(run.trace.adjusted_count)
            out[k + tag + "_counts"] = np.array(run.distances.point_filled_counts)
            out[k + tag + "_rates"] = np.array([[f.numerator, f.denominator] for _, _, f in run.trace.samples],
                                               dtype=np.int64)
        cases += 1
    out["n_cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "ref_strategies.npz"), **out)
    print("strategy cases:", cases)


def make_harness():
    """Reference test-image families and a small experiment's CSV reports."""
    gp = _ref()
    from geopairs.harness import (GeneratorKind, generate_image, hairpin_corridor_mask,
                                  run_experiment, write_report_csv, write_trace_csv)
    out = {}
    sizes = [(25, 25), (12, 9), (7, 16), (31, 20)]
    for kind in GeneratorKind:
        for si, size in enumerate(sizes):
            for seed in (0, 3, 19):
                out[f"img_{kind.value}_{si}_{seed}"] = generate_image(kind, size, seed).pixels.astype(np.int64)
    for si, (w, h) in enumerate(sizes):
        out[f"mask_{si}"] = hairpin_corridor_mask(w, h)
    images = [(f"{k.value}8", generate_image(k, (8, 7), 5)) for k in GeneratorKind]
    kinds = [gp.StrategyKind.NAIVE, gp.StrategyKind.SPIRAL, gp.StrategyKind.SPIRAL_REPULSION,
             gp.StrategyKind.EXTREMA, gp.StrategyKind.FILLING_RATE]
    rep = run_experiment(images, [gp.Metric.SUM, gp.Metric.MEAN], kinds, [0, 1], verify=True)
    out["trace_csv"] = np.frombuffer(write_trace_csv(rep.records), dtype=np.uint8)
    out["report_csv"] = np.frombuffer(write_report_csv(rep), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "ref_harness.npz"), **out)
    print("harness fixtures:", len(out))


def make_cfg(index: int, nthreads: int):
    spec = CONFIGS[index]
    img = make_image(index)
    isf = spec.dtype == "f32"
    t0 = time.time()
    if not isf:
        gp = _ref()
        image = gp.Image(img.astype(np.int64))
        kind = gp.StrategyKind.FILLING_RATE if spec.strategy == "filling-rate" else gp.StrategyKind.NAIVE
        run = gp.run_strategy(image, gp.Metric.SUM, kind, force=True)
        D = run.distances.dist
        seq = np.array([s for _, s, _ in run.trace.samples], dtype=np.int64)
        A = spec.total_pairs
        filled = np.array([int(tau * A) for _, _, tau in run.trace.samples], dtype=np.int64)
        new = np.diff(np.concatenate([[0], filled]))
        raw, adjusted = run.trace.raw_count, run.trace.adjusted_count
        centroid = gp.compute_extrema_context(image, gp.Metric.SUM).centroid if spec.strategy != "naive" else -1
        graph = gp.GridGraph(image, gp.Metric.SUM)
        trees = [graph.propagate([int(s)]) for s in seq[:N_TREES]]
        tree_dist = np.stack([t.dist for t in trees])
        tree_parent = np.stack([t.parent for t in trees])
        visits = np.zeros(0, dtype=np.int64)
        source = "reference geopairs (run_strategy, force=True)"
    else:
        sys.path.insert(0, ROOT)
        from oracle import oracle as O

        r = O.run(img, spec.strategy, conn=spec.conn, nthreads=nthreads)
        D, seq, new, raw, adjusted, centroid = r["D"], r["seq"], r["new"], r["raw"], r["adjusted"], r["centroid"]
        visits = r["visits"]
        trees = [O.propagate(img, [int(s)], conn=spec.conn) for s in seq[:N_TREES]]
        tree_dist = np.stack([t[0] for t in trees])
        tree_parent = np.stack([t[1] for t in trees])
        source = "fp32 restatement (oracle/oracle.c)"
    elapsed = time.time() - t0
    si, sj, sv = _samples(D, 1000 + index)
    out = dict(
        seq=seq.astype(np.int32), new=new.astype(np.int64), raw=np.array(raw),
        adjusted=np.array(adjusted), centroid=np.array(centroid), visits=visits,
        d_sha256=np.array(d_digest(D, isf)), row_sum=D.astype(np.float64).sum(axis=1),
        samp_i=si, samp_j=sj, samp_v=sv, tree_src=seq[:N_TREES].astype(np.int32),
        tree_dist=tree_dist, tree_parent=tree_parent.astype(np.int32),
        source=np.array(source), cpu_seconds=np.array(elapsed),
        cpu_threads=np.array(1 if not isf else nthreads),
    )
    np.savez_compressed(os.path.join(HERE, f"cfg{index}.npz"), **out)
    print(f"cfg{index}: raw={raw} adjusted={adjusted} elapsed={elapsed:.1f}s src={source}")


def make_extrema(index: int):
    """The reference's EXTREMA strategy (strategies.py:195-210) on an integer
    config image: sequence, per-commit new pairs, counts and a digest of D."""
    gp = _ref()
    spec = CONFIGS[index]
    image = gp.Image(make_image(index).astype(np.int64))
    t0 = time.time()
    run = gp.run_strategy(image, gp.Metric.SUM, gp.StrategyKind.EXTREMA, force=True)
    elapsed = time.time() - t0
    A = spec.total_pairs
    filled = np.array([int(tau * A) for _, _, tau in run.trace.samples], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, f"extrema{index}.npz"),
                        seq=np.array([s for _, s, _ in run.trace.samples], dtype=np.int32),
                        new=np.diff(np.concatenate([[0], filled])), raw=np.array(run.trace.raw_count),
                        adjusted=np.array(run.trace.adjusted_count),
                        d_sha256=np.array(d_digest(run.distances.dist, False)),
                        source=np.array("reference geopairs run_strategy(EXTREMA)"),
                        cpu_seconds=np.array(elapsed))
    print(f"extrema{index}: raw={run.trace.raw_count} elapsed={elapsed:.1f}s")


def make_apgd():
    """APGD dumps written by the reference (DistanceArray.to_bytes,
    distances.py:149-154): a partially filled store (three trees: sentinels)
    and a complete filling-rate run, per image; the fill sources are recorded."""
    gp = _ref()
    rng = np.random.default_rng(2550)
    out = {}
    for i, (h, w) in enumerate([(5, 6), (9, 7), (12, 11)]):
        img = rng.integers(1, 256, (h, w))
        image = gp.Image(img)
        graph = gp.GridGraph(image, gp.Metric.SUM)
        store = gp.DistanceArray(h * w)
        roots = rng.choice(h * w, 3, replace=False)
        for r in roots:
            store.fill_from_tree(gp.build_tree(graph.propagate([int(r)]), int(r)))
        out[f"c{i}_img"] = img.astype(np.int64)
        out[f"c{i}_roots"] = roots.astype(np.int64)
        out[f"c{i}_partial"] = np.frombuffer(store.to_bytes(), dtype=np.uint8)
        run = gp.run_strategy(image, gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
        out[f"c{i}_full"] = np.frombuffer(run.distances.to_bytes(), dtype=np.uint8)
        back = gp.DistanceArray.from_bytes(store.to_bytes())
        out[f"c{i}_partial_counts"] = np.array(back.point_filled_counts)
        out[f"c{i}_partial_filled"] = np.array(back.pairs_filled)
    out["n_cases"] = np.array(3)
    np.savez_compressed(os.path.join(HERE, "ref_apgd.npz"), **out)
    print("apgd cases: 3")


def tree_digest(a: np.ndarray) -> np.ndarray:
    """16-byte sha256 prefix of an int64 per-pixel array (dist or parent)."""
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).digest()[:16],
                         dtype=np.uint8)


def make_trees(index: int):
    """Predecessor identity at config scale: propagations of
    the UNMODIFIED reference (GridGraph.propagate -> dijkstra_csr) on the config
    image, stored as per-source digests of dist and parent (int64 LE):
    cfg2 every source (4096), cfg4 256 seeded random sources plus the first 64
    committed sources of the reference run (cfg4.npz seq)."""
    gp = _ref()
    spec = CONFIGS[index]
    img = make_image(index)
    graph = gp.GridGraph(gp.Image(img.astype(np.int64)), gp.Metric.SUM)
    if index == 2:
        srcs = np.arange(spec.n, dtype=np.int64)
    else:
        seq = np.load(os.path.join(HERE, f"cfg{index}.npz"))["seq"].astype(np.int64)
        rnd = np.random.default_rng(9000 + index).choice(spec.n, 256, replace=False)
        srcs = np.concatenate([seq[:64], rnd]).astype(np.int64)
    t0 = time.time()
    dd = np.zeros((len(srcs), 16), np.uint8)
    pd = np.zeros((len(srcs), 16), np.uint8)
    for i, s in enumerate(srcs):
        r = graph.propagate([int(s)])
        dd[i] = tree_digest(r.dist)
        pd[i] = tree_digest(r.parent)
    elapsed = time.time() - t0
    np.savez_compressed(os.path.join(HERE, f"trees{index}.npz"), src=srcs.astype(np.int32),
                        dist_digest=dd, parent_digest=pd,
                        source=np.array("reference geopairs GridGraph.propagate"),
                        cpu_seconds=np.array(elapsed))
    print(f"trees{index}: {len(srcs)} sources in {elapsed:.1f}s")


if __name__ == "__main__":
    if sys.argv[1] == "small":
        make_small()
    elif sys.argv[1] == "strategies":
        make_strategies()
    elif sys.argv[1] == "harness":
        make_harness()
    elif sys.argv[1] == "extrema":
        make_extrema(int(sys.argv[2]))
    elif sys.argv[1] == "apgd":
        make_apgd()
    elif sys.argv[1] == "trees":
        make_trees(int(sys.argv[2]))
    else:
        make_cfg(int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 8)
