"""Dev diagnostic: replay the committed sequence of a config with gp_commit_source and,
at sample steps, histogram the next tree's ancestor visits (sum of subtree sizes) by
subtree size and by the ancestor row's unfilled count.  Informs fill-path choices."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2007_16076_b200 as gp
from paper_2007_16076_b200.configs import CONFIGS, make_image
from paper_2007_16076_b200.strategies import _pinned_i32

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
every = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
last = int(sys.argv[3]) if len(sys.argv) > 3 else 22000
spec = CONFIGS[idx]
img = make_image(idx)
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"cfg{idx}.npz"))
seq = g["seq"]
graph = gp.GridGraph(gp.Image(img), gp.Metric.SUM, connectivity=spec.conn)
N = graph.n
store = gp.DistanceArray(N, force=True)
store._integer = bool(np.issubdtype(img.dtype, np.integer))
counts = _pinned_i32(N)
counts[:] = 0
t0 = time.time()


def subtree_sizes(parent, dist):
    root = int(np.flatnonzero(parent < 0)[0])
    p = parent.copy()
    p[root] = root
    hop = np.ones(N, dtype=np.int64)
    hop[root] = 0
    while not (p == root).all():
        hop = hop + hop[p]
        p = p[p]
    depth = hop
    sz = np.zeros(N, dtype=np.int64)
    for d in range(int(depth.max()), 0, -1):
        v = np.flatnonzero(depth == d)
        np.add.at(sz, parent[v], sz[v] + 1)
    return sz, depth


for t in range(min(last, len(seq))):
    s = int(seq[t])
    if t % every == 0 or t in (10, 100, 300):
        res = graph.propagate([s])
        sz, depth = subtree_sizes(res.parent, res.dist)
        c = np.asarray(counts).astype(np.int64)
        zeros = (N - 1) - c
        full = zeros == 0
        V = int(sz.sum())
        line = [f"t={t} filled={store.pairs_filled/spec.total_pairs:.4f} V={V} full_rows={int(full.sum())} V_full={int(sz[full].sum())}"]
        for S in (128, 512, 2048, 8192):
            m = (sz >= S) & ~full
            line.append(f"S>={S}: n={int(m.sum())} V={int(sz[m].sum())} zeros={int(zeros[m].sum())} zmed={int(np.median(zeros[m])) if m.any() else 0}")
        # adaptive: rows where a scan (64 word loads + zeros tests) beats sz/32 chunks
        for c1 in (0.25, 1.0):
            cost_scan = 64 + zeros * c1
            cost_chunk = np.ceil(sz / 32.0)
            m = (~full) & (sz > 0) & (cost_scan < cost_chunk)
            tot_chunk = cost_chunk[(~full) & (sz > 0)].sum()
            line.append(f"adapt c1={c1}: rows={int(m.sum())} chunks {int(tot_chunk)} -> {int(tot_chunk - cost_chunk[m].sum() + cost_scan[m].sum())}")
        print(" | ".join(line), f"[{time.time()-t0:.0f}s]", flush=True)
    store._commit_source(graph, s, counts)
