"""Time the UNMODIFIED reference (geopairs, installed in baseline/_ref) on a
BASELINE config image: the CPU leg of bench.py (cpu_baseline.reference_*).

    python baseline/ref_timing.py full 2          # run_strategy(FILLING_RATE), whole image
    python baseline/ref_timing.py replay 4 200    # the reference's own per-commit path
                                                  # (propagate -> build_tree -> fill_from_tree)
                                                  # over the first 200 sources of the
                                                  # committed sequence (tests/golden/cfg4.npz)

Install once:
    pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>
The reference is single-threaded (numba @njit without parallel), so this is
one host core.  Prints one JSON line.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(HERE, "_ref"))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    mode, index = sys.argv[1], int(sys.argv[2])
    import geopairs as ref  # the reference package, unmodified

    from paper_2007_16076_b200.configs import CONFIGS, make_image

    spec = CONFIGS[index]
    if spec.dtype == "f32":
        print(json.dumps({"unavailable": "the reference rejects fp32 images (grid.py:49-50)"}))
        return
    img = make_image(index).astype(np.int64)  # zeros already remapped to 1 (pgm.py:42-47)
    # JIT warm-up on an 8x8 image (test_acceptance.py:185), excluded from the timing
    w = ref.Image(np.random.default_rng(0).integers(1, 256, (8, 8)))
    ref.run_strategy(w, ref.Metric.SUM, ref.StrategyKind.FILLING_RATE)
    image = ref.Image(img)
    out = {"reference": ref.__file__, "config": spec.name, "cores": 1, "cores_available": os.cpu_count()}
    if mode == "full":
        t0 = time.perf_counter()
        run = ref.run_strategy(image, ref.Metric.SUM, ref.StrategyKind.FILLING_RATE, force=True)
        dt = time.perf_counter() - t0
        out.update(mode="full run_strategy", seconds=dt, ms_per_image=dt * 1e3,
                   pairs_per_s=spec.total_pairs / dt, raw=run.trace.raw_count,
                   adjusted=run.trace.adjusted_count)
    else:
        m = int(sys.argv[3])
        g = np.load(os.path.join(ROOT, "tests", "golden", f"cfg{index}.npz"))
        seq = g["seq"][:m]
        P = int(g["raw"])
        graph = ref.GridGraph(image, ref.Metric.SUM)
        store = ref.DistanceArray(spec.n, force=True)
        t0 = time.perf_counter()
        for s in seq:
            store.fill_from_tree(ref.build_tree(graph.propagate([int(s)]), int(s)))
        dt = time.perf_counter() - t0
        per = dt / len(seq)
        out.update(mode=f"replay of the first {len(seq)} committed sources (propagate -> build_tree -> "
                        "fill_from_tree; selection excluded)",
                   seconds=dt, commits=len(seq), per_commit_ms=per * 1e3, P=P,
                   ms_per_image_extrapolated=per * P * 1e3,
                   pairs_per_s_extrapolated=spec.total_pairs / (per * P),
                   filled_by_prefix=int(store.pairs_filled))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
