"""Small runs of the round-2 paths for compute-sanitizer (dev helper):
    compute-sanitizer --tool memcheck python scripts/sanitize_small.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
os.environ.setdefault("GP_LIST_BATCH", "1")
os.environ.setdefault("GP_E2E_CUT", "3000")
import paper_2007_16076_b200 as gp
from paper_2007_16076_b200 import _lib

img = np.random.default_rng(5).integers(1, 256, (40, 36))
run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
D = run.distances.dist
assert np.array_equal(D, D.T)
L = _lib.lib()
n = img.size
ctx, st = ctypes.c_void_p(), ctypes.c_void_p()
px = np.ascontiguousarray(img.astype(np.int64))
_lib.check(L.gp_ctx_create(40, 36, 0, _lib.ptr(px), 1, 8, ctypes.byref(ctx)))
_lib.check(L.gp_store_create(n, ctypes.byref(st)))
host = np.full((n, n), -7.0, dtype=np.float32)
seq = np.zeros(n, np.int32)
stats = _lib.RunStats()
_lib.check(L.gp_run_to_host(ctx, st, 1, 0, 0, _lib.ptr(seq), None, ctypes.byref(stats), _lib.ptr(host)))
assert np.array_equal(host.astype(np.int64), D), "host array differs"
L.gp_store_destroy(st)
L.gp_ctx_destroy(ctx)
print("sanitize_small ok", stats.raw_count)
