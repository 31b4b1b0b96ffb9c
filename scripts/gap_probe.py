"""Distribution of the device time outside commit/propagation/setup over repeated runs (dev helper)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_16076_b200 import _lib
from paper_2007_16076_b200.configs import CONFIGS, make_image

L = _lib.load_library()
spec = CONFIGS[5]
px = np.ascontiguousarray(make_image(5).astype(np.float32))
h, st = ctypes.c_void_p(), ctypes.c_void_p()
_lib.check(L.gp_ctx_create(256, 256, _lib.DTYPE_F32, _lib.ptr(px), 1, 8, ctypes.byref(h)))
_lib.check(L.gp_store_create(spec.n, ctypes.byref(st)))
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    s = _lib.RunStats()
    _lib.check(L.gp_run(h, st, _lib.STRATEGY_FILLING_RATE, 0, 0, None, None, ctypes.byref(s)))
    gap = s.ms_total - s.ms_commit - s.ms_propagate - s.ms_setup
    print(f"total {s.ms_total:8.2f} commit {s.ms_commit:7.2f} prop {s.ms_propagate:7.2f} setup {s.ms_setup:5.2f} gap {gap:6.2f}", flush=True)
