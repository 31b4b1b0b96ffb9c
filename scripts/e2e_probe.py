"""Break the e2e path (gp_ctx_load + gp_run_to_host) into its parts (dev helper)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2007_16076_b200 import _lib
from paper_2007_16076_b200.configs import CONFIGS, make_image

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
spec = CONFIGS[idx]
img = make_image(idx)
L = _lib.load_library()
N = spec.n
px = np.ascontiguousarray(img.astype(np.float32) if spec.dtype == "f32" else img)
dtype = _lib.DTYPE_F32 if spec.dtype == "f32" else _lib.DTYPE_U8
strat = _lib.STRATEGY_FILLING_RATE
h = ctypes.c_void_p()
_lib.check(L.gp_ctx_create(spec.shape[0], spec.shape[1], dtype, _lib.ptr(px), 1, spec.conn, ctypes.byref(h)))
st = ctypes.c_void_p()
_lib.check(L.gp_store_create(N, ctypes.byref(st)))
seq = np.zeros(N, dtype=np.int32)
new = np.zeros(N, dtype=np.int64)
Dh = torch.empty((N, N), dtype=torch.float32, pin_memory=True)
pxp = torch.from_numpy(px.copy()).pin_memory()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(L.gp_ctx_load(h, dtype, ctypes.c_void_p(pxp.data_ptr())))
    t1 = time.perf_counter()
    s = _lib.RunStats()
    _lib.check(L.gp_run_to_host(h, st, strat, 0, 0, _lib.ptr(seq), _lib.ptr(new), ctypes.byref(s),
                                ctypes.c_void_p(Dh.data_ptr())))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep{rep} commit {s.ms_commit:.1f} prop {s.ms_propagate:.1f} load {1e3*(t1-t0):.2f} ms  run_to_host wall {1e3*(t2-t1):.1f} ms  device {s.ms_total:.1f} ms"
          f"  -> host/copy overhead {1e3*(t2-t1)-s.ms_total:.1f} ms", flush=True)
