"""e2e phase timing of the C-ABI (NUMPMP_TIMING=1): create -> run -> destroy."""
import ctypes as C
import os
import sys
import time

os.environ["NUMPMP_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_10722_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "B"
p = bench.make_problem(name)
cfg = bench.solver_config(name)
L = _lib.lib()
arrays = [p.capacities, p.weights, p.kinds, p.stream_offsets, p.route_links]
for a in arrays:
    L.numpmp_gpu_pin_host(_lib.ptr(a), a.nbytes)
import numpy as np  # noqa: E402

x, s, lam, lraw = np.empty(p.n), np.empty(p.m), np.empty(p.m), np.empty(p.m)
for a in (x, s, lam, lraw):
    L.numpmp_gpu_pin_host(_lib.ptr(a), a.nbytes)
cap = cfg.max_iters // cfg.trace_every + 2
trace = (_lib.TraceRow * cap)()
info = _lib.SolutionInfo()
for rep in range(3):
    t = time.perf_counter()
    h = C.c_void_p()
    view = p.view()
    assert L.numpmp_gpu_create(C.byref(view), C.byref(cfg._c()), 0, C.byref(h)) == 0
    t1 = time.perf_counter()
    assert L.numpmp_gpu_run(h, _lib.ptr(x), _lib.ptr(s), _lib.ptr(lam), _lib.ptr(lraw), C.byref(info), trace, cap) == 0
    t2 = time.perf_counter()
    L.numpmp_gpu_destroy(h)
    t3 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t):.1f} ms, run {1e3*(t2-t1):.1f} ms ({info.iterations} it), destroy {1e3*(t3-t2):.1f} ms", flush=True)
