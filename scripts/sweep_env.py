"""Engine switches on one generated instance: for each setting, a fresh solver
(the switches are read at create) runs a fixed number of iterations.

    python scripts/sweep_env.py G 200 "NUMPMP_COL_BLOCKS=4" "NUMPMP_COL_BLOCKS=8,NUMPMP_L2_PERSIST_MB=0" ...
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2509_10722_b200 as pmp  # noqa: E402

name, iters = sys.argv[1], int(sys.argv[2])
p = bench.make_problem(name)
cfg = bench.solver_config(name, max_iters=iters)
cfg.eps_abs = 1e-300  # run exactly `iters` iterations
for setting in sys.argv[3:]:
    kv = dict(x.split("=") for x in setting.split(",") if x)
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update(kv)
    with pmp.PmpSolver(p, cfg) as s:
        s.solve()  # warm-up (graphs, L2)
        t = time.perf_counter()
        sol = s.solve()
        dt = time.perf_counter() - t
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    print(f"{name} {setting:50s} iters {sol.iterations} ms/it {1e3 * dt / sol.iterations:.4f}", flush=True)
