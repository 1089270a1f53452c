"""Degrade workflow at config C/D scale (BASELINE configs[3]):
cold solve of C (the prior), degrade 50% of the capacities by 0.5 (config D),
then re-solve D cold and warm-started with warm.hpp's warm_start_after_degrade
computed on the device (numpmp_gpu_warm_after_degrade).  One JSON line.

    python scripts/bench_degrade_warm.py [--steps K]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2509_10722_b200 as pmp  # noqa: E402
from paper_2509_10722_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    base = bench.make_problem("C")
    deg = pmp.degrade(base, 0.5, 0.5, 99)
    cfg = bench.solver_config("C")
    with pmp.PmpSolver(base, cfg) as s:
        prior = s.solve()
    L = _lib.lib()
    info = _lib.SolutionInfo()
    ms = C.c_double()
    out = {"workload": "D: C with 50% of capacities x0.5 (seed 99), re-solved after a cold solve of C",
           "prior_iterations": prior.iterations}
    with pmp.PmpSolver(deg, cfg) as s:
        h = s.handle()
        cold, warm, recipe_ms = [], [], []
        for step in range(args.steps + 1):
            L.numpmp_gpu_set_cold(h)
            L.numpmp_gpu_run_device(h, C.byref(info))
            L.numpmp_gpu_last_run_ms(h, C.byref(ms))
            if step:
                cold.append((int(info.iterations), ms.value))
            torch.cuda.synchronize()
            t = time.perf_counter()
            s.warm_start_after_degrade(base, prior)
            torch.cuda.synchronize()
            rec = (time.perf_counter() - t) * 1e3
            L.numpmp_gpu_run_device(h, C.byref(info))
            L.numpmp_gpu_last_run_ms(h, C.byref(ms))
            if step:
                warm.append((int(info.iterations), ms.value))
                recipe_ms.append(rec)
    out["cold"] = {"iterations": cold[0][0], "time_to_tol_s": float(np.mean([c[1] for c in cold])) / 1e3}
    out["warm"] = {"iterations": warm[0][0], "time_to_tol_s": float(np.mean([w[1] for w in warm])) / 1e3,
                   "recipe_ms": float(np.mean(recipe_ms)),
                   "recipe": "warm.hpp:25-57 on the device (+ host->device copy of c_before, prior x, lambda_raw)"}
    out["speedup_warm_vs_cold"] = out["cold"]["time_to_tol_s"] / (out["warm"]["time_to_tol_s"] + out["warm"]["recipe_ms"] / 1e3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
