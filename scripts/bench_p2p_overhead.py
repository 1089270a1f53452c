"""Cost of the sharded engine's machinery on one GPU: the same config solved
by the single-device engine and by the peer-memory sharded engine with
world = 1 and world = 2 ranks in this process (ranks time-share the GPU, so
world = 2 measures protocol overhead + contention, not scaling).  One JSON line.

    python scripts/bench_p2p_overhead.py [--config B] [--steps K]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2509_10722_b200 as pmp  # noqa: E402
from paper_2509_10722_b200 import _lib  # noqa: E402
from paper_2509_10722_b200.shard import p2p_local_group, run_ranks  # noqa: E402


def timed(handles, steps):
    L = _lib.lib()

    def one(h):
        info = _lib.SolutionInfo()
        ms = C.c_double()
        L.numpmp_gpu_set_cold(h)
        if L.numpmp_gpu_run_device(h, C.byref(info)):
            raise RuntimeError(L.numpmp_gpu_last_error(h).decode())
        L.numpmp_gpu_last_run_ms(h, C.byref(ms))
        return int(info.iterations), ms.value

    out = []
    for step in range(steps + 1):
        r = run_ranks([lambda h=h: one(h) for h in handles])
        if step:
            out.append((r[0][0], max(x[1] for x in r)))
    it = out[0][0]
    ms = sum(x[1] for x in out) / len(out)
    return {"iterations": it, "ms_per_iteration": ms / it, "time_to_tol_s": ms / 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="B")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    p = bench.make_problem(args.config)
    cfg = bench.solver_config(args.config)
    res = {"workload": bench.CONFIGS[args.config]["desc"]}
    with pmp.PmpSolver(p, cfg) as s:
        res["single_device"] = timed([s.handle()], args.steps)
    for world in (1, 2):
        ranks = p2p_local_group(p, cfg, world)
        try:
            res[f"p2p_world{world}_one_gpu"] = timed([r.handle() for r in ranks], args.steps)
        finally:
            for r in ranks:
                r.close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
