"""Short device run for ncu captures: config (default C), a few cold-start
iterations through the C-ABI, nothing else.

    ncu --set full -k regex:k_ -c 4 python scripts/profile_run.py C 6
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2509_10722_b200 as pmp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
p = bench.make_problem(name)
cfg = bench.solver_config(name, max_iters=iters)
with pmp.PmpSolver(p, cfg) as s:
    sol = s.solve()
print("iterations", sol.iterations, "r", sol.r_norm, "s", sol.s_norm)
