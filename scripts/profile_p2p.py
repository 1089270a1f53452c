"""Short run of the peer-memory sharded engine (world ranks in-process) for
ncu captures of its per-iteration kernels.
    ncu -k regex:k_ python scripts/profile_p2p.py B 1 6"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2509_10722_b200.shard import p2p_local_group, run_ranks  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "B"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 6
p = bench.make_problem(name)
cfg = bench.solver_config(name, max_iters=iters)
ranks = p2p_local_group(p, cfg, world)
sols = run_ranks([r.solve for r in ranks])
for r in ranks:
    r.close()
print("iterations", sols[0].iterations)
