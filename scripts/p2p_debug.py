"""Which in-process peer-memory setups complete p2p_start (debug aid)."""
import sys
import time

import paper_2509_10722_b200 as pmp
from paper_2509_10722_b200.shard import p2p_local_group, run_ranks

for m, n, tl, mi in [(2000, 4000, 0.0, 50000), (20000, 200000, 0.0, 50000), (2000, 4000, 0.05, 10**7),
                     (20000, 200000, 0.05, 50000), (20000, 200000, 0.0, 10**7)]:
    p = pmp.gen_uncongested(pmp.GenSpec(m=m, n=n, avg_links_per_stream=10.0, seed=3))
    cfg = pmp.SolverConfig(eps_abs=1e-14 if tl else 1e-4, max_iters=mi, time_limit=tl, trace_every=10)
    t = time.time()
    try:
        ranks = p2p_local_group(p, cfg, 2)
        sols = run_ranks([s.solve for s in ranks])
        print(m, n, tl, mi, "ok", [(int(s.status), s.iterations) for s in sols], f"{time.time() - t:.1f}s", flush=True)
        for s in ranks:
            s.close()
    except Exception as e:
        print(m, n, tl, mi, "FAIL", e, f"{time.time() - t:.1f}s", flush=True)
        sys.exit(1)
