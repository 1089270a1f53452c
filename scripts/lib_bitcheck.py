"""Digest of a few solves with the library NUMPMP_LIB points at, for bit-identity
checks between build variants (forms forced through env):
    NUMPMP_LIB=build/variants/lib_X.so python scripts/lib_bitcheck.py"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2509_10722_b200 as pmp  # noqa: E402


def gen(m, n, avg, seed):
    return pmp.gen_uncongested(pmp.GenSpec(m=m, n=n, avg_links_per_stream=avg, kind=pmp.GenKind.Mixed,
                                           weights=pmp.WeightDist.uniform(0.5, 1.5), seed=seed))


cases = [("mixed 3000x7001", gen(3000, 7001, 10.0, 17), {}),
         ("units", gen(2000, 40000, 8.0, 3), {"NUMPMP_ROW_MODE_MAX": "0"}),
         ("row mode 3 blocks", gen(20000, 30000, 10.0, 5), {"NUMPMP_COL_BLOCKS": "3"})]
for name, p, env in cases:
    os.environ.update(env)
    with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)) as s:
        sol = s.solve()
    for k in env:
        os.environ.pop(k)
    h = hashlib.sha256(np.ascontiguousarray(sol.x).tobytes() + np.ascontiguousarray(sol.lambda_raw).tobytes())
    print(f"{name}: {sol.iterations} iterations {h.hexdigest()[:16]}")
