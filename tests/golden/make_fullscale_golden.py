"""Full-scale goldens for BASELINE.json configs C, D and E, generated from the
reference itself (oracle/_ref: the unmodified numpmp headers compiled by
oracle/Makefile).  TEST INFRASTRUCTURE ONLY: run here, where /root/reference
exists; the compact fixtures are committed so the GPU box (which has neither
/root/reference nor hours of CPU) can check the device solver against the
reference's own run to 1e-4.

    python tests/golden/make_fullscale_golden.py [C] [D] [E] [--threads 8]

Per config it stores (fullscale_<cfg>.npz):

* sha256 digests of the reference generator's Problem arrays and of its
  TerminalLayout CSR (model.hpp:159-201), so the repo's generator and the
  device layout builder are checked bit-exactly at full size;
* the stock ``PmpSolver::solve()`` (solver.hpp:411,441-508) to eps_abs 1e-4
  with trace_every = 1: status, iterations, every iteration's (r, s, rho,
  objective), the final scalars, checksums and 10^4 seeded samples of x and
  lambda_raw (plus the full lambda_raw when m is small);
* the same at max_iters K in {10, 100, 1000} (separate stock solves).

Every rho branch and the termination decision are decided by strict
comparisons of r, s, mu*s, mu*r and eps*sqrt(J); the test derives each
decision's margin from the stored trace.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as o  # noqa: E402

# bench.py CONFIGS C / D / E
SPECS = {
    "C": dict(gen=(1000000, 10000000, 10.0, 2, ("uniform", 0.5, 1.5), 7)),
    "D": dict(gen=(1000000, 10000000, 10.0, 2, ("uniform", 0.5, 1.5), 7), degrade=(0.5, 0.5, 99)),
    "E": dict(transit=(100, 192, 5.0, 952, 9900, 9, 192, 50.0, 4)),
}
SNAPSHOTS = (10, 100, 1000)
NSAMPLE = 10000


def digest(a) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(a)).cast("B")).hexdigest()


def problem_digests(a: o.Arrays) -> dict:
    return dict(
        d_capacities=digest(a.capacities), d_weights=digest(a.weights), d_kinds=digest(a.kinds),
        d_stream_offsets=digest(a.stream_offsets), d_route_links=digest(a.route_links),
        d_link_offsets=digest(a.link_offsets), d_link_terminals=digest(a.link_terminals),
        d_link_counts=digest(a.link_counts),
    )


def sample_idx(size: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    k = min(NSAMPLE, size)
    return np.sort(rng.choice(size, size=k, replace=False)).astype(np.int64)


def vec_summary(prefix: str, v: np.ndarray, idx: np.ndarray) -> dict:
    return {
        prefix + "_idx": idx, prefix + "_val": v[idx],
        prefix + "_sum": np.array([np.sum(v), np.sum(v * v), np.max(np.abs(v))]),
    }


def make(name: str, threads: int) -> None:
    ref = o.Reference()
    sp = SPECS[name]
    t0 = time.time()
    if "transit" in sp:
        rp = ref.gen_transit(*sp["transit"])
    else:
        rp = ref.gen(*sp["gen"])
        if "degrade" in sp:
            rp = rp.degrade(*sp["degrade"])
    a = rp.arrays()
    print(f"{name}: m={a.m} n={a.n} nnz={a.nnz} generated in {time.time() - t0:.1f}s", flush=True)
    out = dict(m=a.m, n=a.n, nnz=a.nnz, **problem_digests(a))
    xi, li = sample_idx(a.n, 1), sample_idx(a.m, 2)
    out["cfg"] = np.array([1e-4, 1000.0, 1.6, 2.0, 1.1, 0.0, 50, 50000, 1], np.float64)
    del a
    for k in SNAPSHOTS:
        cfg = o.Config(eps_abs=1e-4, rho0=1000.0, max_iters=k, trace_every=1, threads=threads)
        t0 = time.time()
        res = rp.solve(cfg)
        assert res.error is None, res.error
        print(f"{name}: K={k} status={res.status} it={res.iterations} ({time.time() - t0:.0f}s)", flush=True)
        p = f"k{k}"
        out[p + "_ints"] = np.array([res.status, res.iterations], np.int64)
        out[p + "_scalars"] = np.array([res.objective, res.r_norm, res.s_norm, res.rho_final])
        out[p + "_trace"] = res.trace
        out.update(vec_summary(p + "_x", res.x, xi))
        out.update(vec_summary(p + "_lraw", res.lambda_raw, li))
        if res.status == 0:  # converged before K: the full run below covers it
            break
    cfg = o.Config(eps_abs=1e-4, rho0=1000.0, max_iters=50000, trace_every=1, threads=threads)
    t0 = time.time()
    res = rp.solve(cfg)
    assert res.error is None, res.error
    print(f"{name}: full status={res.status} it={res.iterations} obj={res.objective!r} ({res.seconds:.0f}s)",
          flush=True)
    out["ints"] = np.array([res.status, res.iterations], np.int64)
    out["scalars"] = np.array([res.objective, res.r_norm, res.s_norm, res.rho_final])
    out["seconds"] = np.array([res.seconds, threads])
    out["trace"] = res.trace
    out.update(vec_summary("x", res.x, xi))
    out.update(vec_summary("lraw", res.lambda_raw, li))
    out.update(vec_summary("s", res.s, li))
    if rp.m <= 200000:
        out["lraw_full"] = res.lambda_raw
    np.savez_compressed(os.path.join(HERE, f"fullscale_{name}.npz"), **out)
    print(f"{name}: saved", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C", "D", "E"])
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    for c in args.configs:
        make(c, args.threads)


if __name__ == "__main__":
    main()
