"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel form of the engine on instances the sanitizers
finish in minutes.  Each case prints one line and checks its iteration count
against the oracle restatement (the sanitizer must not change results).

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py A forms B p2p1 p2p2

Cases:
  A      config A (10k streams / 1k links, log), single device, 300 iterations
  forms  row mode, warp units, split-row pieces (gen_congested hot links),
         pair tiles (transit), 3 column blocks, fused epilogue variant
  B      config B (1M streams / 100k links), 20 iterations
  p2p1   the peer-memory engine, world 1 (fused owner epilogue)
  p2p2   world 2 in this process on one GPU (separate wait / finalize
         kernels).  The sanitizers serialize a process's kernels, so the
         ranks' barrier spin cannot complete here (it traps after 60 s);
         use ipcrank instead.
  ipcrank R PORT  rank R of 2 over CUDA IPC (one process per rank, both on
         cuda:0, gloo for the 64-byte handles): run two of these, each under
         its own compute-sanitizer, for the exchange's barriers and the
         slot / v / xs stores between processes
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_10722_b200 as pmp  # noqa: E402
from oracle import oracle as o  # noqa: E402  (test infrastructure: the checker)

R = o.Restatement()


def gen(m, n, avg, kind, uniform, seed):
    w = pmp.WeightDist.uniform(0.5, 1.5) if uniform else pmp.WeightDist.constant(1.0)
    return pmp.gen_uncongested(pmp.GenSpec(m=m, n=n, avg_links_per_stream=avg, kind=pmp.GenKind(kind),
                                           weights=w, seed=seed))


def ocfg(c):
    return o.Config(eps_abs=c.eps_abs, rho0=c.rho0, max_iters=c.max_iters)


def solve_check(name, p, cfg, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        with pmp.PmpSolver(p, cfg) as s:
            sol = s.solve()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ref = R.solve(o.arrays_from(p), ocfg(cfg))
    ok = sol.iterations == ref.iterations
    print(f"{name}: m={p.m} n={p.n} iterations {sol.iterations} (oracle {ref.iterations}) {'ok' if ok else 'MISMATCH'}",
          flush=True)
    return ok


def case_A():
    return solve_check("A (300 iterations)", gen(1000, 10000, 5.0, 0, False, 7),
                       pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0, max_iters=300))


def case_forms():
    ok = True
    p = gen(2000, 4000, 6.0, 2, True, 11)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0, max_iters=300)
    ok &= solve_check("forms/row-mode 3 blocks", p, cfg, {"NUMPMP_COL_BLOCKS": "3", "NUMPMP_ROW_MODE_MAX": "100000"})
    ok &= solve_check("forms/units 2 blocks", p, cfg, {"NUMPMP_COL_BLOCKS": "2", "NUMPMP_ROW_MODE_MAX": "0"})
    ok &= solve_check("forms/fused epilogue", p, cfg, {"NUMPMP_SPLIT_EPILOGUE": "0", "NUMPMP_ROW_MODE_MAX": "0"})
    spec = pmp.GenSpec(m=400, n=6000, avg_links_per_stream=5.0, kind=pmp.GenKind.Mixed,
                       weights=pmp.WeightDist.uniform(0.5, 1.5), seed=5)
    hot = pmp.gen_congested(spec, 0.01, 0.4)  # hot rows of ~2400 entries: split-row pieces
    ok &= solve_check("forms/pieces", hot, cfg, {"NUMPMP_ROW_MODE_MAX": "0"})
    tp, _ = pmp.gen_transit(pmp.TransitSpec(12, 24, 5.0, 40, 60, 3, 24, 50.0, 4))
    ok &= solve_check("forms/pair tiles (transit)", tp, cfg)
    return ok


def case_B():
    p = gen(100000, 1000000, 10.0, 0, False, 7)
    return solve_check("B (20 iterations)", p, pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0, max_iters=20))


def p2p_case(world):
    from paper_2509_10722_b200.shard import p2p_local_group, run_ranks

    p = gen(1200, 2400, 5.0, 2, True, 41)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0, max_iters=200)
    ranks = p2p_local_group(p, cfg, world)
    try:
        sols = run_ranks([s.solve for s in ranks])
    finally:
        for s in ranks:
            s.close()
    ref = R.solve(o.arrays_from(p), ocfg(cfg))
    ok = all(s.iterations == ref.iterations for s in sols)
    print(f"p2p world {world}: iterations {[s.iterations for s in sols]} (oracle {ref.iterations}) "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def ipc_rank(rank, port):
    import torch.distributed as dist

    from paper_2509_10722_b200.shard import ShardedPmpSolver

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    p = gen(1200, 2500, 5.0, 2, True, 3)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0, max_iters=200)

    def allgather(mine):
        out = [None, None]
        dist.all_gather_object(out, mine)
        return out

    s = ShardedPmpSolver(p, cfg, rank, 2, device=0, exchange="p2p", ipc_allgather=allgather)
    sol = s.solve()
    s.close()
    dist.destroy_process_group()
    ref = R.solve(o.arrays_from(p), ocfg(cfg))
    ok = sol.iterations == ref.iterations
    print(f"ipc rank {rank}/2: iterations {sol.iterations} (oracle {ref.iterations}) {'ok' if ok else 'MISMATCH'}",
          flush=True)
    return ok


CASES = {"A": case_A, "forms": case_forms, "B": case_B, "p2p1": lambda: p2p_case(1), "p2p2": lambda: p2p_case(2)}

if __name__ == "__main__":
    if sys.argv[1:2] == ["ipcrank"]:
        sys.exit(0 if ipc_rank(int(sys.argv[2]), int(sys.argv[3])) else 1)
    names = sys.argv[1:] or list(CASES)
    good = all([CASES[n]() for n in names])
    sys.exit(0 if good else 1)
