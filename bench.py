#!/usr/bin/env python
"""bench.py -- PMP iterations/s and time-to-1e-4 on BASELINE.json's config
(configs[2]: 10M streams / 1M links, mixed log+linear utilities) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]
    torchrun --nproc-per-node N bench.py --gpus N ...

One "step" is one full cold-start solve to eps_abs = 1e-4 (the time-to-
tolerance half of the metric); ``value`` = total PMP iterations / total
device time (CUDA events on the engine's stream, max over ranks), with the
problem already resident in HBM.  ``e2e`` is the same metric through the
C-ABI from pinned HOST buffers: problem upload + device CSR build + solve +
solution download per step.  The reference arm times the reference's own
CPU PmpSolver (oracle/_ref, compiled from /root/reference) on the host.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PMP iterations/sec and time-to-1e-4 residual, 10M streams, 1/2/4/8 B200"
UNIT = "iterations/s"

# BASELINE.json configs / SURVEY.md Appendix B (reference generators, fixed seeds)
CONFIGS = {
    "A": dict(ref_iters=50000, m=1000, n=10000, avg=5.0, kind=0, uniform=False, seed=7, rho0=1000.0,
              desc="A: 10k streams / 1k links, log, w=1"),
    "B": dict(ref_iters=100, m=100000, n=1000000, avg=10.0, kind=0, uniform=False, seed=7, rho0=1000.0,
              desc="B: 1M streams / 100k links, log, w=1"),
    "C": dict(ref_iters=12, m=1000000, n=10000000, avg=10.0, kind=2, uniform=True, seed=7, rho0=1000.0,
              desc="C: 10M streams / 1M links, mixed log+linear (Bernoulli 0.5), w~U(0.5,1.5)"),
    "D": dict(ref_iters=12, m=1000000, n=10000000, avg=10.0, kind=2, uniform=True, seed=7, rho0=1000.0, degrade=(0.5, 0.5, 99),
              desc="D: C with 50% of capacities x0.5 (degrade seed 99)"),
    "E": dict(ref_iters=20, transit=(100, 192, 5.0, 952, 9900, 9, 192, 50.0, 4), rho0=1000.0,
              desc="E: time-expanded transit, S=100 T=192 |E|=952, 9900 OD x 9 routes x 192 departures, seats 50"),
    # SURVEY.md 8(d) optional paper-shape cross-check (1847 s on an A100, tolerance and
    # iteration count unstated): more links than streams
    # gen_congested (hot links on 10% of the streams each): the heavy-tailed
    # streams-per-link distribution; hot rows are split over several warp units in the link pass
    "F": dict(ref_iters=50, m=100000, n=1000000, avg=10.0, kind=2, uniform=True, seed=7, rho0=1000.0, congested=(0.001, 0.10),
              desc="F: B-size congested, 100 hot links on ~10% of 1M streams each (mixed, w~U(0.5,1.5))"),
    "G": dict(ref_iters=2, m=1000000, n=10000000, avg=10.0, kind=2, uniform=True, seed=7, rho0=1000.0, congested=(0.001, 0.10),
              desc="G: C congested, 1000 hot links on ~10% of 10M streams each (1.1e9 nonzeros)"),
    "P": dict(ref_iters=12, m=10000000, n=5000000, avg=10.0, kind=0, uniform=False, seed=7, rho0=1000.0,
              desc="P: paper shape, 5M streams / 10M links, log, w=1"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_problem(name):
    import paper_2509_10722_b200 as pmp

    c = CONFIGS[name]
    if "transit" in c:
        p, _ = pmp.gen_transit(pmp.TransitSpec(*c["transit"]))
        return p
    w = pmp.WeightDist.uniform(0.5, 1.5) if c["uniform"] else pmp.WeightDist.constant(1.0)
    spec = pmp.GenSpec(m=c["m"], n=c["n"], avg_links_per_stream=c["avg"], kind=pmp.GenKind(c["kind"]), weights=w,
                       seed=c["seed"])
    p = pmp.gen_congested(spec, *c["congested"]) if "congested" in c else pmp.gen_uncongested(spec)
    if "degrade" in c:
        p = pmp.degrade(p, *c["degrade"])
    return p


DATA = "synthetic (the reference generator recipe of the config, fixed seed)"


def repo_libs_loaded():
    """Shared objects under this repo mapped into this process (/proc/self/maps)."""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                path = ln.split()[-1] if len(ln.split()) >= 6 else ""
                if path.endswith(".so") and os.path.realpath(path).startswith(os.path.realpath(ROOT) + os.sep):
                    out.add(os.path.relpath(os.path.realpath(path), os.path.realpath(ROOT)))
    except OSError:
        pass
    return sorted(out)


def bench_config(name, m, n, nnz):
    """The `config` object both arms print (identical by construction)."""
    return {"workload": CONFIGS[name]["desc"], "m": m, "n": n, "nnz": nnz, "eps_abs": 1e-4,
            "rho0": CONFIGS[name]["rho0"], "alpha": 1.6, "mu": 2.0, "gamma": 1.1, "rho_update_interval": 50,
            "l2": "inputs larger than L2 (>1 GB touched per iteration at C/D/E vs 126 MB L2)"}


def solver_config(name, max_iters=50000):
    import paper_2509_10722_b200 as pmp

    return pmp.SolverConfig(eps_abs=1e-4, rho0=CONFIGS[name]["rho0"], alpha=1.6, mu=2.0, gamma=1.1,
                            rho_update_interval=50, max_iters=max_iters, trace_every=10)


def alg_bytes(m, n, nnz):
    """SURVEY.md 8(d) yardstick (fp64 values, int32 indices), per kernel."""
    k1 = 4 * nnz + 4 * (n + 1) + n * (8 + 1 + 16 + 8) + 8 * m  # row_idx, col_ptr, w, kind, A r/w, x w, v gather
    k2 = 4 * nnz + 4 * (m + 1) + 8 * n + m * (8 + 16 + 16 + 16 + 8)  # col_idx, row_ptr, x gather, c, price/B/zs r/w, v w
    return k1, k2


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# Test hooks for the multi-rank bench path on a one-GPU box (never set by
# the driver): NUMPMP_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 and
# NUMPMP_BENCH_BACKEND=gloo carries the plumbing collectives on CPU (NCCL
# refuses two ranks on one GPU).  The ranks then time-share the GPU, so the
# numbers measure nothing; the code path is what is exercised.
BACKEND = os.environ.get("NUMPMP_BENCH_BACKEND", "nccl")


def dist_setup(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("NUMPMP_BENCH_SAME_DEVICE") == "1":
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group(BACKEND, init_method="env://")
    return rank, world, local


def _coll_device():
    return "cpu" if BACKEND == "gloo" else "cuda"


def barrier_sync(world):
    import torch

    if torch.cuda.is_available():
        torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        torch.cuda.synchronize()


def max_over_ranks(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------- reference arm
def make_ref_problem(name):
    """The config's Problem built by the REFERENCE's own generators (oracle/_ref:
    gen.hpp / transit.hpp compiled from /root/reference), so the reference arm
    maps no library of this repo."""
    from oracle import oracle as o

    ref = o.Reference()
    c = CONFIGS[name]
    if "transit" in c:
        return ref.gen_transit(*c["transit"])
    w = ("uniform", 0.5, 1.5) if c["uniform"] else ("constant", 1.0, 1.0)
    if "congested" in c:
        rp = ref.gen(c["m"], c["n"], c["avg"], c["kind"], w, c["seed"], congested=True,
                     hot_link_fraction=c["congested"][0], hot_stream_fraction=c["congested"][1])
    else:
        rp = ref.gen(c["m"], c["n"], c["avg"], c["kind"], w, c["seed"])
    if "degrade" in c:
        rp = rp.degrade(*c["degrade"])
    return rp


def reference_solves(rp, name, steps, warmup, iters):
    """The reference's stock PmpSolver::solve() (solver.hpp:411, run 441-508 +
    post-processing) on the held solver, cfg.max_iters = `iters` (a bounded
    sample; small configs converge first), all host threads.  Returns
    (seconds per step, iterations per step, cores)."""
    from oracle import oracle as o

    cores = os.cpu_count() or 1
    cfg = o.Config(eps_abs=1e-4, rho0=CONFIGS[name]["rho0"], alpha=1.6, mu=2.0, gamma=1.1,
                   rho_update_interval=50, max_iters=iters, trace_every=10, threads=cores)
    sess = rp.bench_session(cfg)
    for _ in range(warmup):
        sess.solve()
    secs, its = [], []
    for _ in range(steps):
        t, _, k = sess.solve()
        secs.append(t)
        its.append(k)
    sess.close()
    return secs, its, cores


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    name = args.config
    from oracle import oracle as o

    if not os.path.exists(o.REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libnumpmp_ref.so not built"}), flush=True)
        return 0
    rp = make_ref_problem(name)
    k = args.ref_iters or CONFIGS[name]["ref_iters"]
    secs, its, cores = reference_solves(rp, name, args.steps, args.warmup, k)
    total = float(sum(secs))
    value = sum(its) / total if total > 0 else None
    sample = (f"each step = the reference's stock PmpSolver::solve() (solver.hpp:411,441-508) from the cold state "
              f"with max_iters={k} on config {name} (eps_abs 1e-4; iterations per step {its}), problem from the "
              f"reference's own generator, {cores} host threads; steady_clock around solve() only")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": bench_config(name, rp.m, rp.n, rp.nnz),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "iterations_per_step": its,
        "repo_libs_loaded": repo_libs_loaded(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def rank_topology(solver, rank, world, local, exchange):
    """Proof that all N ranks connected: per rank its device, PCI bus id,
    peer access to every other rank's device, its stream range and (p2p) the
    links it owns.  Gathered on every rank (collective)."""
    import torch
    import torch.distributed as dist
    from paper_2509_10722_b200.shard import link_owners

    devs = [None] * world
    dist.all_gather_object(devs, local)
    mine = {"rank": rank, "device": local, "pci_bus_id": getattr(torch.cuda.get_device_properties(local), "pci_bus_id", None),
            "streams": [solver.stream_begin, solver.stream_begin + solver.local.n],
            "peer_access": [True if d == local else bool(torch.cuda.can_device_access_peer(local, d)) for d in devs]}
    if exchange == "p2p":
        b = link_owners(solver.full.m, world)
        mine["links_owned"] = [int(b[rank]), int(b[rank + 1])]
    out = [None] * world
    dist.all_gather_object(out, mine)
    return {"world": world, "exchange": exchange, "distinct_devices": len(set(devs)), "ranks": out}


def run_ours(args):
    import paper_2509_10722_b200 as pmp
    from paper_2509_10722_b200 import _lib
    from paper_2509_10722_b200.shard import ShardedPmpSolver, nccl_unique_id

    rank, world, local = dist_setup(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks")
    same_device = os.environ.get("NUMPMP_BENCH_SAME_DEVICE") == "1"
    if world > 1 and not same_device:
        import torch

        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench.py --gpus {world}: only {torch.cuda.device_count()} GPUs visible")
    name = args.config
    t_gen = time.perf_counter()
    problem = make_problem(name)
    t_gen = time.perf_counter() - t_gen
    cfg = solver_config(name)
    L = _lib.lib()

    exchange = os.environ.get("NUMPMP_EXCHANGE", "p2p")

    def make_sharded():
        import torch.distributed as dist

        if exchange == "p2p":  # fused peer-memory exchange (csrc/pmp_p2p.cuh)
            def ipc_allgather(mine):
                out = [None] * world
                dist.all_gather_object(out, mine)
                return out

            return ShardedPmpSolver(problem, cfg, rank, world, device=local, exchange="p2p",
                                    ipc_allgather=ipc_allgather)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return ShardedPmpSolver(problem, cfg, rank, world, obj[0], device=local, exchange="nccl")

    topology = None
    if world > 1:
        solver = make_sharded()
        h = solver.handle()
        topology = rank_topology(solver, rank, world, local, exchange)
    else:
        solver = pmp.PmpSolver(problem, cfg, device=local)
        h = solver.handle()

    def check(rc):
        if rc:
            raise RuntimeError(L.numpmp_gpu_last_error(h).decode())

    info = _lib.SolutionInfo()
    ms = C.c_double()
    # warm-up: full solves (graph instantiation, clocks)
    for _ in range(args.warmup):
        check(L.numpmp_gpu_set_cold(h))
        check(L.numpmp_gpu_run_device(h, C.byref(info)))
    check(L.numpmp_gpu_set_profiling(h, 0))  # resets the launch counter; production graphs
    iters, dev_ms, statuses = [], [], []
    with ClockSampler(local) as clocks:
        barrier_sync(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            check(L.numpmp_gpu_set_cold(h))
            check(L.numpmp_gpu_run_device(h, C.byref(info)))
            check(L.numpmp_gpu_last_run_ms(h, C.byref(ms)))
            iters.append(int(info.iterations))
            statuses.append(int(info.status))
            dev_ms.append(ms.value)
        barrier_sync(world)
        wall = time.perf_counter() - t0
    launches, ms1, ms2, it_t = C.c_int64(), C.c_double(), C.c_double(), C.c_int64()
    check(L.numpmp_gpu_profile(h, C.byref(launches), C.byref(ms1), C.byref(ms2), C.byref(it_t)))
    timed_launches = int(launches.value)
    # Kernel split for the roofline: one more (untimed) solve with CUDA events
    # around every launch of the serial graph.
    check(L.numpmp_gpu_set_profiling(h, 1))
    check(L.numpmp_gpu_set_cold(h))
    check(L.numpmp_gpu_run_device(h, C.byref(info)))
    check(L.numpmp_gpu_profile(h, C.byref(launches), C.byref(ms1), C.byref(ms2), C.byref(it_t)))
    check(L.numpmp_gpu_set_profiling(h, 0))
    total_ms = max_over_ranks(world, float(sum(dev_ms)))
    total_iters = int(sum(iters))
    value = total_iters / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # roofline of the dominant kernel (per launch, this rank's shard)
    lp = solver.local if world > 1 else problem
    k1b, k2b = alg_bytes(lp.m, lp.n, lp.nnz)
    n_it = max(int(it_t.value), 1)
    avg1, avg2 = ms1.value / n_it, ms2.value / n_it
    hbm, peak_kind = peaks()
    if avg2 >= avg1:
        dom, dom_bytes, dom_ms = "k_link_pass (R.x gather + link epilogue + finalize)", k2b, avg2
    else:
        dom, dom_bytes, dom_ms = "k_stream_pass (R^T.v gather + prox)", k1b, avg1
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    iter_ms = (ms1.value + ms2.value) / n_it
    iter_gbs = (k1b + k2b) / (iter_ms * 1e-3) / 1e9
    # DRAM traffic of the dominant kernel per iteration, from the committed
    # ncu --set full capture (profiles/traffic_r2.json; config C, one GPU)
    traffic, xbar_pct, iter_dram = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_r2.json")) as f:
            tr = json.load(f)
        if tr.get("config") == name and world == 1:
            key = "k_link_pass" if avg2 >= avg1 else "k_stream_pass"
            traffic = tr["per_iteration"][key]["dram_bytes"]
            xbar_pct = tr["per_iteration"][key].get("xbar_req_pct")
            iter_dram = sum(v["dram_bytes"] for v in tr["per_iteration"].values())
    except Exception:
        traffic = None
    # The structural bound: one random 8-byte gather per nonzero and pass,
    # each one L1->L2 request; an SM issues at most one such request per
    # cycle (ncu l1tex__m_l1tex2xbar_req_cycles_active).  Measured ceiling:
    # scripts/gather_lanes_bench.cu, 269 G gathers/s from an L2-resident
    # vector at 92.5% of that request rate (profiles/r1_gather_lanes.txt).
    gather_peak = 269.0e9
    gather_rate = lp.nnz / (dom_ms * 1e-3)

    # e2e: the public C-ABI from pinned host buffers, per step:
    # create (H2D problem + device CSR build) -> solve -> D2H solution -> destroy
    e2e = None
    if world > 1:
        # e2e at N GPUs through the public sharded API, per step: create the
        # rank's handle from host buffers (H2D + device CSR build + exchange
        # setup) -> solve -> download x shard and link vectors -> destroy;
        # max over ranks.
        import torch

        e_iters, e_secs = [], []
        for step in range(args.steps + 1):  # first is warm-up
            barrier_sync(world)
            t = time.perf_counter()
            ss = make_sharded()
            sol = ss.solve()
            ss.close()
            torch.cuda.synchronize()
            el = max_over_ranks(world, time.perf_counter() - t)
            if step > 0:
                e_iters.append(int(sol.iterations))
                e_secs.append(el)
        lp_ = solver.local
        h2d = sum_over_ranks(world, float(lp_.capacities.nbytes + lp_.weights.nbytes + lp_.kinds.nbytes
                                          + lp_.stream_offsets.nbytes + lp_.route_links.nbytes))
        d2h = sum_over_ranks(world, float(8 * lp_.n + 3 * 8 * lp_.m))
        e2e = {"value": sum(e_iters) / sum(e_secs), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * sum(e_secs) / len(e_secs),
               "timing": "host wall clock around create+solve+download+destroy on every rank, max over ranks"}
    if world == 1:
        arrays = [problem.capacities, problem.weights, problem.kinds, problem.stream_offsets, problem.route_links]
        for a in arrays:
            check(L.numpmp_gpu_pin_host(_lib.ptr(a), a.nbytes))
        x = np.empty(problem.n)
        s = np.empty(problem.m)
        lam = np.empty(problem.m)
        lraw = np.empty(problem.m)
        outs = [x, s, lam, lraw]
        for a in outs:
            check(L.numpmp_gpu_pin_host(_lib.ptr(a), a.nbytes))
        h2d = sum(a.nbytes for a in arrays)
        d2h = sum(a.nbytes for a in outs)
        cap = cfg.max_iters // cfg.trace_every + 2
        trace = (_lib.TraceRow * cap)()
        e_iters, e_secs = [], []
        solver_e2e = None
        for step in range(args.steps + 1):  # first is warm-up
            import torch

            torch.cuda.synchronize()
            t = time.perf_counter()
            hh = C.c_void_p()
            view = problem.view()
            check(L.numpmp_gpu_create(C.byref(view), C.byref(cfg._c()), local, C.byref(hh)))
            rc = L.numpmp_gpu_run(hh, _lib.ptr(x), _lib.ptr(s), _lib.ptr(lam), _lib.ptr(lraw), C.byref(info), trace, cap)
            L.numpmp_gpu_destroy(hh)
            torch.cuda.synchronize()
            el = time.perf_counter() - t
            if rc:
                raise RuntimeError("e2e run failed")
            if step > 0:
                e_iters.append(int(info.iterations))
                e_secs.append(el)
        for a in arrays + outs:
            L.numpmp_gpu_unpin_host(_lib.ptr(a))
        e2e = {"value": sum(e_iters) / sum(e_secs), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * sum(e_secs) / len(e_secs),
               "timing": "host wall clock around create+solve+download+destroy, synchronized"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as o

        if os.path.exists(o.REF_SO):
            rp = o.Reference().build_problem(problem.m, problem.n, problem.stream_offsets, problem.route_links,
                                             problem.kinds, problem.weights, problem.capacities)
            k = args.ref_iters or CONFIGS[name]["ref_iters"]
            secs, its, cores = reference_solves(rp, name, 1, 0, k)
            del rp
            cpu = {"value": sum(its) / sum(secs), "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"one stock PmpSolver::solve() of the reference (oracle/_ref = reference headers "
                             f"compiled -O3) with max_iters={k} ({its[0]} iterations) on config {name}, "
                             f"{cores} host threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": (topology["distinct_devices"] if topology else 1), "ranks": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": bench_config(name, problem.m, problem.n, problem.nnz),
            "parallelism": f"stream shards x{world}" + (
                (" + fused peer-memory exchange (NVLink stores into link owners, owner epilogue)"
                 if exchange == "p2p" else " + NCCL all-reduce of link loads") if world > 1 else ""),
            "step": "one cold-start solve to eps_abs=1e-4 (time-to-tolerance)",
            "iterations_per_solve": iters, "status": statuses,
            "time_to_tol_s": ms_per_step / 1e3,
            "ms_per_iteration": total_ms / max(total_iters, 1),
            "wall_s_timed": wall,
            "gen_s": t_gen,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "peak_kind": peak_kind, "traffic": traffic,
                         "frac_vs_8tbs_spec": achieved / 8000.0,
                         "alg_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                         "launch": "one pass over all column blocks per iteration",
                         "gather_bound": {"achieved_gathers_per_s": gather_rate, "peak_gathers_per_s": gather_peak,
                                          "frac": gather_rate / gather_peak,
                                          "l1_to_l2_request_pct_ncu": xbar_pct,
                                          "source": "scripts/gather_lanes_bench.cu (profiles/r1_gather_lanes.txt); "
                                                    "request utilisation: profiles/traffic_r2.json"}},
            "iteration_roofline": {"alg_bytes": k1b + k2b, "alg_bytes_per_nnz": (k1b + k2b) / max(lp.nnz, 1),
                                   "dram_bytes_ncu": iter_dram,
                                   "dram_bytes_per_nnz_ncu": (iter_dram / max(lp.nnz, 1)) if iter_dram else None,
                                   "ms": iter_ms, "achieved_gbs": iter_gbs,
                                   "frac": iter_gbs / hbm, "stream_pass_ms": avg1, "link_pass_ms": avg2},
            "gpu_launches": timed_launches + args.steps,
            "kernel_split": "per-launch CUDA events from one extra untimed solve of the serial graph",
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "topology": topology,
            "repo_libs_loaded": repo_libs_loaded(),
        }
        if same_device and world > 1:
            line["functional_only"] = True  # ranks time-share one GPU: not a scaling result
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


def spawn_ranks(args):
    """`--gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1; rank 0's JSON line is passed through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C", choices=sorted(CONFIGS))
    ap.add_argument("--ref-iters", type=int, default=0,
                    help="max_iters of each reference solve (0: the config's default sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
