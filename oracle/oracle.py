"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes front-end of the two CPU checkers:

* ``Restatement``: oracle/lib/libpmp_oracle.so, the plain-C restatement of
  the reference PMP engine (pmp_oracle.c, file:line map in its header);
* ``Reference``: oracle/_ref/libnumpmp_ref.so, the reference numpmp headers
  themselves compiled through ref_harness.cpp (built where /root/reference
  exists; the prebuilt .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline /
reference legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "libpmp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnumpmp_ref.so")

P = C.c_void_p
I64 = C.c_int64
D = C.c_double


def build() -> None:
    """make -C oracle (restatement always; the reference where present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


# ----------------------------------------------------------- problem arrays
@dataclass
class Arrays:
    """Problem + TerminalLayout as flat arrays (model.hpp:47-65)."""

    m: int
    n: int
    capacities: np.ndarray
    weights: np.ndarray
    kinds: np.ndarray
    stream_offsets: np.ndarray
    terminal_link: np.ndarray  # J
    link_offsets: np.ndarray
    link_terminals: np.ndarray
    link_counts: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.stream_offsets[-1])

    @property
    def J(self) -> int:
        return self.nnz + self.m

    @property
    def route_links(self) -> np.ndarray:
        return self.terminal_link[: self.nnz]


@dataclass
class Config:
    eps_abs: float = 1e-5
    rho0: float = 1.0
    alpha: float = 1.6
    mu: float = 2.0
    gamma: float = 1.1
    time_limit: float = 0.0
    rho_update_interval: int = 50
    max_iters: int = 50000
    trace_every: int = 10
    threads: int = 1


@dataclass
class Result:
    x: np.ndarray
    s: np.ndarray
    lambda_: np.ndarray
    lambda_raw: np.ndarray
    objective: float
    status: int
    iterations: int
    r_norm: float
    s_norm: float
    rho_final: float
    trace: np.ndarray  # rows (iter, r, s, rho, objective)
    seconds: float = 0.0
    final_p: Optional[np.ndarray] = None
    final_z: Optional[np.ndarray] = None
    final_pbar: Optional[np.ndarray] = None
    final_price: Optional[np.ndarray] = None
    final_prev_z: Optional[np.ndarray] = None
    error: Optional[str] = None


# ------------------------------------------------------------ restatement
class _OProblem(C.Structure):
    _fields_ = [("m", I64), ("n", I64), ("nnz", I64), ("capacities", P), ("weights", P), ("kinds", P),
                ("stream_offsets", P), ("terminal_link", P), ("link_offsets", P), ("link_terminals", P),
                ("link_counts", P)]


class _OConfig(C.Structure):
    _fields_ = [("eps_abs", D), ("rho0", D), ("alpha", D), ("mu", D), ("gamma", D), ("time_limit", D),
                ("rho_update_interval", I64), ("max_iters", I64), ("trace_every", I64)]


class _OState(C.Structure):
    _fields_ = [("p", P), ("z", P), ("p_bar", P), ("price", P), ("rho", D), ("iter", I64)]


class _OTrace(C.Structure):
    _fields_ = [("iter", I64), ("r_norm", D), ("s_norm", D), ("rho", D), ("objective", D)]


class _OSolution(C.Structure):
    _fields_ = [("x", P), ("s", P), ("lambda_", P), ("lambda_raw", P), ("objective", D), ("status", C.c_int32),
                ("iterations", I64), ("r_norm", D), ("s_norm", D), ("rho_final", D), ("trace_len", I64)]


class Restatement:
    """The plain-C restatement (oracle/pmp_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.oracle_prox_log.restype = D
        L.oracle_prox_log.argtypes = [D, D, D, I64]
        L.oracle_prox_linear_nonneg.restype = D
        L.oracle_prox_linear_nonneg.argtypes = [D, D, D, I64]
        L.oracle_run.restype = C.c_int
        L.oracle_warm_state.restype = C.c_int
        self.L = L

    @staticmethod
    def _prob(a: Arrays):
        keep = [np.ascontiguousarray(x) for x in (a.capacities, a.weights, a.kinds, a.stream_offsets,
                                                   a.terminal_link, a.link_offsets, a.link_terminals,
                                                   a.link_counts)]
        pr = _OProblem(a.m, a.n, a.nnz, *[k.ctypes.data for k in keep])
        return pr, keep

    @staticmethod
    def _cfg(c: Config):
        return _OConfig(c.eps_abs, c.rho0, c.alpha, c.mu, c.gamma, c.time_limit, c.rho_update_interval,
                        c.max_iters, c.trace_every)

    def build_layout(self, m, n, stream_offsets, route_links):
        nnz = int(stream_offsets[-1])
        J = nnz + m
        tl = np.empty(J, np.int32)
        lo = np.empty(m + 1, np.int64)
        lt = np.empty(J, np.int64)
        lc = np.empty(m, np.int32)
        so = np.ascontiguousarray(stream_offsets, np.int64)
        rl = np.ascontiguousarray(route_links, np.int32)
        self.L.oracle_build_layout(I64(n), I64(m), _p(so), _p(rl), _p(tl), _p(lo), _p(lt), _p(lc))
        return tl, lo, lt, lc

    def prox_log(self, z, w, rho, tau):
        return self.L.oracle_prox_log(z, w, rho, tau)

    def prox_linear_nonneg(self, z, w, rho, tau):
        return self.L.oracle_prox_linear_nonneg(z, w, rho, tau)

    def cold_state(self, a: Arrays, cfg: Config):
        return dict(p=np.zeros(a.J), z=np.zeros(a.J), p_bar=np.zeros(a.m), price=np.zeros(a.m), rho=cfg.rho0, iter=0)

    def warm_state(self, a: Arrays, cfg: Config, x0, price=None, rho=0.0):
        pr, keep = self._prob(a)
        st = dict(p=np.zeros(a.J), z=np.zeros(a.J), p_bar=np.zeros(a.m), price=np.zeros(a.m))
        os_ = _OState(st["p"].ctypes.data, st["z"].ctypes.data, st["p_bar"].ctypes.data, st["price"].ctypes.data, 0.0, 0)
        err = C.create_string_buffer(256)
        x0 = np.ascontiguousarray(x0, np.float64)
        price = None if price is None else np.ascontiguousarray(price, np.float64)
        rc = self.L.oracle_warm_state(C.byref(pr), C.byref(self._cfg(cfg)), _p(x0), _p(price), D(rho), C.byref(os_), err, 256)
        if rc:
            raise ValueError(err.value.decode())
        st["rho"] = os_.rho
        st["iter"] = os_.iter
        return st

    def step(self, a: Arrays, cfg: Config, st: dict):
        """One PmpSolver::step on the dict state (in place); returns (r, s, x)."""
        pr, keep = self._prob(a)
        os_ = _OState(st["p"].ctypes.data, st["z"].ctypes.data, st["p_bar"].ctypes.data, st["price"].ctypes.data,
                      st["rho"], st["iter"])
        u = np.empty(max(a.m, 1))
        x = np.empty(a.n)
        r, s = D(), D()
        self.L.oracle_step(C.byref(pr), C.byref(self._cfg(cfg)), C.byref(os_), _p(u), _p(x), C.byref(r), C.byref(s))
        st["iter"] = os_.iter
        return r.value, s.value, x

    def solve(self, a: Arrays, cfg: Config, warm=None) -> Result:
        """PmpSolver::solve / solve(WarmStart); warm = (x0, price|None, rho)."""
        st = self.cold_state(a, cfg) if warm is None else self.warm_state(a, cfg, *warm)
        pr, keep = self._prob(a)
        os_ = _OState(st["p"].ctypes.data, st["z"].ctypes.data, st["p_bar"].ctypes.data, st["price"].ctypes.data,
                      st["rho"], st["iter"])
        x, s, lam, lraw = np.empty(a.n), np.empty(a.m), np.empty(a.m), np.empty(a.m)
        prev_z = np.empty(a.J)
        sol = _OSolution(x.ctypes.data, s.ctypes.data, lam.ctypes.data, lraw.ctypes.data)
        cap = cfg.max_iters // cfg.trace_every + 2
        trace = (_OTrace * cap)()
        err = C.create_string_buffer(256)
        rc = self.L.oracle_run(C.byref(pr), C.byref(self._cfg(cfg)), C.byref(os_), _p(prev_z), C.byref(sol), trace,
                               I64(cap), err, 256)
        tr = np.array([[trace[i].iter, trace[i].r_norm, trace[i].s_norm, trace[i].rho, trace[i].objective]
                       for i in range(sol.trace_len)]).reshape(-1, 5)
        res = Result(x, s, lam, lraw, sol.objective, sol.status, sol.iterations, sol.r_norm, sol.s_norm,
                     sol.rho_final, tr, final_p=st["p"], final_z=st["z"], final_pbar=st["p_bar"],
                     final_price=st["price"], final_prev_z=prev_z)
        if rc:
            res.error = err.value.decode()
        return res


# --------------------------------------------------------------- reference
class Reference:
    """The reference numpmp compiled from /root/reference (oracle/_ref)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (no /root/reference here)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_gen.argtypes = [I64, I64, D, C.c_int, C.c_int, D, D, C.c_uint64, C.c_int, D, D, C.POINTER(P)]
        L.ref_gen_transit.argtypes = [C.c_int32, C.c_int32, D, I64, I64, C.c_int32, C.c_int32, D, C.c_uint64,
                                      C.POINTER(P), C.POINTER(I64)]
        L.ref_degrade.argtypes = [P, D, D, C.c_uint64, C.POINTER(P)]
        L.ref_transit_meta.argtypes = [P, C.POINTER(I64), P, P, P, P, P]
        L.ref_write_trace_csv.argtypes = [C.c_char_p, I64, P, P, P, P, P]
        L.ref_write_transit_metadata.argtypes = [P, C.c_char_p]
        L.ref_check_transit_metadata.argtypes = [C.c_char_p]
        L.ref_transit_report.argtypes = [P, P, P, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(I64), P, P, P, P,
                                         I64]
        L.ref_fail_and_prune.argtypes = [P, D, C.c_uint64, C.POINTER(P)]
        L.ref_prune_maps.argtypes = [P, P, P]
        L.ref_write_problem.argtypes = [P, C.c_char_p, C.c_int]
        L.ref_read_problem.argtypes = [C.c_char_p, C.POINTER(P)]
        L.ref_build_problem.argtypes = [I64, I64, P, P, P, P, P, C.POINTER(P)]
        L.ref_sizes.argtypes = [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]
        L.ref_free.argtypes = [P]
        L.ref_export.argtypes = [P] * 9
        L.ref_solve.argtypes = [P, P, P, P, P, D, P, P, P, P, P, P, P, I64, P, P, P, P, P]
        L.ref_steps.argtypes = [P, P, P, C.c_int, P, P, D, I64, P, P, P, P, P, P, P]
        L.ref_time_iterations.argtypes = [P, P, P, I64, P, P]
        L.ref_warm_after_degrade.argtypes = [P, P, P, P, D, P, P, P]
        L.ref_warm_after_prune.argtypes = [P, P, I64, P, I64, D, P, P, P]
        L.ref_bench_open.argtypes = [P, P, P, C.POINTER(P)]
        L.ref_bench_solve.argtypes = [P, P, P, P]
        L.ref_bench_close.argtypes = [P]
        L.ref_groups.argtypes = [P, C.POINTER(I64), C.POINTER(I64), P, P, P, P]
        L.ref_prox_log.restype = D
        L.ref_prox_log.argtypes = [D, D, D, I64]
        L.ref_prox_linear_nonneg.restype = D
        L.ref_prox_linear_nonneg.argtypes = [D, D, D, I64]
        self.L = L

    def _err(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def gen(self, m, n, avg=10.0, kind=0, weights=("constant", 1.0, 1.0), seed=0, congested=False,
            hot_link_fraction=0.001, hot_stream_fraction=0.10) -> "RefProblem":
        h = P()
        wk = 0 if weights[0] == "constant" else 1
        self._err(self.L.ref_gen(m, n, avg, kind, wk, weights[1], weights[2], seed, int(congested),
                                 hot_link_fraction, hot_stream_fraction, C.byref(h)))
        return RefProblem(self, h)

    def gen_transit(self, stations, time_bins, bin_minutes, spatial_edges, od_pairs, routes_per_od,
                    departures_per_route, seats, seed) -> "RefProblem":
        h = P()
        dropped = I64()
        self._err(self.L.ref_gen_transit(stations, time_bins, bin_minutes, spatial_edges, od_pairs, routes_per_od,
                                         departures_per_route, seats, seed, C.byref(h), C.byref(dropped)))
        rp = RefProblem(self, h)
        rp.dropped = dropped.value
        return rp

    def read_problem(self, path) -> "RefProblem":
        """io.hpp:172-279; raises RuntimeError with the reference's message."""
        h = P()
        self._err(self.L.ref_read_problem(os.fsencode(path), C.byref(h)))
        return RefProblem(self, h)

    def build_problem(self, m, n, stream_offsets, routes, kinds, weights, capacities) -> "RefProblem":
        h = P()
        arrs = [np.ascontiguousarray(stream_offsets, np.int64), np.ascontiguousarray(routes, np.int32),
                np.ascontiguousarray(kinds, np.uint8), np.ascontiguousarray(weights, np.float64),
                np.ascontiguousarray(capacities, np.float64)]
        rc = self.L.ref_build_problem(n, m, *[_p(a) for a in arrs], C.byref(h))
        if rc:
            return rc, self.L.ref_last_error().decode()
        return RefProblem(self, h)

    def prox_log(self, z, w, rho, tau):
        return self.L.ref_prox_log(z, w, rho, tau)

    def prox_linear_nonneg(self, z, w, rho, tau):
        return self.L.ref_prox_linear_nonneg(z, w, rho, tau)


def _cfg_arrays(cfg: Config):
    d = np.array([cfg.eps_abs, cfg.rho0, cfg.alpha, cfg.mu, cfg.gamma, cfg.time_limit], np.float64)
    i = np.array([cfg.rho_update_interval, cfg.max_iters, cfg.trace_every, cfg.threads], np.int64)
    return d, i


def ref_write_trace_csv(ref: "Reference", path, it, r, s, rho, obj):
    """io.hpp:393-404 through the reference."""
    arrs = [np.ascontiguousarray(it, np.int64)] + [np.ascontiguousarray(a, np.float64) for a in (r, s, rho, obj)]
    ref._err(ref.L.ref_write_trace_csv(os.fsencode(path), len(arrs[0]), *[_p(a) for a in arrs]))


class RefProblem:
    def __init__(self, ref: Reference, h):
        self.ref = ref
        self.h = h
        self.dropped = 0
        m, n, nnz = I64(), I64(), I64()
        ref.L.ref_sizes(h, C.byref(m), C.byref(n), C.byref(nnz))
        self.m, self.n, self.nnz = m.value, n.value, nnz.value

    def __del__(self):
        try:
            self.ref.L.ref_free(self.h)
        except Exception:
            pass

    def arrays(self) -> Arrays:
        m, n, nnz = self.m, self.n, self.nnz
        J = nnz + m
        a = Arrays(m, n, np.empty(m), np.empty(n), np.empty(n, np.uint8), np.empty(n + 1, np.int64),
                   np.empty(J, np.int32), np.empty(m + 1, np.int64), np.empty(J, np.int64), np.empty(m, np.int32))
        self.ref.L.ref_export(self.h, _p(a.capacities), _p(a.weights), _p(a.kinds), _p(a.stream_offsets),
                              _p(a.terminal_link), _p(a.link_offsets), _p(a.link_terminals), _p(a.link_counts))
        return a

    def groups(self):
        """group_streams (model.hpp:255-286): list of (tau, kind, members)."""
        ng, nm = I64(), I64()
        self.ref.L.ref_groups(self.h, C.byref(ng), C.byref(nm), None, None, None, None)
        tau, kind = np.empty(ng.value, np.int32), np.empty(ng.value, np.int32)
        cnt, mem = np.empty(ng.value, np.int64), np.empty(nm.value, np.int64)
        self.ref.L.ref_groups(self.h, C.byref(ng), C.byref(nm), _p(tau), _p(kind), _p(cnt), _p(mem))
        ends = np.cumsum(cnt)
        return [(int(t), int(k), mem[e - c:e]) for t, k, c, e in zip(tau, kind, cnt, ends)]

    def write_problem(self, path, encoding="auto"):
        self.ref._err(self.ref.L.ref_write_problem(self.h, os.fsencode(path),
                                                   {"auto": 0, "text": 1, "binary": 2}[encoding]))

    def transit_meta(self):
        """(od, route, t0) per stream and (origin, dest) per OD (transit.hpp:35-57)."""
        k = I64()
        self.ref.L.ref_transit_meta(self.h, C.byref(k), None, None, None, None, None)
        od, route, t0 = (np.empty(self.n, np.int32) for _ in range(3))
        origin, dest = np.empty(k.value, np.int32), np.empty(k.value, np.int32)
        self.ref.L.ref_transit_meta(self.h, C.byref(k), _p(od), _p(route), _p(t0), _p(origin), _p(dest))
        return od, route, t0, origin, dest

    def write_transit_metadata(self, path):
        self.ref._err(self.ref.L.ref_write_transit_metadata(self.h, os.fsencode(path)))

    def transit_report(self, x, lam, od, t0, csv_path):
        """transit_report rows (stream ids, pi, lambda_hat per row) and the
        reference CLI's CSV of them at csv_path."""
        x = np.ascontiguousarray(x, np.float64)
        lam = np.ascontiguousarray(lam, np.float64)
        cap = self.nnz
        nrows = I64()
        stream, pi, hl = np.empty(self.n, np.int64), np.empty(self.n), np.empty(self.n, np.int64)
        hats = np.empty(max(cap, 1))
        self.ref._err(self.ref.L.ref_transit_report(self.h, _p(x), _p(lam), od, t0, os.fsencode(csv_path),
                                                    C.byref(nrows), _p(stream), _p(pi), _p(hl), _p(hats), cap))
        k = nrows.value
        ends = np.cumsum(hl[:k])
        rows = [hats[e - l:e] for e, l in zip(ends, hl[:k])]
        return stream[:k], pi[:k], rows

    def degrade(self, p_degrade, factor, seed) -> "RefProblem":
        h = P()
        self.ref._err(self.ref.L.ref_degrade(self.h, p_degrade, factor, seed, C.byref(h)))
        return RefProblem(self.ref, h)

    def fail_and_prune(self, p_fail, seed) -> "RefProblem":
        h = P()
        self.ref._err(self.ref.L.ref_fail_and_prune(self.h, p_fail, seed, C.byref(h)))
        out = RefProblem(self.ref, h)
        out.prior_m, out.prior_n = self.m, self.n
        return out

    def prune_maps(self):
        """(link_map[prior m], stream_map[prior n]) of a fail_and_prune result."""
        lm = np.empty(self.prior_m, np.int32)
        sm = np.empty(self.prior_n, np.int64)
        self.ref.L.ref_prune_maps(self.h, _p(lm), _p(sm))
        return lm, sm

    def solve(self, cfg: Config, warm=None, final_state=False) -> Result:
        d, i = _cfg_arrays(cfg)
        m, n, J = self.m, self.n, self.nnz + self.m
        x, s, lam, lraw = np.empty(n), np.empty(m), np.empty(m), np.empty(m)
        scal = np.empty(5)
        ints = np.empty(3, np.int64)
        cap = cfg.max_iters // cfg.trace_every + 2
        trace = np.empty((cap, 5))
        fp = fz = fpb = fpr = fpz = None
        if final_state:
            fp, fz, fpb, fpr, fpz = np.empty(J), np.empty(J), np.empty(m), np.empty(m), np.empty(J)
        wx = wp = None
        wr = 0.0
        if warm is not None:
            wx = np.ascontiguousarray(warm[0], np.float64)
            wp = None if warm[1] is None else np.ascontiguousarray(warm[1], np.float64)
            wr = float(warm[2])
        rc = self.ref.L.ref_solve(self.h, _p(d), _p(i), _p(wx), _p(wp), wr, _p(x), _p(s), _p(lam), _p(lraw),
                                  _p(scal), _p(ints), _p(trace), cap, _p(fp), _p(fz), _p(fpb), _p(fpr), _p(fpz))
        res = Result(x, s, lam, lraw, scal[0], int(ints[0]), int(ints[1]), scal[1], scal[2], scal[3],
                     trace[: min(int(ints[2]), cap)].copy(), scal[4], fp, fz, fpb, fpr, fpz)
        if rc:
            res.error = self.ref.L.ref_last_error().decode()
        return res

    def steps(self, cfg: Config, k: int, init="cold", state=None, warm=None):
        """Run k PmpSolver::step calls; returns (state dict, rs array k x 2)."""
        d, i = _cfg_arrays(cfg)
        m, J = self.m, self.nnz + self.m
        if state is None:
            st = dict(p=np.zeros(J), z=np.zeros(J), p_bar=np.zeros(m), price=np.zeros(m), rho=cfg.rho0, iter=0)
        else:
            st = {kk: (v.copy() if isinstance(v, np.ndarray) else v) for kk, v in state.items()}
        rho = D(st["rho"])
        it = I64(st["iter"])
        rs = np.empty((max(k, 1), 2))
        mode = {"cold": 0, "warm": 1, "state": 2}[init]
        wx = wp = None
        wr = 0.0
        if warm is not None:
            wx = np.ascontiguousarray(warm[0], np.float64)
            wp = None if warm[1] is None else np.ascontiguousarray(warm[1], np.float64)
            wr = float(warm[2])
        self.ref._err(self.ref.L.ref_steps(self.h, _p(d), _p(i), mode, _p(wx), _p(wp), wr, k, _p(st["p"]),
                                           _p(st["z"]), _p(st["p_bar"]), _p(st["price"]), C.byref(rho),
                                           C.byref(it), _p(rs)))
        st["rho"] = rho.value
        st["iter"] = it.value
        return st, rs[:k]

    def time_iterations(self, cfg: Config, iters: int):
        """Wall seconds of `iters` iterations of the reference run loop."""
        d, i = _cfg_arrays(cfg)
        secs = np.zeros(1)
        last = np.zeros(2)
        self.ref._err(self.ref.L.ref_time_iterations(self.h, _p(d), _p(i), iters, _p(secs), _p(last)))
        return float(secs[0]), last

    def bench_session(self, cfg: Config) -> "RefBenchSession":
        return RefBenchSession(self, cfg)

    def warm_after_degrade(self, after: "RefProblem", prior: Result):
        x0, price, rho = np.empty(after.n), np.empty(after.m), np.zeros(1)
        self.ref._err(self.ref.L.ref_warm_after_degrade(self.h, after.h, _p(prior.x), _p(prior.lambda_raw),
                                                        prior.rho_final, _p(x0), _p(price), _p(rho)))
        return x0, price, float(rho[0])

    def warm_after_prune(self, prior: Result, prior_n: int, prior_m: int):
        x0, price, rho = np.empty(self.n), np.empty(self.m), np.zeros(1)
        self.ref._err(self.ref.L.ref_warm_after_prune(self.h, _p(prior.x), prior_n, _p(prior.lambda_raw), prior_m,
                                                      prior.rho_final, _p(x0), _p(price), _p(rho)))
        return x0, price, float(rho[0])


class RefBenchSession:
    """A reference PmpSolver held open for timing its stock solve() (ref_bench_*)."""

    def __init__(self, rp: RefProblem, cfg: Config):
        self.rp = rp
        d, i = _cfg_arrays(cfg)
        self.h = P()
        rp.ref._err(rp.ref.L.ref_bench_open(rp.h, _p(d), _p(i), C.byref(self.h)))

    def solve(self):
        """One stock PmpSolver::solve() on the held solver: (seconds, status, iterations)."""
        secs = np.zeros(1)
        ints = np.zeros(2, np.int64)
        rs = np.zeros(2)
        self.rp.ref._err(self.rp.ref.L.ref_bench_solve(self.h, _p(secs), _p(ints), _p(rs)))
        return float(secs[0]), int(ints[0]), int(ints[1])

    def close(self):
        if self.h:
            self.rp.ref.L.ref_bench_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def arrays_from(problem) -> Arrays:
    """Oracle arrays for a product ``Problem`` (layout via the restatement)."""
    o = Restatement()
    tl, lo, lt, lc = o.build_layout(problem.m, problem.n, problem.stream_offsets, problem.route_links)
    return Arrays(problem.m, problem.n, problem.capacities, problem.weights, problem.kinds, problem.stream_offsets,
                  tl, lo, lt, lc)
