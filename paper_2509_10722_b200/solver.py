"""The PMP engine API -- a Python mirror of the reference's
``proj/include/numpmp/solver.hpp`` (``SolverConfig``, ``SolverState``,
``Solution``, ``WarmStart``, ``PmpSolver`` and the free functions), backed by
the sm_100a engine in libnumpmp_cuda.so through its C-ABI.

Every ``PmpSolver`` method runs on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from .errors import SolverError, raise_for
from .model import Problem, StreamKind


@dataclass
class SolverConfig:  # solver.hpp:19-30
    eps_abs: float = 1e-5
    rho0: float = 1.0
    alpha: float = 1.6
    mu: float = 2.0
    gamma: float = 1.1
    rho_update_interval: int = 50
    max_iters: int = 50000
    trace_every: int = 10
    threads: int = 0
    time_limit: float = 0.0

    def _c(self) -> _lib.Config:
        return _lib.Config(
            self.eps_abs, self.rho0, self.alpha, self.mu, self.gamma, self.time_limit,
            self.rho_update_interval, self.max_iters, self.trace_every, self.threads, 0,
        )


@dataclass
class SolverState:  # solver.hpp:51-62 (terminal space)
    p: np.ndarray
    z: np.ndarray
    p_bar: np.ndarray
    price: np.ndarray
    rho: float = 1.0
    iter: int = 0

    def u(self, link: int) -> float:
        return float(self.price[link] / self.rho)

    def copy(self) -> "SolverState":
        return SolverState(self.p.copy(), self.z.copy(), self.p_bar.copy(), self.price.copy(), self.rho, self.iter)


@dataclass
class TraceRecord:  # solver.hpp:64-70
    iter: int
    r_norm: float
    s_norm: float
    rho: float
    objective: float


class SolveStatus(IntEnum):  # solver.hpp:74
    Converged = 0
    MaxIters = 1
    TimeLimit = 2


def to_string(status: SolveStatus) -> str:
    return {0: "converged", 1: "maxiters", 2: "timelimit"}[int(status)]


@dataclass
class Solution:  # solver.hpp:85-97 (``lambda`` is spelled ``lambda_``)
    x: np.ndarray
    s: np.ndarray
    lambda_: np.ndarray
    lambda_raw: np.ndarray
    objective: float = 0.0
    status: SolveStatus = SolveStatus.MaxIters
    iterations: int = 0
    r_norm: float = 0.0
    s_norm: float = 0.0
    rho_final: float = 0.0
    trace: List[TraceRecord] = field(default_factory=list)


@dataclass
class WarmStart:  # solver.hpp:101-105
    x0: np.ndarray
    price: Optional[np.ndarray] = None  # None -> start prices at zero
    rho: float = 0.0  # 0 -> use config rho0


# ------------------------------------------------------------ free functions
def check_termination(r_norm: float, s_norm: float, total_terminals: int, config: SolverConfig) -> bool:
    """solver.hpp:157-163: both norms strictly below eps_abs * sqrt(J)."""
    eps_tol = config.eps_abs * math.sqrt(float(total_terminals))
    return r_norm < eps_tol and s_norm < eps_tol


def update_rho(state: SolverState, r_norm: float, s_norm: float, config: SolverConfig) -> None:
    """solver.hpp:168-174 (the unscaled price is left untouched)."""
    if r_norm > config.mu * s_norm:
        state.rho *= config.gamma
    elif s_norm > config.mu * r_norm:
        state.rho /= config.gamma


def recover_duals(state: SolverState) -> np.ndarray:
    """solver.hpp:177-182: lambda = max(price, 0)."""
    return np.where(state.price < 0.0, 0.0, state.price)


def _check(h, rc):
    if rc:
        raise_for(rc, _lib.lib().numpmp_gpu_last_error(h).decode())


class PmpSolver:
    """Device-resident PMP engine with the reference's PmpSolver interface
    (solver.hpp:265-519).  ``device`` selects the CUDA device."""

    def __init__(self, problem: Problem, config: Optional[SolverConfig] = None, extensions=None, device: int = 0):
        self._problem = problem
        self._cfg = config if config is not None else SolverConfig()
        if extensions is not None:
            raise SolverError("extension utilities are not supported by the device engine")
        L = _lib.lib()
        h = C.c_void_p()
        view = problem.view()
        rc = L.numpmp_gpu_create(C.byref(view), C.byref(self._cfg._c()), device, C.byref(h))
        if rc:
            raise_for(rc, L.numpmp_gpu_last_error(None).decode())
        self._h = h
        self._final: Optional[Tuple[SolverState, np.ndarray]] = None
        self._groups = None

    # solver.hpp:289-291
    def problem(self) -> Problem:
        return self._problem

    def config(self) -> SolverConfig:
        return self._cfg

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().numpmp_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---------------------------------------------------------------- states
    def _download_state(self, with_prev_z=False):
        p = self._problem
        J = p.nnz + p.m
        st = SolverState(np.empty(J), np.empty(J), np.empty(p.m), np.empty(p.m))
        rho = C.c_double()
        it = C.c_int64()
        prev = np.empty(J) if with_prev_z else None
        _check(self._h, _lib.lib().numpmp_gpu_get_state(
            self._h, _lib.ptr(st.p), _lib.ptr(st.z), _lib.ptr(st.p_bar), _lib.ptr(st.price),
            C.byref(rho), C.byref(it), _lib.ptr(prev)))
        st.rho = rho.value
        st.iter = it.value
        return st, prev

    def cold_state(self) -> SolverState:
        """solver.hpp:293-303."""
        _check(self._h, _lib.lib().numpmp_gpu_set_cold(self._h))
        return self._download_state()[0]

    def warm_state(self, warm: WarmStart) -> SolverState:
        """solver.hpp:305-314 + warm_start_from 218-259."""
        self._set_warm(warm)
        return self._download_state()[0]

    def _set_warm(self, warm: WarmStart) -> None:
        p = self._problem
        x0 = np.ascontiguousarray(warm.x0, np.float64)
        if x0.shape[0] != p.n:
            raise ValueError("warm start: x0 length does not match n")
        price = None
        if warm.price is not None and len(warm.price) > 0:
            price = np.ascontiguousarray(warm.price, np.float64)
            if price.shape[0] != p.m:
                raise ValueError("warm start: price length mismatch")
        _check(self._h, _lib.lib().numpmp_gpu_set_warm(self._h, _lib.ptr(x0), _lib.ptr(price), float(warm.rho)))

    def step(self, state: SolverState) -> Tuple[float, float]:
        """solver.hpp:316-409: one iteration on the device; ``state`` is
        updated in place; returns (r_norm, s_norm)."""
        L = _lib.lib()
        arrs = [np.ascontiguousarray(a, np.float64) for a in (state.p, state.z, state.p_bar, state.price)]
        _check(self._h, L.numpmp_gpu_set_state(self._h, *[_lib.ptr(a) for a in arrs], float(state.rho), int(state.iter)))
        r, s = C.c_double(), C.c_double()
        _check(self._h, L.numpmp_gpu_step(self._h, C.byref(r), C.byref(s)))
        new, _ = self._download_state()
        state.p, state.z, state.p_bar, state.price = new.p, new.z, new.p_bar, new.price
        state.rho, state.iter = new.rho, new.iter
        return r.value, s.value

    def residuals(self, state: SolverState, prev: SolverState) -> Tuple[float, float]:
        """residuals(state, prev, layout) (solver.hpp:139-154) on the device:
        the reduction step() uses, so step() returns exactly
        ``residuals(after, before)`` for the states it issued."""
        p = self._problem
        J = p.nnz + p.m
        pb = np.ascontiguousarray(state.p_bar, np.float64)
        z = np.ascontiguousarray(state.z, np.float64)
        zp = np.ascontiguousarray(prev.z, np.float64)
        if pb.shape[0] != p.m or z.shape[0] != J or zp.shape[0] != J:
            raise ValueError("residuals: state arrays do not fit the problem")
        r, s = C.c_double(), C.c_double()
        _check(self._h, _lib.lib().numpmp_gpu_residuals(self._h, _lib.ptr(pb), _lib.ptr(z), _lib.ptr(zp),
                                                        float(state.rho), C.byref(r), C.byref(s)))
        return r.value, s.value

    def groups(self):
        """solver.hpp:291 groups(): group_streams of the problem (model.hpp:246-286).
        The device engine does not batch by group; this is the reference's
        partition, for callers that inspect it."""
        if self._groups is None:
            from .model import group_streams

            self._groups = group_streams(self._problem)
        return self._groups

    # ------------------------------------------- warm-start recipes (warm.hpp)
    def warm_start_after_degrade(self, before: "Problem", prior: Solution) -> WarmStart:
        """warm.hpp:25-57 computed on the device for this solver's (degraded)
        problem; the warm state is applied, so solve_prepared() continues
        from it.  Returns the recipe's WarmStart."""
        p = self._problem
        if before.m != p.m or before.n != p.n:
            raise ValueError("degrade warm start: problems differ in structure")
        x0, price, rho = np.empty(p.n), np.empty(p.m), C.c_double()
        cap_b = np.ascontiguousarray(before.capacities, np.float64)
        px = np.ascontiguousarray(prior.x, np.float64)
        pl = np.ascontiguousarray(prior.lambda_raw, np.float64)
        _check(self._h, _lib.lib().numpmp_gpu_warm_after_degrade(
            self._h, _lib.ptr(cap_b), _lib.ptr(px), _lib.ptr(pl), float(prior.rho_final), _lib.ptr(x0),
            _lib.ptr(price), C.byref(rho)))
        return WarmStart(x0, price, rho.value)

    def warm_start_after_prune(self, prune_map, prior: Solution) -> WarmStart:
        """warm.hpp:62-94 on the device for this solver's (pruned) problem;
        the projection onto the survivors is the PruneMap's host gather."""
        p = self._problem
        x0p = prune_map.project_streams(prior.x)
        prp = prune_map.project_links(prior.lambda_raw)
        if x0p.shape[0] != p.n or prp.shape[0] != p.m:
            raise ValueError("prune warm start: map does not fit problem")
        x0, price, rho = np.empty(p.n), np.empty(p.m), C.c_double()
        _check(self._h, _lib.lib().numpmp_gpu_warm_after_prune(
            self._h, _lib.ptr(x0p), _lib.ptr(prp), float(prior.rho_final), _lib.ptr(x0), _lib.ptr(price),
            C.byref(rho)))
        return WarmStart(x0, price, rho.value)

    def path_prices(self, lam) -> np.ndarray:
        """transit.hpp:290-302 on the device (route-order sums)."""
        lam = np.ascontiguousarray(lam, np.float64)
        if lam.shape[0] != self._problem.m:
            raise ValueError("path_prices: lambda length mismatch")
        pi = np.empty(self._problem.n)
        _check(self._h, _lib.lib().numpmp_gpu_path_prices(self._h, _lib.ptr(lam), _lib.ptr(pi)))
        return pi

    def solve_prepared(self) -> Solution:
        """run() from the state the last warm-start recipe applied."""
        return self._run()

    # ----------------------------------------------------------------- solve
    def solve(self, warm: Optional[WarmStart] = None) -> Solution:
        """solver.hpp:411-413 + run 441-508, entirely on the device."""
        if warm is None:
            _check(self._h, _lib.lib().numpmp_gpu_set_cold(self._h))
        else:
            self._set_warm(warm)
        return self._run()

    def _run(self) -> Solution:
        p = self._problem
        cfg = self._cfg
        x = np.empty(p.n)
        s = np.empty(p.m)
        lam = np.empty(p.m)
        lam_raw = np.empty(p.m)
        info = _lib.SolutionInfo()
        cap = cfg.max_iters // cfg.trace_every + 2
        trace = (_lib.TraceRow * cap)()
        self._final = None
        _check(self._h, _lib.lib().numpmp_gpu_run(
            self._h, _lib.ptr(x), _lib.ptr(s), _lib.ptr(lam), _lib.ptr(lam_raw), C.byref(info), trace, cap))
        rows = [TraceRecord(trace[i].iter, trace[i].r_norm, trace[i].s_norm, trace[i].rho, trace[i].objective)
                for i in range(min(info.trace_len, cap))]
        return Solution(x, s, lam, lam_raw, info.objective, SolveStatus(info.status), info.iterations,
                        info.r_norm, info.s_norm, info.rho_final, rows)

    # solver.hpp:415-417
    def final_state(self) -> SolverState:
        if self._final is None:
            self._final = self._download_state(with_prev_z=True)
        return self._final[0]

    def final_prev_z(self) -> np.ndarray:
        if self._final is None:
            self._final = self._download_state(with_prev_z=True)
        return self._final[1]

    # ------------------------------------------------------------ device info
    def export_layout(self):
        """The device-built link-major CSR in the reference's TerminalLayout
        form: (link_offsets, link_terminals, link_counts)."""
        p = self._problem
        lo = np.empty(p.m + 1, np.int64)
        lt = np.empty(p.nnz + p.m, np.int64)
        lc = np.empty(p.m, np.int32)
        _check(self._h, _lib.lib().numpmp_gpu_export_layout(self._h, _lib.ptr(lo), _lib.ptr(lt), _lib.ptr(lc)))
        return lo, lt, lc

    def handle(self):
        return self._h


def objective(problem: Problem, x: np.ndarray) -> float:
    """solver.hpp:186-213 for log/linear streams (host reporting helper)."""
    x = np.asarray(x, np.float64)
    if x.shape[0] != problem.n:
        raise ValueError("objective: x length mismatch")
    lg = problem.kinds == int(StreamKind.Log)
    if np.any(~(x[lg] > 0.0)):
        from .errors import DomainError

        bad = int(np.flatnonzero(lg & ~(x > 0.0))[0])
        raise DomainError(f"objective: log stream {bad} has non-positive rate")
    with np.errstate(divide="ignore"):
        terms = np.where(lg, problem.weights * np.log(np.where(lg, x, 1.0)), problem.weights * x)
    return float(np.sum(terms))
