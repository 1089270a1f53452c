"""Multi-GPU stream sharding: one process per GPU.

Streams (columns of R) are split into contiguous ranges balanced by
nonzeros; every rank holds its streams' CSC and a local CSR over all m
links.  Two exchanges are available for the per-iteration sum of the
partial link loads R_g x_g:

* ``exchange="p2p"`` (bench.py's default; pass it explicitly): the fused peer-memory exchange of
  csrc/pmp_p2p.cuh.  Links are owned in contiguous ranges; the link pass
  stores each row's partial load straight into the owner's HBM over NVLink
  (overlapped with the remaining gathers), the owner runs the link epilogue
  for its links only and stores v into every rank's HBM, and all ranks sum
  the same per-rank residual partials in rank order, so they take the same
  termination and rho decisions.  No NCCL kernel sits in the loop.
* ``exchange="nccl"`` (the constructor's default): replicated link state, one NCCL all-reduce of the m
  partial loads (+2 scalars) inside the device graph, replicated epilogue.
  Kept as the library baseline the fused path is measured against.

torch.distributed is only plumbing: it moves the 128-byte NCCL unique id or
the 64-byte CUDA IPC handles of the exchange regions between the ranks.
"""
from __future__ import annotations

import ctypes as C
from typing import Tuple

import numpy as np

from . import _lib
from .errors import raise_for
from .model import Problem
from .solver import Solution, SolverConfig, SolveStatus, TraceRecord


def shard_bounds(stream_offsets: np.ndarray, world: int) -> np.ndarray:
    """Stream boundaries b[0]=0 <= ... <= b[world]=n balancing nnz per rank."""
    so = np.asarray(stream_offsets, np.int64)
    n = so.shape[0] - 1
    nnz = int(so[-1])
    targets = (np.arange(1, world, dtype=np.int64) * nnz) // world
    inner = np.searchsorted(so, targets, side="left")
    b = np.concatenate([[0], np.clip(inner, 0, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(b)


def local_shard(problem: Problem, rank: int, world: int) -> Tuple[Problem, int]:
    """This rank's stream range as a standalone Problem (offsets rebased;
    link ids and capacities global) and its first global stream id."""
    b = shard_bounds(problem.stream_offsets, world)
    j0, j1 = int(b[rank]), int(b[rank + 1])
    so = problem.stream_offsets
    t0, t1 = int(so[j0]), int(so[j1])
    local = Problem(problem.m, j1 - j0, problem.capacities, problem.weights[j0:j1], problem.kinds[j0:j1],
                    so[j0 : j1 + 1] - t0, problem.route_links[t0:t1])
    return local, j0


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    rc = _lib.lib().numpmp_gpu_nccl_unique_id(buf)
    if rc:
        raise_for(rc, _lib.lib().numpmp_gpu_last_error(None).decode())
    return bytes(buf.raw)


def link_owners(m: int, world: int) -> np.ndarray:
    """Owner ranges of the peer-memory exchange: rank q owns links
    [b[q], b[q+1]), mo = ceil(m / world) per rank (pmp_solver.cu create_impl)."""
    mo = -(-m // world)
    return np.minimum(np.arange(world + 1, dtype=np.int64) * mo, m)


def p2p_create(problem: Problem, config: SolverConfig, rank: int, world: int, device: int = 0):
    """Unconnected peer-memory handle of this rank's shard: (handle, local, stream_begin)."""
    local, j0 = local_shard(problem, rank, world)
    L = _lib.lib()
    h = C.c_void_p()
    view = local.view()
    rc = L.numpmp_gpu_create_p2p(C.byref(view), C.byref(config._c()), device, rank, world, j0, problem.n,
                                 C.byref(h))
    if rc:
        raise_for(rc, L.numpmp_gpu_last_error(None).decode())
    return h, local, j0


def p2p_export(h) -> bytes:
    buf = (C.c_char * 64)()
    L = _lib.lib()
    rc = L.numpmp_gpu_p2p_export(h, buf)
    if rc:
        raise_for(rc, L.numpmp_gpu_last_error(h).decode())
    return bytes(buf.raw)


class ShardedPmpSolver:
    """PmpSolver over this rank's stream shard (see the module docstring).

    exchange="p2p" needs ``ipc_allgather``: a callable taking this rank's
    64-byte handle and returning the rank-ordered list of all ranks' handles
    (e.g. torch.distributed.all_gather_object).  Construction is collective.
    """

    def __init__(self, problem: Problem, config: SolverConfig, rank: int, world: int, nccl_id: bytes = None,
                 device: int = 0, exchange: str = "nccl", ipc_allgather=None, handle=None):
        self.full = problem
        self._cfg = config
        self.exchange = exchange
        L = _lib.lib()
        if handle is not None:  # an already connected peer-memory handle (in-process ranks)
            self._h = handle
            self.local, self.stream_begin = local_shard(problem, rank, world)
            return
        if exchange == "p2p":
            if ipc_allgather is None:
                raise ValueError('exchange="p2p" needs ipc_allgather (see the class docstring)')
            h, self.local, self.stream_begin = p2p_create(problem, config, rank, world, device)
            self._h = h
            handles = ipc_allgather(p2p_export(h))
            blob = C.create_string_buffer(b"".join(handles), 64 * world)
            for rc in (L.numpmp_gpu_p2p_connect(h, blob), L.numpmp_gpu_p2p_start(h)):
                if rc:
                    raise_for(rc, L.numpmp_gpu_last_error(h).decode())
            return
        if exchange != "nccl":
            raise ValueError(f"unknown exchange {exchange!r} (p2p | nccl)")
        if nccl_id is None:
            raise ValueError('exchange="nccl" needs the broadcast nccl_id')
        self.local, self.stream_begin = local_shard(problem, rank, world)
        h = C.c_void_p()
        view = self.local.view()
        idbuf = C.create_string_buffer(nccl_id, 128)
        rc = L.numpmp_gpu_create_sharded(C.byref(view), C.byref(config._c()), device, rank, world, idbuf,
                                         self.stream_begin, problem.n, C.byref(h))
        if rc:
            raise_for(rc, L.numpmp_gpu_last_error(None).decode())
        self._h = h

    def handle(self):
        return self._h

    def _start(self):
        L = _lib.lib()
        rc = L.numpmp_gpu_p2p_start(self._h)
        if rc:
            raise_for(rc, L.numpmp_gpu_last_error(self._h).decode())

    def solve(self, warm=None) -> Solution:
        """solve() / solve(WarmStart) (solver.hpp:411-413), collective over the
        ranks.  warm.x0 is the GLOBAL start (each rank takes its shard), price
        is global.  x of the result is this rank's shard; link vectors are
        global and identical on every rank."""
        L = _lib.lib()
        p = self.local
        x, s, lam, lraw = np.empty(p.n), np.empty(p.m), np.empty(p.m), np.empty(p.m)
        info = _lib.SolutionInfo()
        cap = self._cfg.max_iters // self._cfg.trace_every + 2
        trace = (_lib.TraceRow * cap)()
        if warm is None:
            rc = L.numpmp_gpu_set_cold(self._h)
        else:
            xg = np.asarray(warm.x0, np.float64)
            if xg.shape[0] != self.full.n:
                raise ValueError("warm start: x0 length does not match n")
            x0 = np.ascontiguousarray(xg[self.stream_begin:self.stream_begin + p.n])
            price = None
            if warm.price is not None and len(warm.price) > 0:  # empty: start prices at zero (solver.hpp:101-105)
                price = np.ascontiguousarray(warm.price, np.float64)
                if price.shape[0] != p.m:
                    raise ValueError("warm start: price length mismatch")
            rc = L.numpmp_gpu_set_warm(self._h, _lib.ptr(x0), _lib.ptr(price), float(warm.rho))
        if rc:
            raise_for(rc, L.numpmp_gpu_last_error(self._h).decode())
        rc = L.numpmp_gpu_run(self._h, _lib.ptr(x), _lib.ptr(s), _lib.ptr(lam), _lib.ptr(lraw), C.byref(info),
                              trace, cap)
        if rc:
            raise_for(rc, L.numpmp_gpu_last_error(self._h).decode())
        rows = [TraceRecord(trace[i].iter, trace[i].r_norm, trace[i].s_norm, trace[i].rho, trace[i].objective)
                for i in range(min(info.trace_len, cap))]
        return Solution(x, s, lam, lraw, info.objective, SolveStatus(info.status), info.iterations,
                        info.r_norm, info.s_norm, info.rho_final, rows)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().numpmp_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def p2p_local_group(problem: Problem, config: SolverConfig, world: int, device: int = 0):
    """`world` peer-memory ranks of one problem inside this process (one GPU,
    or several with peer access), wired and started.  Every collective call
    on them (solve, set_warm, step) must then be made from one thread per
    rank, e.g. with run_ranks()."""
    L = _lib.lib()
    made = [p2p_create(problem, config, r, world, device) for r in range(world)]
    arr = (C.c_void_p * world)(*[m[0] for m in made])
    rc = L.numpmp_gpu_p2p_connect_local(arr, world)
    if rc:
        raise_for(rc, L.numpmp_gpu_last_error(None).decode())
    solvers = [ShardedPmpSolver(problem, config, r, world, exchange="p2p", handle=made[r][0]) for r in range(world)]
    run_ranks([lambda s=s: s._start() for s in solvers])
    return solvers


def run_ranks(fns):
    """Run one callable per rank concurrently (threads; the C calls release
    the GIL) and return their results in rank order; re-raises the first error."""
    import threading

    out = [None] * len(fns)
    err = [None] * len(fns)

    def go(i):
        try:
            out[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001
            err[i] = e

    ts = [threading.Thread(target=go, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
