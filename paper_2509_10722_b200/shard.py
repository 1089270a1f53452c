"""Multi-GPU stream sharding: one process per GPU.

Streams (columns of R) are split into contiguous ranges balanced by
nonzeros; every rank holds its streams' CSC, a local CSR over all m links,
and a replicated copy of the link state.  Each iteration the ranks run the
stream pass locally, sum their partial link loads R_g x_g (plus two scalar
partials) with one NCCL all-reduce over NVLink inside the device graph, and
then run the identical replicated link update, so every rank takes the same
termination and rho decisions without further communication.

torch.distributed is only plumbing here: it broadcasts the 128-byte NCCL
unique id that the engine's own communicator is built from.
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


class ShardedPmpSolver:
    """PmpSolver over this rank's stream shard; link state replicated."""

    def __init__(self, problem: Problem, config: SolverConfig, rank: int, world: int, nccl_id: bytes,
                 device: int = 0):
        self.full = problem
        self.local, self.stream_begin = local_shard(problem, rank, world)
        self._cfg = config
        L = _lib.lib()
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

    def solve(self) -> Solution:
        """Cold solve; x is this rank's shard, link vectors are global."""
        L = _lib.lib()
        p = self.local
        x, s, lam, lraw = np.empty(p.n), np.empty(p.m), np.empty(p.m), np.empty(p.m)
        info = _lib.SolutionInfo()
        cap = self._cfg.max_iters // self._cfg.trace_every + 2
        trace = (_lib.TraceRow * cap)()
        for rc in (L.numpmp_gpu_set_cold(self._h),
                   L.numpmp_gpu_run(self._h, _lib.ptr(x), _lib.ptr(s), _lib.ptr(lam), _lib.ptr(lraw),
                                    C.byref(info), trace, cap)):
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
