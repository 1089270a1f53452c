"""Problem model, generators and validation -- the host side of the hot path.

Mirrors the reference's ``proj/include/numpmp/model.hpp`` and ``gen.hpp``
names and semantics (``Stream``, ``Problem``, ``TerminalLayout``,
``build_problem``, ``validate``, ``GenSpec``, ``gen_uncongested``, ...).
Problems are held in the compact stream-major form the device consumes
(``stream_offsets`` + ``route_links`` = ``TerminalLayout::terminal_link[0:nnz)``)
plus per-stream ``weights``/``kinds`` and per-link ``capacities``.  The
heavy lifting (generation, validation, layout) runs in C++ in
libnumpmp_cuda.so (csrc/host_gen.cpp).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import GenError, ValidationError


class StreamKind(IntEnum):  # model.hpp:18
    Log = 0
    Linear = 1
    Extension = 2


@dataclass
class Stream:  # model.hpp:32-38
    id: int = -1
    kind: StreamKind = StreamKind.Log
    extension: str = ""
    weight: float = 1.0
    route: List[int] = field(default_factory=list)


@dataclass
class TerminalLayout:  # model.hpp:47-57
    total_terminals: int
    nnz: int
    stream_offsets: np.ndarray  # int64 n+1
    terminal_link: np.ndarray  # int32 J
    link_offsets: np.ndarray  # int64 m+1
    link_terminals: np.ndarray  # int64 J
    link_counts: np.ndarray  # int32 m

    def slack_terminal(self, link: int) -> int:
        return self.nnz + link


class Problem:
    """model.hpp:59-65 in stream-major array form."""

    def __init__(self, m, n, capacities, weights, kinds, stream_offsets, route_links):
        self.m = int(m)
        self.n = int(n)
        self.capacities = np.ascontiguousarray(capacities, dtype=np.float64)
        self.weights = np.ascontiguousarray(weights, dtype=np.float64)
        self.kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
        self.stream_offsets = np.ascontiguousarray(stream_offsets, dtype=np.int64)
        self.route_links = np.ascontiguousarray(route_links, dtype=np.int32)
        self._layout: Optional[TerminalLayout] = None

    @property
    def nnz(self) -> int:
        return int(self.stream_offsets[-1])

    @property
    def total_terminals(self) -> int:
        return self.nnz + self.m

    def route(self, j: int) -> np.ndarray:
        return self.route_links[self.stream_offsets[j] : self.stream_offsets[j + 1]]

    @property
    def streams(self) -> List[Stream]:
        return [
            Stream(j, StreamKind(int(self.kinds[j])), "", float(self.weights[j]), self.route(j).tolist())
            for j in range(self.n)
        ]

    @property
    def layout(self) -> TerminalLayout:
        """The reference TerminalLayout (model.hpp:159-201), built on the host."""
        if self._layout is None:
            m, n, nnz = self.m, self.n, self.nnz
            J = nnz + m
            tl = np.empty(J, np.int32)
            lo = np.empty(m + 1, np.int64)
            lt = np.empty(J, np.int64)
            lc = np.empty(m, np.int32)
            _lib.lib().numpmp_build_layout(
                m, n, _lib.ptr(self.stream_offsets), _lib.ptr(self.route_links), _lib.ptr(tl),
                _lib.ptr(lo), _lib.ptr(lt), _lib.ptr(lc),
            )
            self._layout = TerminalLayout(J, nnz, self.stream_offsets, tl, lo, lt, lc)
        return self._layout

    def view(self) -> _lib.ProblemView:
        return _lib.ProblemView(
            self.m, self.n, self.nnz,
            self.capacities.ctypes.data, self.weights.ctypes.data, self.kinds.ctypes.data,
            self.stream_offsets.ctypes.data, self.route_links.ctypes.data,
        )

    def with_capacities(self, capacities) -> "Problem":
        return Problem(self.m, self.n, capacities, self.weights, self.kinds, self.stream_offsets, self.route_links)


def validate(problem: Problem) -> int:
    """Number of model violations (model.hpp:76-155)."""
    return _validate(problem)[0]


def _validate(p: Problem):
    buf = C.create_string_buffer(4096)
    nv = _lib.lib().numpmp_validate(
        p.m, p.n, _lib.ptr(p.capacities), _lib.ptr(p.weights), _lib.ptr(p.kinds),
        _lib.ptr(p.stream_offsets), _lib.ptr(p.route_links), buf, len(buf),
    )
    return int(nv), buf.value.decode()


def problem_from_arrays(m, n, capacities, weights, kinds, stream_offsets, route_links) -> Problem:
    p = Problem(m, n, capacities, weights, kinds, stream_offsets, route_links)
    nv, msg = _validate(p)
    if nv:
        raise ValidationError(msg)
    return p


def build_problem(streams: Sequence[Stream], capacities: Sequence[float]) -> Problem:
    """model.hpp:222-241: dense ids, validation, layout."""
    if len(streams) == 0:
        raise ValidationError("stream list is empty")
    if len(capacities) == 0:
        raise ValidationError("capacity list is empty")
    n = len(streams)
    offsets = np.zeros(n + 1, np.int64)
    for j, s in enumerate(streams):
        offsets[j + 1] = offsets[j] + len(s.route)
    routes = np.zeros(int(offsets[-1]), np.int32)
    for j, s in enumerate(streams):
        routes[offsets[j] : offsets[j + 1]] = s.route
    kinds = np.array([int(s.kind) for s in streams], np.uint8)
    weights = np.array([s.weight for s in streams], np.float64)
    return problem_from_arrays(len(capacities), n, np.asarray(capacities, np.float64), weights, kinds, offsets, routes)


# ---------------------------------------------------------------- generators
@dataclass
class TypeGroup:  # model.hpp:243-253
    kind: StreamKind
    extension: str
    tau: int
    members: np.ndarray         # stream ids, ascending
    weights: np.ndarray
    terminal_links: np.ndarray  # [tau][len(members)]: link of terminal i of member k


def group_streams(problem: Problem) -> List[TypeGroup]:
    """model.hpp:255-286: streams partitioned by (tau, kind), ordered by
    ascending tau, then kind, then first member (the extension name is part
    of the key only for Extension streams, which this package rejects)."""
    so = np.asarray(problem.stream_offsets, np.int64)
    tau = np.diff(so)
    kinds = np.asarray(problem.kinds, np.int64)
    key = tau * 8 + kinds
    order = np.lexsort((np.arange(problem.n), key))  # stable: members ascending within a key
    out = []
    if problem.n == 0:
        return out
    ks = key[order]
    cuts = np.flatnonzero(np.diff(ks)) + 1
    for seg in np.split(order, cuts):
        t = int(tau[seg[0]])
        links = problem.route_links[(so[seg][:, None] + np.arange(t)[None, :]).reshape(-1)].reshape(len(seg), t)
        out.append(TypeGroup(StreamKind(int(kinds[seg[0]])), "", t, seg.astype(np.int64),
                             np.asarray(problem.weights, np.float64)[seg], np.ascontiguousarray(links.T)))
    out.sort(key=lambda g: (g.tau, int(g.kind), int(g.members[0])))
    return out


class GenKind(IntEnum):  # gen.hpp:18
    Log = 0
    Linear = 1
    Mixed = 2


@dataclass
class WeightDist:  # gen.hpp:21-33
    uniform_: bool = False
    a: float = 1.0
    b: float = 1.0

    @staticmethod
    def constant(w: float) -> "WeightDist":
        return WeightDist(False, w, w)

    @staticmethod
    def uniform(lo: float, hi: float) -> "WeightDist":
        return WeightDist(True, lo, hi)


@dataclass
class GenSpec:  # gen.hpp:35-44
    m: int = 0
    n: int = 0
    avg_links_per_stream: float = 10.0
    kind: GenKind = GenKind.Log
    weights: WeightDist = field(default_factory=lambda: WeightDist.constant(1.0))
    seed: int = 0

    def _c(self) -> _lib.GenSpecC:
        return _lib.GenSpecC(
            self.m, self.n, self.avg_links_per_stream, int(self.kind),
            1 if self.weights.uniform_ else 0, self.weights.a, self.weights.b, self.seed,
        )


def _from_instance(inst) -> Problem:
    L = _lib.lib()
    m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    L.numpmp_instance_sizes(inst, C.byref(m), C.byref(n), C.byref(nnz))
    caps = np.empty(m.value, np.float64)
    w = np.empty(n.value, np.float64)
    k = np.empty(n.value, np.uint8)
    off = np.empty(n.value + 1, np.int64)
    rl = np.empty(max(nnz.value, 1), np.int32)[: nnz.value]
    L.numpmp_instance_export(inst, _lib.ptr(caps), _lib.ptr(w), _lib.ptr(k), _lib.ptr(off), _lib.ptr(rl))
    L.numpmp_instance_free(inst)
    return Problem(m.value, n.value, caps, w, k, off, rl)


def gen_uncongested(spec: GenSpec) -> Problem:
    """gen.hpp:91-97 (bit-identical to the reference for the same spec)."""
    L = _lib.lib()
    inst = C.c_void_p()
    rc = L.numpmp_gen_uncongested(C.byref(spec._c()), C.byref(inst))
    if rc:
        raise GenError(L.numpmp_host_last_error().decode())
    return _from_instance(inst)


def gen_congested(spec: GenSpec, hot_link_fraction=0.001, hot_stream_fraction=0.10) -> Problem:
    """gen.hpp:103-128."""
    L = _lib.lib()
    inst = C.c_void_p()
    rc = L.numpmp_gen_congested(C.byref(spec._c()), hot_link_fraction, hot_stream_fraction, C.byref(inst))
    if rc:
        raise GenError(L.numpmp_host_last_error().decode())
    return _from_instance(inst)


@dataclass
class TransitSpec:  # transit.hpp:22-32
    stations: int = 0
    time_bins: int = 0
    bin_minutes: float = 5.0
    spatial_edges: int = 0
    od_pairs: int = 0
    routes_per_od: int = 1
    departures_per_route: int = 1
    seats: float = 50.0
    seed: int = 0


@dataclass
class TransitMetadata:  # transit.hpp:41-57 (edges and warnings not carried)
    stations: int
    time_bins: int
    bin_minutes: float
    seats: float
    od_origin: np.ndarray  # per usable OD (TransitMetadata::ods)
    od_dest: np.ndarray
    stream_od: np.ndarray  # per stream (TransitMetadata::streams)
    stream_route: np.ndarray
    stream_t0: np.ndarray
    dropped_streams: int = 0
    # spatial graph and OD routes (edge sequences): OD q's routes are
    # [od_route_ptr[q], od_route_ptr[q+1]), route r's edges
    # route_edges[route_ptr[r]:route_ptr[r+1]]
    edges: Optional[np.ndarray] = None  # (E, 2) int32 (from, to)
    od_route_ptr: Optional[np.ndarray] = None
    route_ptr: Optional[np.ndarray] = None
    route_edges: Optional[np.ndarray] = None

    def link_id(self, edge: int, t: int) -> int:
        return edge * self.time_bins + t


def _transit_meta(inst, spec: "TransitSpec", n: int, dropped: int) -> TransitMetadata:
    L = _lib.lib()
    k = C.c_int64()
    rc = L.numpmp_transit_meta(inst, C.byref(k), None, None, None, None, None)
    if rc:
        raise ValidationError(L.numpmp_host_last_error().decode())
    od, route, t0 = (np.empty(n, np.int32) for _ in range(3))
    origin, dest = np.empty(k.value, np.int32), np.empty(k.value, np.int32)
    L.numpmp_transit_meta(inst, C.byref(k), _lib.ptr(od), _lib.ptr(route), _lib.ptr(t0), _lib.ptr(origin),
                          _lib.ptr(dest))
    ne, nr, nre = C.c_int64(), C.c_int64(), C.c_int64()
    L.numpmp_transit_graph(inst, C.byref(ne), C.byref(nr), C.byref(nre), None, None, None, None, None)
    ef, et = np.empty(ne.value, np.int32), np.empty(ne.value, np.int32)
    orp, rp = np.empty(k.value + 1, np.int64), np.empty(nr.value + 1, np.int64)
    re_ = np.empty(max(nre.value, 1), np.int32)[: nre.value]
    L.numpmp_transit_graph(inst, C.byref(ne), C.byref(nr), C.byref(nre), _lib.ptr(ef), _lib.ptr(et), _lib.ptr(orp),
                           _lib.ptr(rp), _lib.ptr(re_))
    return TransitMetadata(spec.stations, spec.time_bins, spec.bin_minutes, spec.seats, origin, dest, od, route, t0,
                           dropped, np.stack([ef, et], axis=1), orp, rp, re_)


def gen_transit(spec: TransitSpec, with_meta: bool = False):
    """transit.hpp:152-287 (bit-identical streams); returns (Problem, dropped),
    or (Problem, TransitMetadata) with with_meta=True (the reference's pair)."""
    L = _lib.lib()
    inst = C.c_void_p()
    dropped = C.c_int64()
    cs = _lib.TransitSpecC(spec.stations, spec.time_bins, spec.bin_minutes, spec.spatial_edges, spec.od_pairs,
                           spec.routes_per_od, spec.departures_per_route, spec.seats, spec.seed)
    rc = L.numpmp_gen_transit(C.byref(cs), C.byref(inst), C.byref(dropped))
    if rc:
        raise GenError(L.numpmp_host_last_error().decode())
    if with_meta:
        m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        L.numpmp_instance_sizes(inst, C.byref(m), C.byref(n), C.byref(nnz))
        try:
            meta = _transit_meta(inst, spec, n.value, dropped.value)
        except BaseException:
            L.numpmp_instance_free(inst)
            raise
        return _from_instance(inst), meta
    return _from_instance(inst), dropped.value


def degrade(problem: Problem, p_degrade=0.25, factor=0.5, seed=0) -> Problem:
    """gen.hpp:132-143: structure unchanged, capacities cut."""
    caps = problem.capacities.copy()
    L = _lib.lib()
    rc = L.numpmp_degrade(problem.m, _lib.ptr(caps), p_degrade, factor, seed)
    if rc:
        raise GenError(L.numpmp_host_last_error().decode())
    return problem.with_capacities(caps)


@dataclass
class PruneMap:  # gen.hpp:146-178
    link_map: np.ndarray    # old link -> new link or -1 (int32)
    stream_map: np.ndarray  # old stream -> new stream or -1 (int64)

    def removed_streams(self) -> np.ndarray:
        return np.nonzero(self.stream_map < 0)[0].astype(np.int64)

    def project_streams(self, v) -> np.ndarray:
        v = np.asarray(v, np.float64)
        if v.shape[0] != self.stream_map.shape[0]:
            raise ValueError("prune map: stream vector length mismatch")
        return v[self.stream_map >= 0].copy()

    def project_links(self, v) -> np.ndarray:
        v = np.asarray(v, np.float64)
        if v.shape[0] != self.link_map.shape[0]:
            raise ValueError("prune map: link vector length mismatch")
        return v[self.link_map >= 0].copy()


def fail_and_prune(problem: Problem, p_fail=0.25, seed=0):
    """gen.hpp:181-223 (bit-identical): returns (pruned Problem, PruneMap)."""
    L = _lib.lib()
    inst = C.c_void_p()
    lm = np.empty(problem.m, np.int32)
    sm = np.empty(problem.n, np.int64)
    rc = L.numpmp_fail_and_prune(problem.m, problem.n, _lib.ptr(problem.capacities), _lib.ptr(problem.weights),
                                 _lib.ptr(problem.kinds), _lib.ptr(problem.stream_offsets),
                                 _lib.ptr(problem.route_links), p_fail, seed, C.byref(inst), _lib.ptr(lm),
                                 _lib.ptr(sm))
    if rc:
        raise GenError(L.numpmp_host_last_error().decode())
    return _from_instance(inst), PruneMap(lm, sm)


def read_problem(path: str) -> Problem:
    """io.hpp:172-279: text "NUMP 1" or binary "NUMPB 1" (by magic)."""
    from .errors import IoError, ValidationError

    L = _lib.lib()
    inst = C.c_void_p()
    rc = L.numpmp_read_problem(os.fsencode(path), C.byref(inst))
    if rc == 2:
        raise ValidationError(L.numpmp_host_last_error().decode())
    if rc:
        raise IoError(L.numpmp_host_last_error().decode())
    return _from_instance(inst)


def write_problem(problem: Problem, path: str, encoding: str = "auto") -> None:
    """io.hpp:126-170 (encoding: "auto" | "text" | "binary")."""
    from .errors import IoError

    L = _lib.lib()
    enc = {"auto": 0, "text": 1, "binary": 2}[encoding]
    rc = L.numpmp_write_problem(problem.m, problem.n, _lib.ptr(problem.capacities), _lib.ptr(problem.weights),
                                _lib.ptr(problem.kinds), _lib.ptr(problem.stream_offsets),
                                _lib.ptr(problem.route_links), os.fsencode(path), enc)
    if rc:
        raise IoError(L.numpmp_host_last_error().decode())
