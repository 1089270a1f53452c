"""Reports around a solution: the transit route report
(transit.hpp:304-374) and the trace CSV (io.hpp:393-404).

The per-stream path prices come from the device (PmpSolver.path_prices,
transit.hpp:290-302) when a solver is passed; the report itself only touches
the few streams of one (OD, departure) and is assembled on the host, as in
the reference.
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import IoError, ValidationError
from .model import Problem, TransitMetadata


@dataclass
class TransitReportRow:  # transit.hpp:332-340
    stream: int
    od: int
    route: int
    t0: int
    x: float
    pi: float
    lambda_hat: List[float] = field(default_factory=list)


def _route(problem: Problem, j: int) -> np.ndarray:
    so = problem.stream_offsets
    return problem.route_links[int(so[j]):int(so[j + 1])]


def normalized_route_prices(problem: Problem, lam, stream_ids: Sequence[int]) -> List[List[float]]:
    """transit.hpp:304-325: link prices along each route over the maximum on
    the union of the routes (0 when that maximum is not positive)."""
    lam = np.asarray(lam, np.float64)
    max_price = 0.0
    for j in stream_ids:
        for l in _route(problem, j):
            max_price = max(max_price, float(lam[l]))  # std::max(max, v): NaN-free prices
    return [[float(lam[l]) / max_price if max_price > 0.0 else 0.0 for l in _route(problem, j)] for j in stream_ids]


def transit_report(problem: Problem, x, lam, meta: TransitMetadata, od: int, t0: int,
                   pi: Optional[np.ndarray] = None, solver=None) -> List[TransitReportRow]:
    """transit.hpp:342-374.  pi: the path prices if already computed; else the
    solver's device path_prices when `solver` is given; else the selected
    streams' route sums in route order (the same bits as path_prices)."""
    # std::invalid_argument in the reference (transit.hpp:292,343,349) -> ValueError
    if len(meta.stream_od) != problem.n:
        raise ValueError("transit report: metadata does not match problem")
    k = len(meta.od_origin)
    if od < 0 or od >= k:
        raise ValueError(f"unknown OD id {od}; available: 0..{k - 1}")
    selected = np.flatnonzero((meta.stream_od == od) & (meta.stream_t0 == t0)).tolist()
    lam = np.asarray(lam, np.float64)
    if lam.shape[0] != problem.m:
        raise ValueError("path_prices: lambda length mismatch")
    hats = normalized_route_prices(problem, lam, selected)
    if pi is None and solver is not None:
        pi = solver.path_prices(lam)
    rows = []
    for i, j in enumerate(selected):
        if pi is not None:
            p = float(pi[j])
        else:
            p = 0.0
            for l in _route(problem, j):  # sequential, route order (transit.hpp:296-298)
                p += float(lam[l])
        rows.append(TransitReportRow(j, int(meta.stream_od[j]), int(meta.stream_route[j]), int(meta.stream_t0[j]),
                                     float(x[j]), p, hats[i]))
    return rows


def write_transit_report_csv(rows: Sequence[TransitReportRow], path: str) -> None:
    """The CSV the reference CLI writes for a report (tools/numpmp.cpp:333-342;
    default ostream formatting, i.e. %g)."""
    try:
        with open(path, "w", newline="\n") as f:
            f.write("stream,od,route,t0,x,pi,lambda_hat_path\n")
            for r in rows:
                hat = " ".join("%g" % v for v in r.lambda_hat)
                f.write(f"{r.stream},{r.od},{r.route},{r.t0},{'%g' % r.x},{'%g' % r.pi},\"{hat}\"\n")
    except OSError:
        raise IoError(f"cannot write '{path}'") from None


def write_trace_csv(trace, path: str) -> None:
    """io.hpp:393-404: the same bytes as the reference (%.17g values)."""
    n = len(trace)
    it = np.array([t.iter for t in trace], np.int64)
    cols = [np.array([getattr(t, a) for t in trace], np.float64) for a in ("r_norm", "s_norm", "rho", "objective")]
    L = _lib.lib()
    rc = L.numpmp_write_trace_csv(os.fsencode(path), n, _lib.ptr(it), *[_lib.ptr(c) for c in cols])
    if rc:
        raise IoError(L.numpmp_host_last_error().decode())


def write_transit_metadata(meta: TransitMetadata, path: str) -> None:
    """io.hpp:444-467: the "NUMT 1" sidecar, the same bytes as the reference."""
    if meta.edges is None:
        raise ValidationError("transit metadata: no spatial graph (use gen_transit(..., with_meta=True))")
    e = np.ascontiguousarray(meta.edges, np.int32)
    ef, et = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
    arrs = dict(origin=np.ascontiguousarray(meta.od_origin, np.int32), dest=np.ascontiguousarray(meta.od_dest, np.int32),
                orp=np.ascontiguousarray(meta.od_route_ptr, np.int64), rp=np.ascontiguousarray(meta.route_ptr, np.int64),
                re=np.ascontiguousarray(meta.route_edges, np.int32), od=np.ascontiguousarray(meta.stream_od, np.int32),
                route=np.ascontiguousarray(meta.stream_route, np.int32), t0=np.ascontiguousarray(meta.stream_t0, np.int32))
    L = _lib.lib()
    rc = L.numpmp_write_transit_metadata(
        os.fsencode(path), meta.stations, meta.time_bins, meta.bin_minutes, meta.seats, meta.dropped_streams,
        len(ef), _lib.ptr(ef), _lib.ptr(et), len(arrs["origin"]), _lib.ptr(arrs["origin"]), _lib.ptr(arrs["dest"]),
        _lib.ptr(arrs["orp"]), _lib.ptr(arrs["rp"]), _lib.ptr(arrs["re"]), len(arrs["od"]), _lib.ptr(arrs["od"]),
        _lib.ptr(arrs["route"]), _lib.ptr(arrs["t0"]))
    if rc:
        raise IoError(L.numpmp_host_last_error().decode())


_INT = re.compile(r"^[+-]?[0-9]+$")


def read_transit_metadata(path: str) -> TransitMetadata:
    """io.hpp:469-540 with the reference's IoError messages."""
    try:
        f = open(path, "r", newline="\n")
    except OSError:
        raise IoError(f"cannot open '{path}'") from None
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    pos = [0]

    def toks():
        if pos[0] >= len(lines):
            raise IoError(f"parse error at line {pos[0] + 1}: unexpected end of '{path}'")
        pos[0] += 1
        return lines[pos[0] - 1].split()

    def pint(t, line):
        if not _INT.match(t):
            raise IoError(f"parse error at line {line}: expected an integer, got '{t}'")
        return int(t)

    def pdbl(t, line):
        try:
            if "_" in t:
                raise ValueError
            return float(t)
        except ValueError:
            raise IoError(f"parse error at line {line}: expected a number, got '{t}'") from None

    head = toks()
    if len(head) != 7 or head[0] != "NUMT":
        raise IoError("parse error at line 1: expected 'NUMT 1 <S> <T> <E> <ods> <streams>'")
    if pint(head[1], 1) != 1:
        raise IoError("parse error at line 1: unsupported metadata version")
    S, T, ne, nods, ns = (pint(h, 1) for h in head[2:7])
    extra = toks()
    if len(extra) != 3:
        raise IoError("parse error at line 2: expected '<bin_minutes> <seats> <dropped>'")
    bin_minutes, seats, dropped = pdbl(extra[0], 2), pdbl(extra[1], 2), pint(extra[2], 2)
    edges = np.empty((ne, 2), np.int32)
    for e in range(ne):
        t = toks()
        if len(t) != 2:
            raise IoError(f"parse error at line {pos[0]}: expected '<from> <to>'")
        edges[e] = (pint(t[0], pos[0]), pint(t[1], pos[0]))
    origin, dest = np.empty(nods, np.int32), np.empty(nods, np.int32)
    orp, rp, redges = [0], [0], []
    for q in range(nods):
        t = toks()
        if len(t) != 3:
            raise IoError(f"parse error at line {pos[0]}: expected '<origin> <dest> <routes>'")
        origin[q], dest[q] = pint(t[0], pos[0]), pint(t[1], pos[0])
        nr = pint(t[2], pos[0])
        for _ in range(nr):
            rt = toks()
            line = pos[0]
            if not rt:
                raise IoError(f"parse error at line {line}: expected a route")
            n = pint(rt[0], line)
            if len(rt) != 1 + n:
                raise IoError(f"parse error at line {line}: route length mismatch")
            redges.extend(pint(x, line) for x in rt[1:])
            rp.append(len(redges))
        orp.append(len(rp) - 1)
    trip = np.empty((ns, 3), np.int32)
    for j in range(ns):
        t = toks()
        if len(t) != 3:
            raise IoError(f"parse error at line {pos[0]}: expected '<od> <route> <t0>'")
        trip[j] = (pint(t[0], pos[0]), pint(t[1], pos[0]), pint(t[2], pos[0]))
    return TransitMetadata(S, T, bin_minutes, seats, origin, dest, np.ascontiguousarray(trip[:, 0]),
                           np.ascontiguousarray(trip[:, 1]), np.ascontiguousarray(trip[:, 2]), dropped, edges,
                           np.asarray(orp, np.int64), np.asarray(rp, np.int64), np.asarray(redges, np.int32))
