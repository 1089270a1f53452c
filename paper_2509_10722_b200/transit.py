"""Reports around a solution: the transit route report
(transit.hpp:304-374) and the trace CSV (io.hpp:393-404).

The per-stream path prices come from the device (PmpSolver.path_prices,
transit.hpp:290-302) when a solver is passed; the report itself only touches
the few streams of one (OD, departure) and is assembled on the host, as in
the reference.
"""
from __future__ import annotations

import os
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
    if len(meta.stream_od) != problem.n:
        raise ValidationError("transit report: metadata does not match problem")
    k = len(meta.od_origin)
    if od < 0 or od >= k:
        raise ValidationError(f"unknown OD id {od}; available: 0..{k - 1}")
    selected = np.flatnonzero((meta.stream_od == od) & (meta.stream_t0 == t0)).tolist()
    lam = np.asarray(lam, np.float64)
    if lam.shape[0] != problem.m:
        raise ValidationError("path_prices: lambda length mismatch")
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
