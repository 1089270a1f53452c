"""ctypes binding of libnumpmp_cuda.so (include/numpmp_gpu.h, include/numpmp_host.h).

The library is built in-tree by ``paper_2509_10722_b200.build`` (called from
``__graft_entry__.build()``).  There is deliberately no fallback: if the
shared object is missing, importing the solver fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# NUMPMP_LIB selects an alternative in-tree build (tuning sweeps, scripts/variants.sh)
LIB_PATH = os.environ.get("NUMPMP_LIB") or os.path.join(_HERE, "lib", "libnumpmp_cuda.so")


class ProblemView(C.Structure):
    _fields_ = [
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("nnz", C.c_int64),
        ("capacities", C.c_void_p),
        ("weights", C.c_void_p),
        ("kinds", C.c_void_p),
        ("stream_offsets", C.c_void_p),
        ("route_links", C.c_void_p),
    ]


class Config(C.Structure):
    _fields_ = [
        ("eps_abs", C.c_double),
        ("rho0", C.c_double),
        ("alpha", C.c_double),
        ("mu", C.c_double),
        ("gamma", C.c_double),
        ("time_limit", C.c_double),
        ("rho_update_interval", C.c_int64),
        ("max_iters", C.c_int64),
        ("trace_every", C.c_int64),
        ("threads", C.c_int32),
        ("_pad", C.c_int32),
    ]


class TraceRow(C.Structure):
    _fields_ = [
        ("iter", C.c_int64),
        ("r_norm", C.c_double),
        ("s_norm", C.c_double),
        ("rho", C.c_double),
        ("objective", C.c_double),
    ]


class SolutionInfo(C.Structure):
    _fields_ = [
        ("objective", C.c_double),
        ("r_norm", C.c_double),
        ("s_norm", C.c_double),
        ("rho_final", C.c_double),
        ("iterations", C.c_int64),
        ("status", C.c_int32),
        ("_pad", C.c_int32),
        ("trace_len", C.c_int64),
    ]


class GenSpecC(C.Structure):
    _fields_ = [
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("avg_links_per_stream", C.c_double),
        ("kind", C.c_int32),
        ("weight_kind", C.c_int32),
        ("weight_a", C.c_double),
        ("weight_b", C.c_double),
        ("seed", C.c_uint64),
    ]


class TransitSpecC(C.Structure):
    _fields_ = [
        ("stations", C.c_int32),
        ("time_bins", C.c_int32),
        ("bin_minutes", C.c_double),
        ("spatial_edges", C.c_int64),
        ("od_pairs", C.c_int64),
        ("routes_per_od", C.c_int32),
        ("departures_per_route", C.c_int32),
        ("seats", C.c_double),
        ("seed", C.c_uint64),
    ]


P = C.c_void_p
I64 = C.c_int64
D = C.c_double
PI64 = C.POINTER(C.c_int64)
PD = C.POINTER(C.c_double)

# (name, restype, argtypes) for every symbol the two headers declare.
SIGNATURES = {
    # numpmp_gpu.h
    "numpmp_gpu_create": (C.c_int, [C.POINTER(ProblemView), C.POINTER(Config), C.c_int, C.POINTER(P)]),
    "numpmp_gpu_create_sharded": (
        C.c_int,
        [C.POINTER(ProblemView), C.POINTER(Config), C.c_int, C.c_int, C.c_int, P, I64, I64, C.POINTER(P)],
    ),
    "numpmp_gpu_nccl_unique_id": (C.c_int, [P]),
    "numpmp_gpu_create_p2p": (
        C.c_int,
        [C.POINTER(ProblemView), C.POINTER(Config), C.c_int, C.c_int, C.c_int, I64, I64, C.POINTER(P)],
    ),
    "numpmp_gpu_p2p_export": (C.c_int, [P, P]),
    "numpmp_gpu_p2p_connect": (C.c_int, [P, P]),
    "numpmp_gpu_p2p_connect_local": (C.c_int, [C.POINTER(P), C.c_int]),
    "numpmp_gpu_p2p_start": (C.c_int, [P]),
    "numpmp_gpu_warm_after_degrade": (C.c_int, [P, P, P, P, D, P, P, PD]),
    "numpmp_gpu_warm_after_prune": (C.c_int, [P, P, P, D, P, P, PD]),
    "numpmp_gpu_path_prices": (C.c_int, [P, P, P]),
    "numpmp_gpu_set_cold": (C.c_int, [P]),
    "numpmp_gpu_set_warm": (C.c_int, [P, P, P, D]),
    "numpmp_gpu_set_state": (C.c_int, [P, P, P, P, P, D, I64]),
    "numpmp_gpu_get_state": (C.c_int, [P, P, P, P, P, PD, PI64, P]),
    "numpmp_gpu_step": (C.c_int, [P, PD, PD]),
    "numpmp_gpu_residuals": (C.c_int, [P, P, P, P, D, PD, PD]),
    "numpmp_gpu_run": (C.c_int, [P, P, P, P, P, C.POINTER(SolutionInfo), P, I64]),
    "numpmp_gpu_run_device": (C.c_int, [P, C.POINTER(SolutionInfo)]),
    "numpmp_gpu_export_layout": (C.c_int, [P, P, P, P]),
    "numpmp_gpu_sizes": (C.c_int, [P, PI64, PI64, PI64]),
    "numpmp_gpu_set_profiling": (C.c_int, [P, C.c_int]),
    "numpmp_gpu_profile": (C.c_int, [P, PI64, PD, PD, PI64]),
    "numpmp_gpu_transfer_bytes": (C.c_int, [P, PI64, PI64]),
    "numpmp_gpu_last_error": (C.c_char_p, [P]),
    "numpmp_gpu_destroy": (None, [P]),
    # numpmp_host.h
    "numpmp_gen_uncongested": (C.c_int, [C.POINTER(GenSpecC), C.POINTER(P)]),
    "numpmp_gen_congested": (C.c_int, [C.POINTER(GenSpecC), D, D, C.POINTER(P)]),
    "numpmp_instance_sizes": (None, [P, PI64, PI64, PI64]),
    "numpmp_instance_export": (None, [P, P, P, P, P, P]),
    "numpmp_instance_free": (None, [P]),
    "numpmp_gen_transit": (C.c_int, [C.POINTER(TransitSpecC), C.POINTER(P), PI64]),
    "numpmp_degrade": (C.c_int, [I64, P, D, D, C.c_uint64]),
    "numpmp_fail_and_prune": (C.c_int, [I64, I64, P, P, P, P, P, D, C.c_uint64, C.POINTER(P), P, P]),
    "numpmp_read_problem": (C.c_int, [C.c_char_p, C.POINTER(P)]),
    "numpmp_transit_meta": (C.c_int, [P, PI64, P, P, P, P, P]),
    "numpmp_transit_graph": (C.c_int, [P, PI64, PI64, PI64, P, P, P, P, P]),
    "numpmp_write_transit_metadata": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, D, D, I64, I64, P, P, I64, P, P,
                                                P, P, P, I64, P, P, P]),
    "numpmp_write_trace_csv": (C.c_int, [C.c_char_p, I64, P, P, P, P, P]),
    "numpmp_write_problem": (C.c_int, [I64, I64, P, P, P, P, P, C.c_char_p, C.c_int]),
    "numpmp_validate": (I64, [I64, I64, P, P, P, P, P, C.c_char_p, I64]),
    "numpmp_build_layout": (C.c_int, [I64, I64, P, P, P, P, P, P]),
    "numpmp_host_last_error": (C.c_char_p, []),
}

_lib = None


def lib():
    """Load the in-tree shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("NUMPMP_LIB") and not hasattr(L, name):
                continue  # an older variant build (A/B against earlier rounds) lacks later entry points
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a):
    """Data pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


SIGNATURES.update({
    "numpmp_gpu_last_run_ms": (C.c_int, [P, PD]),
    "numpmp_gpu_pin_host": (C.c_int, [P, I64]),
    "numpmp_gpu_unpin_host": (C.c_int, [P]),
})
