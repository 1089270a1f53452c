"""CPU tests of the C-ABI boundary: libnumpmp_cuda.so loads without a GPU,
exports every symbol include/*.h declares, and its host-side argument
checks return the reference's error classes before touching a device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2509_10722_b200 as pmp
from paper_2509_10722_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("numpmp_gpu.h", "numpmp_host.h")]


def declared_functions():
    names = set()
    for h in HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for mt in re.finditer(r"\b(numpmp_\w+)\s*\(", src):
            names.add(mt.group(1))
    return names


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 25
    L = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing


def test_binding_covers_the_headers():
    assert declared_functions() == set(_lib.SIGNATURES)


def test_library_not_linked_against_nccl():
    # NCCL is dlopen'ed lazily for sharded handles only (csrc/pmp_solver.cu)
    import subprocess

    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl" not in out


def _cfg(**kw):
    c = pmp.SolverConfig(**kw)
    return c._c()


def _single_view():
    p = pmp.problem_from_arrays(1, 1, [1.0], [1.0], [0], [0, 1], [0])
    return p, p.view()


@pytest.mark.parametrize("bad, msg", [
    (dict(eps_abs=0.0), "eps_abs must be > 0"),
    (dict(rho0=0.0), "rho0 must be > 0"),
    (dict(alpha=0.5), "alpha must be in [1, 2]"),
    (dict(mu=1.0), "mu must be > 1"),
    (dict(gamma=0.9), "gamma must be > 1"),
    (dict(rho_update_interval=0), "rho_update_interval must be >= 1"),
    (dict(max_iters=0), "max_iters must be >= 1"),
    (dict(trace_every=0), "trace_every must be >= 1"),
    (dict(threads=-1), "threads must be >= 0"),
    (dict(time_limit=-1.0), "time_limit must be >= 0"),
])
def test_config_errors_are_invalid_argument(bad, msg):
    # solver.hpp:32-44, same messages; checked before any device work
    L = _lib.lib()
    p, view = _single_view()
    h = C.c_void_p()
    rc = L.numpmp_gpu_create(C.byref(view), C.byref(_cfg(**bad)), 0, C.byref(h))
    assert rc == 1
    assert L.numpmp_gpu_last_error(None).decode() == msg
    assert not h.value


def test_malformed_view_is_rejected_on_host():
    L = _lib.lib()
    p = pmp.Problem(1, 1, [1.0], [1.0], [0], [0, 2], [0, 0])
    view = p.view()
    view.nnz = 1  # offsets say 2 terminals
    h = C.c_void_p()
    assert L.numpmp_gpu_create(C.byref(view), C.byref(_cfg()), 0, C.byref(h)) == 2
    assert "incidence-nnz" in L.numpmp_gpu_last_error(None).decode()


def test_null_handle_calls_fail_cleanly():
    L = _lib.lib()
    assert L.numpmp_gpu_set_cold(None) == 1
    assert L.numpmp_gpu_step(None, None, None) == 1
    assert L.numpmp_gpu_sizes(None, None, None, None) == 1
    L.numpmp_gpu_destroy(None)


def test_error_mapping_to_reference_exceptions():
    from paper_2509_10722_b200.errors import raise_for

    with pytest.raises(ValueError):
        raise_for(1, "x")
    with pytest.raises(pmp.ValidationError):
        raise_for(2, "x")
    with pytest.raises(pmp.SolverError):
        raise_for(3, "x")
    with pytest.raises(pmp.DomainError):
        raise_for(4, "x")
    with pytest.raises(pmp.DeviceError):
        raise_for(10, "x")


def test_free_functions():
    # solver.hpp:157-182 (test_solver.cpp:264-303)
    cfg = pmp.SolverConfig(eps_abs=1e-5)
    assert pmp.check_termination(9e-5, 9e-5, 100, cfg)
    assert not pmp.check_termination(1.1e-4, 9e-5, 100, cfg)
    assert not pmp.check_termination(9e-5, 1.1e-4, 100, cfg)
    assert pmp.check_termination(0.0, 0.0, 100, cfg)
    assert not pmp.check_termination(1e-4, 0.0, 100, cfg)
    st = pmp.SolverState(np.zeros(1), np.zeros(1), np.zeros(2), np.array([3.3, -0.7]), 1.0, 0)
    y = st.price.copy()
    c = pmp.SolverConfig()
    pmp.update_rho(st, 10.0, 1.0, c)
    assert st.rho == 1.1 and np.array_equal(st.price, y)
    pmp.update_rho(st, 1.0, 10.0, c)
    assert st.rho == 1.0
    pmp.update_rho(st, 1.0, 1.0, c)
    assert st.rho == 1.0
    st.price = np.array([-0.5, 2.0, 0.0])
    assert list(pmp.recover_duals(st)) == [0.0, 2.0, 0.0]
    p = pmp.problem_from_arrays(1, 1, [5.0], [2.0], [0], [0, 1], [0])
    assert abs(pmp.objective(p, np.array([np.e])) - 2.0) <= 1e-12
    with pytest.raises(pmp.DomainError):
        pmp.objective(p, np.array([0.0]))
