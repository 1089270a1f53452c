"""GPU tests of the drop-in API contract beyond the numerics: step() against
residuals() (solver.hpp:316-318, test_solver.cpp:245-262), the handle's state
round trip, step after a run, the TimeLimit status (solver.hpp:466-473) on one
device and on peer-memory ranks, the library's process-wide side effects, and
the reference's acceptance criteria 3, 5, 6 and 10 (proj/tests/acceptance.cpp)
restated on the device engine.
"""
import ctypes as C
import math
import time

import numpy as np
import pytest

pmp = pytest.importorskip("paper_2509_10722_b200")
from paper_2509_10722_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


def _mixed(m, n, avg, seed):
    return pmp.gen_uncongested(pmp.GenSpec(m=m, n=n, avg_links_per_stream=avg, kind=pmp.GenKind.Mixed,
                                           weights=pmp.WeightDist.uniform(0.5, 1.5), seed=seed))


def _host_residuals(p, st, prev):
    """residuals() of solver.hpp:139-154 in numpy (a different summation order)."""
    counts = np.bincount(p.route_links, minlength=p.m) + 1
    r = math.sqrt(float(np.sum(counts * st.p_bar * st.p_bar)))
    s = math.sqrt(float(np.sum((st.rho * (st.z - prev.z)) ** 2)))
    return r, s


# ------------------------------------------------------------- step / residuals
def test_step_residuals_match_device_residuals_bit_for_bit():
    # test_solver.cpp:245-262 (StepResidualsMatchFreeFunction) on the device:
    # step() returns exactly the library's residuals(after, before)
    p = pmp.gen_uncongested(pmp.GenSpec(m=40, n=20, avg_links_per_stream=4.0, kind=pmp.GenKind.Mixed, seed=9))
    with pmp.PmpSolver(p, pmp.SolverConfig()) as s:
        st = s.cold_state()
        for _ in range(20):
            prev = st.copy()
            r, sn = s.step(st)
            r_dev, s_dev = s.residuals(st, prev)
            assert (r, sn) == (r_dev, s_dev)
            r_host, s_host = _host_residuals(p, st, prev)
            assert abs(r - r_host) <= 1e-12 * max(1.0, r_host)
            assert abs(sn - s_host) <= 1e-12 * max(1.0, s_host)


def test_steps_continue_the_device_state_bit_for_bit():
    # a state the handle issued is kept on the device (no host
    # re-decomposition): K step() calls == a run of K iterations, bit for bit
    p = _mixed(300, 600, 5.0, 3)
    K = 20  # below the rho interval: step() and run() do the same iterations
    cfg = pmp.SolverConfig(eps_abs=1e-12, max_iters=K, rho0=10.0)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
        fin = s.final_state()
        st = s.cold_state()
        for _ in range(K):
            s.step(st)
    assert sol.iterations == K and st.iter == K
    np.testing.assert_array_equal(st.z, fin.z)
    np.testing.assert_array_equal(st.p, fin.p)
    np.testing.assert_array_equal(st.p_bar, fin.p_bar)
    np.testing.assert_array_equal(st.price, fin.price)
    x_steps = st.p[p.stream_offsets[:-1]]
    np.testing.assert_array_equal(x_steps, sol.x)


def test_modified_state_is_uploaded(restatement, oracle_mod):
    # a caller-modified state is not the one the handle issued: it is
    # uploaded and stepped from, matching the oracle's step from that state
    p = _mixed(50, 80, 3.0, 5)
    cfg = pmp.SolverConfig()
    with pmp.PmpSolver(p, cfg) as s:
        st = s.cold_state()
        s.step(st)
        mod = st.copy()
        mod.price = mod.price * 2.0 + 0.125
        r, sn = s.step(mod)
    a = oracle_mod.arrays_from(p)
    ost = dict(p=st.p.copy(), z=st.z.copy(), p_bar=st.p_bar.copy(), price=st.price * 2.0 + 0.125, rho=st.rho,
               iter=st.iter)
    ro, so, _ = restatement.step(a, oracle_mod.Config(), ost)
    assert mod.iter == ost["iter"] == 2
    assert abs(r - ro) <= 1e-9 * max(ro, 1.0) and abs(sn - so) <= 1e-9 * max(so, 1.0)
    for got, want in [(mod.z, ost["z"]), (mod.price, ost["price"]), (mod.p_bar, ost["p_bar"])]:
        assert np.max(np.abs(got - want)) <= 1e-9 * max(1.0, float(np.max(np.abs(want))))


def test_step_after_run_iterates():
    # numpmp_gpu_step right after numpmp_gpu_run used to exit at
    # entry (the run's `done` flag); it must run one iteration
    p = _mixed(200, 400, 4.0, 8)
    L = _lib.lib()
    with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-6)) as s:
        sol = s.solve()
        h = s.handle()
        r, sn = C.c_double(), C.c_double()
        assert L.numpmp_gpu_step(h, C.byref(r), C.byref(sn)) == 0
        st = s._download_state()[0]
        assert st.iter == sol.iterations + 1
        assert math.isfinite(r.value) and math.isfinite(sn.value)
        fin = s.final_state()  # the state after the extra step
        assert fin.iter == sol.iterations + 1


# ------------------------------------------------------------------ time limit
def _slow_problem():
    return pmp.gen_uncongested(pmp.GenSpec(m=20000, n=200000, avg_links_per_stream=10.0, seed=3))


def test_time_limit_status_single_device():
    # solver.hpp:466-473: TimeLimit is a status, checked after the trace push
    p = _slow_problem()
    limit = 0.05
    cfg = pmp.SolverConfig(eps_abs=1e-14, max_iters=10**7, time_limit=limit, trace_every=10)
    with pmp.PmpSolver(p, cfg) as s:
        t = time.perf_counter()
        sol = s.solve()
        wall = time.perf_counter() - t
    assert sol.status == pmp.SolveStatus.TimeLimit
    assert 0 < sol.iterations < cfg.max_iters
    assert wall >= limit
    assert wall < limit + 5.0
    assert sol.trace[-1].iter == sol.iterations


@pytest.mark.timeout(300)
def test_time_limit_is_collective_on_peer_memory_ranks():
    # every rank must stop at the same iteration (the
    # ranks' time-limit flags travel with the residual partials)
    from paper_2509_10722_b200.shard import p2p_local_group, run_ranks

    p = _slow_problem()
    cfg = pmp.SolverConfig(eps_abs=1e-14, max_iters=10**7, time_limit=0.05, trace_every=10)
    ranks = p2p_local_group(p, cfg, 2)
    try:
        sols = run_ranks([s.solve for s in ranks])
        again = run_ranks([s.solve for s in ranks])  # the exchange is still in step
    finally:
        for s in ranks:
            s.close()
    for out in (sols, again):
        assert all(s.status == pmp.SolveStatus.TimeLimit for s in out)
        assert out[0].iterations == out[1].iterations > 0
        np.testing.assert_array_equal(out[0].lambda_raw, out[1].lambda_raw)


# ----------------------------------------------------------- side effects
def _cudart():
    import glob
    import os

    import torch

    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    for c in cands:
        try:
            return C.CDLL(c)
        except OSError:
            continue
    pytest.skip("libcudart not found")


def test_library_leaves_process_state_alone():
    # the persisting-L2 limit is restored when the last
    # handle is destroyed, and the device's default memory pool keeps its
    # release threshold (the library allocates from its own pool)
    rt = _cudart()
    assert rt.cudaSetDevice(0) == 0
    lim = C.c_size_t()
    assert rt.cudaDeviceSetLimit(C.c_int(6), C.c_size_t(0)) == 0  # cudaLimitPersistingL2CacheSize
    pool = C.c_void_p()
    assert rt.cudaDeviceGetDefaultMemPool(C.byref(pool), 0) == 0
    thr0 = C.c_uint64()
    assert rt.cudaMemPoolGetAttribute(pool, C.c_int(4), C.byref(thr0)) == 0  # ReleaseThreshold
    p = _mixed(300, 600, 5.0, 3)
    a = pmp.PmpSolver(p, pmp.SolverConfig())
    b = pmp.PmpSolver(p, pmp.SolverConfig())
    assert rt.cudaDeviceGetLimit(C.byref(lim), C.c_int(6)) == 0
    assert lim.value > 0  # raised while handles live
    a.solve()
    a.close()
    assert rt.cudaDeviceGetLimit(C.byref(lim), C.c_int(6)) == 0
    assert lim.value > 0  # b still lives
    b.solve()
    b.close()
    assert rt.cudaDeviceGetLimit(C.byref(lim), C.c_int(6)) == 0
    assert lim.value == 0
    thr1 = C.c_uint64()
    assert rt.cudaMemPoolGetAttribute(pool, C.c_int(4), C.byref(thr1)) == 0
    assert thr1.value == thr0.value


# ------------------------------------------- acceptance criteria (acceptance.cpp)
def test_acceptance_2_small_instances_match_reference(reference, oracle_mod):
    # acceptance.cpp:105-150 restated: the same 50 mixed instances (m in
    # [10, 200], seeds 51000 + k) solved to 1e-6.  The reference checks its
    # objective within 1e-3 of an Eigen barrier oracle (absent here, SURVEY
    # 8(c)); the device engine is held to the reference's own PMP solve
    # instead: equal status and iteration count, objective and every log
    # allocation within 1e-6 relative, and the whole sweep under 2 minutes.
    import time

    t0 = time.perf_counter()
    worst_obj = worst_x = 0.0
    for k in range(50):
        m = 10 + (190 * k) // 49
        n = max(1, m // 2)
        p = pmp.gen_uncongested(pmp.GenSpec(m=m, n=n, avg_links_per_stream=4.0, kind=pmp.GenKind.Mixed,
                                            weights=pmp.WeightDist.uniform(0.5, 1.5), seed=51000 + k))
        with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-6)) as s:
            sol = s.solve()
        ref = reference.gen(m, n, 4.0, 2, ("uniform", 0.5, 1.5), 51000 + k).solve(oracle_mod.Config(eps_abs=1e-6))
        assert ref.error is None and ref.status == 0
        assert int(sol.status) == ref.status and sol.iterations == ref.iterations, (k, sol.iterations, ref.iterations)
        worst_obj = max(worst_obj, abs(sol.objective - ref.objective) / abs(ref.objective))
        lg = p.kinds == int(pmp.StreamKind.Log)
        if lg.any():
            worst_x = max(worst_x, float(np.max(np.abs(sol.x[lg] - ref.x[lg]) / np.abs(ref.x[lg]))))
    elapsed = time.perf_counter() - t0
    assert worst_obj <= 1e-6 and worst_x <= 1e-6, (worst_obj, worst_x)
    assert elapsed < 120.0, elapsed


def test_acceptance_8_rho_balancing_on_the_device():
    # acceptance.cpp:365-396 / update_rho (solver.hpp:168-174) as the device
    # finalize runs it: every rho_update_interval iterations, rho * gamma if
    # r > mu s, rho / gamma if s > mu r, unchanged otherwise -- each decision
    # checked against the (r, s) the trace reports for that iteration, all
    # three branches taken.  The unscaled price is what the device stores, so
    # a rescale cannot change it: v = B + price / rho is rebuilt instead.
    p = pmp.gen_uncongested(pmp.GenSpec(m=2000, n=4000, avg_links_per_stream=6.0, kind=pmp.GenKind.Mixed,
                                        weights=pmp.WeightDist.uniform(0.5, 1.5), seed=11))
    cfg = pmp.SolverConfig(eps_abs=1e-7, rho0=1000.0, rho_update_interval=10, trace_every=1, max_iters=4000)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    rows = {t.iter: t for t in sol.trace}
    seen = set()
    for k in sorted(rows):
        if k % cfg.rho_update_interval or k + 1 not in rows:
            continue
        t, nxt = rows[k], rows[k + 1]
        if t.r_norm > cfg.mu * t.s_norm:
            want, branch = t.rho * cfg.gamma, "up"
        elif t.s_norm > cfg.mu * t.r_norm:
            want, branch = t.rho / cfg.gamma, "down"
        else:
            want, branch = t.rho, "keep"
        assert nxt.rho == want, (k, branch, t.rho, nxt.rho)
        seen.add(branch)
        assert all(rows[j].rho == t.rho for j in range(k - cfg.rho_update_interval + 1, k + 1) if j in rows)
    assert seen == {"up", "down", "keep"}, seen


def test_acceptance_3_kkt_stationarity():
    # acceptance.cpp:158-180 over the 50 instances of criterion 2 (:105-150):
    # w_j / x_j = pi_j within 1e-2 relative for every log stream
    worst = 0.0
    for k in range(50):
        m = 10 + (190 * k) // 49
        p = pmp.gen_uncongested(pmp.GenSpec(m=m, n=max(1, m // 2), avg_links_per_stream=4.0,
                                            kind=pmp.GenKind.Mixed, weights=pmp.WeightDist.uniform(0.5, 1.5),
                                            seed=51000 + k))
        with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-6)) as s:
            sol = s.solve()
            assert sol.status == pmp.SolveStatus.Converged
            pi = s.path_prices(sol.lambda_)
        lg = p.kinds == int(pmp.StreamKind.Log)
        ratio = np.abs(p.weights[lg] / sol.x[lg] - pi[lg]) / pi[lg]
        if ratio.size:
            worst = max(worst, float(np.max(ratio)))
    assert worst <= 1e-2, worst


def test_acceptance_5_desk_scale(reference):
    # acceptance.cpp:212-245: m = 1e5 uncongested converges within 3000
    # iterations at eps 1e-4, rho0 = 1000; the congested variant within 2x
    # that count.  Iteration counts equal the reference's own.
    spec = pmp.GenSpec(m=100000, n=50000, avg_links_per_stream=10.0, seed=7)
    cfg = pmp.SolverConfig(eps_abs=1e-4, max_iters=3000, rho0=1000.0)
    u = pmp.gen_uncongested(spec)
    with pmp.PmpSolver(u, cfg) as s:
        us = s.solve()
    assert us.status == pmp.SolveStatus.Converged
    ccfg = pmp.SolverConfig(eps_abs=1e-4, max_iters=2 * us.iterations, rho0=1000.0)
    c = pmp.gen_congested(spec)
    with pmp.PmpSolver(c, ccfg) as s:
        cs = s.solve()
    assert cs.status == pmp.SolveStatus.Converged
    from oracle import oracle as o

    ru = reference.gen(100000, 50000, 10.0, 0, ("constant", 1.0, 1.0), 7).solve(
        o.Config(eps_abs=1e-4, max_iters=3000, rho0=1000.0, threads=0))
    assert ru.iterations == us.iterations
    rc = reference.gen(100000, 50000, 10.0, 0, ("constant", 1.0, 1.0), 7, congested=True).solve(
        o.Config(eps_abs=1e-4, max_iters=2 * us.iterations, rho0=1000.0, threads=0))
    assert rc.iterations == cs.iterations


def test_acceptance_6_warm_start_halves_iterations():
    # acceptance.cpp:247-304 with the device recipes (warm.hpp:25-94)
    cfg = pmp.SolverConfig(eps_abs=1e-5)
    spec = pmp.GenSpec(m=10000, n=5000, avg_links_per_stream=10.0, seed=101)
    base = pmp.gen_uncongested(spec)
    with pmp.PmpSolver(base, cfg) as s:
        sol0 = s.solve()
    assert sol0.status == pmp.SolveStatus.Converged
    deg = pmp.degrade(base, 0.25, 0.5, 102)
    with pmp.PmpSolver(deg, cfg) as s:
        cold = s.solve()
        s.warm_start_after_degrade(base, sol0)
        warm = s.solve_prepared()
    assert cold.status == warm.status == pmp.SolveStatus.Converged
    assert 2 * warm.iterations <= cold.iterations, (warm.iterations, cold.iterations)

    pbase = pmp.gen_uncongested(pmp.GenSpec(m=10000, n=5000, avg_links_per_stream=10.0, seed=202))
    with pmp.PmpSolver(pbase, cfg) as s:
        psol0 = s.solve()
    assert psol0.status == pmp.SolveStatus.Converged
    pruned, pmap = pmp.fail_and_prune(pbase, 0.25, 204)
    with pmp.PmpSolver(pruned, cfg) as s:
        pcold = s.solve()
        s.warm_start_after_prune(pmap, psol0)
        pwarm = s.solve_prepared()
    assert pcold.status == pwarm.status == pmp.SolveStatus.Converged
    assert 2 * pwarm.iterations <= pcold.iterations, (pwarm.iterations, pcold.iterations)


def test_acceptance_10_transit_pipeline():
    # acceptance.cpp:449-502: S=20, T=48 transit instance solved to 1e-6; the
    # route report shows x = w/pi within 2% for every (OD, departure) group
    # with more than one route, lambda_hat in [0, 1]
    spec = pmp.TransitSpec(stations=20, time_bins=48, bin_minutes=5.0, spatial_edges=190, od_pairs=30,
                           routes_per_od=3, departures_per_route=5, seed=100)
    p, meta = pmp.gen_transit(spec, with_meta=True)
    assert p.m == 190 * 48
    with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-6)) as s:
        sol = s.solve()
        assert sol.status == pmp.SolveStatus.Converged
        pi = s.path_prices(sol.lambda_)
    worst, pairs, seen = 0.0, 0, set()
    for od, t0 in zip(meta.stream_od.tolist(), meta.stream_t0.tolist()):
        if (od, t0) in seen:
            continue
        seen.add((od, t0))
        rows = pmp.transit_report(p, sol.x, sol.lambda_, meta, od, t0, pi=pi)
        if len(rows) < 2:
            continue
        pairs += 1
        for row in rows:
            assert row.pi > 0.0
            worst = max(worst, abs(row.x * row.pi - 1.0))
            assert all(0.0 <= h <= 1.0 for h in row.lambda_hat)
    assert pairs > 0
    assert worst <= 0.02, worst
