"""GPU parity tests: the sm_100a engine (through the C-ABI, via the Python
mirror of the reference API) against the CPU oracle and the reference's own
golden vectors.

Tolerance (fp64): 1e-6 relative, measured in the max norm of each compared
vector (|a - b|_inf <= 1e-6 * max(|b|_inf, floor)); iteration counts must
be equal; the layout must be bit-exact.  The golden values of
proj/tests/test_solver.cpp are asserted at the tolerances that file uses.
"""
import math

import numpy as np
import pytest

pmp = pytest.importorskip("paper_2509_10722_b200")

pytestmark = pytest.mark.gpu

RTOL = 1e-6


def close(a, b, rtol=RTOL, floor=1e-12):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, floor)
    err = float(np.max(np.abs(a - b))) if b.size else 0.0
    return err <= rtol * scale, err / scale


def bipartite_fixture():
    # test_solver.cpp:15-20
    S = pmp.Stream
    return pmp.build_problem([S(0, pmp.StreamKind.Log, "", 1.0, [0]),
                              S(1, pmp.StreamKind.Log, "", 1.0, [1, 2]),
                              S(2, pmp.StreamKind.Log, "", 1.0, [1])], [1.0, 1.0, 1.0])


def single(kind=pmp.StreamKind.Log, w=1.0, route=(0,), caps=(1.0,)):
    return pmp.build_problem([pmp.Stream(0, kind, "", w, list(route))], list(caps))


def plain_config(rho0):
    return pmp.SolverConfig(alpha=1.0, rho0=rho0, rho_update_interval=1000000)


def ocfg(o, c: "pmp.SolverConfig"):
    return o.Config(eps_abs=c.eps_abs, rho0=c.rho0, alpha=c.alpha, mu=c.mu, gamma=c.gamma,
                    time_limit=c.time_limit, rho_update_interval=c.rho_update_interval,
                    max_iters=c.max_iters, trace_every=c.trace_every)


# ---------------------------------------------------- golden vectors (reference tests)
def test_first_iteration_from_zero_state():
    # test_solver.cpp:110-124
    p = single()
    with pmp.PmpSolver(p, plain_config(1.0)) as s:
        st = s.cold_state()
        s.step(st)
    assert st.iter == 1
    np.testing.assert_allclose(st.p, [1.0, 0.0], rtol=0, atol=4e-16)
    np.testing.assert_allclose(st.p_bar, [0.5], rtol=0, atol=4e-16)
    np.testing.assert_allclose(st.z, [0.5, -0.5], rtol=0, atol=4e-16)
    np.testing.assert_allclose(st.price, [0.5], rtol=0, atol=4e-16)


@pytest.mark.parametrize("rho0", [1.0, 2.0])
def test_alpha1_matches_plain_transcription(rho0, restatement, oracle_mod):
    # test_solver.cpp:126-146 / acceptance.cpp criterion 7
    p = bipartite_fixture()
    a = oracle_mod.arrays_from(p)
    J = a.J
    pp, uu, pbar, arg = np.zeros(J), np.zeros(J), np.zeros(p.m), np.zeros(J)
    pr, keep = restatement._prob(a)
    with pmp.PmpSolver(p, plain_config(rho0)) as s:
        st = s.cold_state()
        for it in range(100):
            s.step(st)
            restatement.L.oracle_plain_step(
                __import__("ctypes").byref(pr), __import__("ctypes").c_double(rho0),
                *[oracle_mod._p(v) for v in (pp, uu, pbar, arg)])
            ok, err = close(st.p, pp, 1e-12)
            assert ok, (it, err)
            price_ref = rho0 * uu[: J]
            ok, err = close(st.price[a.terminal_link], price_ref, 1e-12)
            assert ok, (it, err)


@pytest.mark.parametrize("alpha", [1.0, 1.6])
def test_fixed_point_is_stationary(alpha):
    # test_solver.cpp:148-171
    p = single()
    cfg = pmp.SolverConfig(alpha=alpha, rho_update_interval=1000000)
    with pmp.PmpSolver(p, cfg) as s:
        st = s.cold_state()
        st.p = np.array([1.0, -1.0])
        st.z = np.array([1.0, -1.0])
        st.p_bar = np.array([0.0])
        st.price = np.array([1.0])
        r, sn = s.step(st)
    np.testing.assert_allclose(st.p, [1.0, -1.0], atol=1e-14)
    np.testing.assert_allclose(st.z, [1.0, -1.0], atol=1e-14)
    np.testing.assert_allclose(st.price, [1.0], atol=1e-14)
    assert abs(r) <= 1e-14 and abs(sn) <= 1e-14


def test_single_log_stream_analytic():
    # test_solver.cpp:75-84
    with pmp.PmpSolver(single(), pmp.SolverConfig(eps_abs=1e-8)) as s:
        sol = s.solve()
    assert sol.status == pmp.SolveStatus.Converged
    assert abs(sol.x[0] - 1.0) <= 1e-6
    assert abs(sol.lambda_[0] - 1.0) <= 1e-6


def test_single_linear_stream_saturates():
    # test_solver.cpp:86-96
    with pmp.PmpSolver(single(pmp.StreamKind.Linear, caps=(5.0,)), pmp.SolverConfig(eps_abs=1e-8)) as s:
        sol = s.solve()
    assert sol.status == pmp.SolveStatus.Converged
    assert abs(sol.x[0] - 5.0) <= 1e-5
    assert abs(sol.objective - 5.0) <= 1e-5


def test_bipartite_fixture_solution():
    # test_solver.cpp:98-108 + test_oracle.cpp:63-76: x = (1, .5, .5), lambda = (1, 2, 0)
    with pmp.PmpSolver(bipartite_fixture(), pmp.SolverConfig(eps_abs=1e-7)) as s:
        sol = s.solve()
    assert sol.status == pmp.SolveStatus.Converged
    for got, want in zip(sol.x, [1.0, 0.5, 0.5]):
        assert abs(got - want) <= 1e-4 * want
    np.testing.assert_allclose(sol.lambda_, [1.0, 2.0, 0.0], atol=1e-3)


def test_non_binding_link_dual_vanishes():
    # test_solver.cpp:370-382
    p = single(route=(0, 1), caps=(1.0, 5.0))
    with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-8)) as s:
        sol = s.solve()
    assert sol.status == pmp.SolveStatus.Converged
    assert abs(sol.x[0] - 1.0) <= 1e-5
    assert abs(sol.lambda_[0] - 1.0) <= 1e-3
    assert abs(sol.lambda_[1]) <= 1e-3


def test_max_iters_status_is_returned_not_thrown():
    # test_solver.cpp:384-393
    with pmp.PmpSolver(bipartite_fixture(), pmp.SolverConfig(max_iters=3, eps_abs=1e-12)) as s:
        sol = s.solve()
    assert sol.status == pmp.SolveStatus.MaxIters
    assert sol.iterations == 3


def test_non_finite_state_reports_iteration_number():
    # test_solver.cpp:173-186
    p = single(w=1e308)
    with pmp.PmpSolver(p, pmp.SolverConfig(rho0=1e-8)) as s:
        with pytest.raises(pmp.SolverError, match="iteration 1"):
            s.solve()


def test_trace_contract():
    # test_solver.cpp:395-415
    p = pmp.gen_uncongested(pmp.GenSpec(m=60, n=30, seed=4))
    with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-6, trace_every=10)) as s:
        sol = s.solve()
    assert sol.trace
    its = [t.iter for t in sol.trace]
    assert all(a < b for a, b in zip(its, its[1:]))
    assert sol.trace[-1].iter == sol.iterations
    assert sol.trace[-1].r_norm == sol.r_norm and sol.trace[-1].s_norm == sol.s_norm
    assert all(t.iter % 10 == 0 for t in sol.trace[:-1])


def test_warm_start_from_optimum_converges_immediately():
    # test_solver.cpp:322-339
    p = pmp.gen_uncongested(pmp.GenSpec(m=80, n=40, avg_links_per_stream=4.0, seed=21))
    with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-7)) as s:
        cold = s.solve()
        assert cold.status == pmp.SolveStatus.Converged
        rerun = s.solve(pmp.WarmStart(cold.x, cold.lambda_raw, cold.rho_final))
    assert rerun.status == pmp.SolveStatus.Converged
    assert rerun.iterations <= 5


def test_warm_start_validation():
    # test_solver.cpp:341-350
    with pmp.PmpSolver(bipartite_fixture(), pmp.SolverConfig()) as s:
        with pytest.raises(ValueError):
            s.warm_state(pmp.WarmStart(np.array([1.0, 1.0])))
        with pytest.raises(pmp.DomainError):
            s.warm_state(pmp.WarmStart(np.array([1.0, 0.0, 1.0])))
        with pytest.raises(ValueError):
            s.warm_state(pmp.WarmStart(np.array([1.0, 1.0, 1.0]), np.array([0.1])))


def test_warm_start_slack_flows():
    # test_solver.cpp:352-368
    p = bipartite_fixture()
    with pmp.PmpSolver(p, pmp.SolverConfig()) as s:
        st = s.warm_state(pmp.WarmStart(np.array([0.25, 0.5, 0.75]), None, 1.0))
    nnz = p.nnz
    np.testing.assert_array_equal(st.p[nnz:], [-0.25, -1.0, -0.5])
    tl = p.layout.terminal_link
    np.testing.assert_array_equal(st.z, st.p - st.p_bar[tl])


# ------------------------------------------------------------ oracle parity
def _gen(m, n, avg, kind, uniform, seed):
    w = pmp.WeightDist.uniform(0.5, 1.5) if uniform else pmp.WeightDist.constant(1.0)
    return pmp.gen_uncongested(pmp.GenSpec(m=m, n=n, avg_links_per_stream=avg, kind=pmp.GenKind(kind),
                                           weights=w, seed=seed))


SOLVE_CASES = [
    # (m, n, avg, kind, uniform weights, seed, eps, rho0)
    (1000, 10000, 5.0, 0, False, 7, 1e-4, 1.0),      # config A, library default rho0
    (1000, 10000, 5.0, 0, False, 7, 1e-4, 1000.0),   # config A, large-instance rho0
    (300, 150, 4.0, 2, True, 3, 1e-6, 1.0),          # mixed log/linear
    (2000, 4000, 6.0, 2, True, 11, 1e-5, 1000.0),    # mixed, rho balancing active
    (100, 50, 5.0, 2, True, 1, 1e-6, 1.0),           # ConvergedRunsAreFeasible instance
]


@pytest.mark.parametrize("case", SOLVE_CASES)
def test_solve_matches_oracle(case, restatement, oracle_mod):
    m, n, avg, kind, uni, seed, eps, rho0 = case
    p = _gen(m, n, avg, kind, uni, seed)
    cfg = pmp.SolverConfig(eps_abs=eps, rho0=rho0)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
        fin = s.final_state()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert ref.error is None
    assert sol.iterations == ref.iterations
    assert int(sol.status) == ref.status
    assert sol.rho_final == ref.rho_final
    for name, got, want in [("x", sol.x, ref.x), ("lambda_raw", sol.lambda_raw, ref.lambda_raw),
                            ("s", sol.s, ref.s), ("lambda", sol.lambda_, ref.lambda_)]:
        ok, err = close(got, want)
        assert ok, (name, err)
    assert abs(sol.objective - ref.objective) <= RTOL * abs(ref.objective)
    assert len(sol.trace) == ref.trace.shape[0]
    for row, want in zip(sol.trace, ref.trace):
        assert row.iter == int(want[0]) and row.rho == want[3]
        for got, w in [(row.r_norm, want[1]), (row.s_norm, want[2]), (row.objective, want[4])]:
            assert abs(got - w) <= RTOL * abs(w) + 1e-300, (row.iter, got, w)
    ok, err = close(fin.z, ref.final_z)
    assert ok, err
    ok, err = close(fin.p, ref.final_p)
    assert ok, err


@pytest.mark.parametrize("blocks", [2, 3, 7])
def test_column_blocks_match_oracle(blocks, restatement, oracle_mod, monkeypatch):
    # the column-blocked pipeline (stream pass / link gather per block) is
    # the same iteration: equal iteration counts, x and prices within 1e-6
    monkeypatch.setenv("NUMPMP_COL_BLOCKS", str(blocks))
    p = _gen(2000, 4000, 6.0, 2, True, 11)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
        st = s.final_state()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert sol.iterations == ref.iterations
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw), (st.p_bar, ref.final_pbar)]:
        ok, err = close(got, want)
        assert ok, err


@pytest.mark.parametrize("blocks", [1, 3])
def test_sharded_path_one_rank_matches_oracle(blocks, restatement, oracle_mod, monkeypatch):
    # The multi-GPU code path (local gather -> NCCL all-reduce of the partial
    # loads + scalars -> replicated epilogue) on a one-rank communicator.
    pytest.importorskip("torch")  # load PyTorch's NCCL first (shared with the engine)
    from paper_2509_10722_b200.shard import ShardedPmpSolver, nccl_unique_id

    monkeypatch.setenv("NUMPMP_COL_BLOCKS", str(blocks))
    p = _gen(2000, 4000, 6.0, 2, True, 11)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    s = ShardedPmpSolver(p, cfg, 0, 1, nccl_unique_id())
    try:
        sol = s.solve()
    finally:
        s.close()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert sol.iterations == ref.iterations
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw), (sol.s, ref.s)]:
        ok, err = close(got, want)
        assert ok, err
    assert abs(sol.objective - ref.objective) <= RTOL * abs(ref.objective)


@pytest.mark.parametrize("world,blocks", [(1, 1), (2, 1), (3, 2), (4, 1)])
def test_p2p_exchange_ranks_match_oracle(world, blocks, restatement, oracle_mod, monkeypatch):
    # The fused peer-memory exchange (csrc/pmp_p2p.cuh) with `world` ranks in
    # this process on one GPU, each driven by its own host thread exactly as
    # one process per GPU would drive it: link-pass stores into the owners'
    # slots, system-scope barriers, owner epilogue + v broadcast, rank-order
    # sums.  The assembled solution must match the single-problem oracle at
    # equal iteration counts (mixed utilities, several rho changes).
    from paper_2509_10722_b200.shard import link_owners, p2p_local_group, run_ranks

    monkeypatch.setenv("NUMPMP_COL_BLOCKS", str(blocks))
    p = _gen(2000, 4000, 6.0, 2, True, 11)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    ranks = p2p_local_group(p, cfg, world)
    try:
        sols = run_ranks([s.solve for s in ranks])
    finally:
        for s in ranks:
            s.close()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    x = np.concatenate([s.x for s in sols])
    for s in sols:
        assert s.iterations == ref.iterations
        # every rank holds the same gathered link vectors and scalars
        np.testing.assert_array_equal(s.lambda_raw, sols[0].lambda_raw)
        assert s.r_norm == sols[0].r_norm and s.s_norm == sols[0].s_norm
    for got, want in [(x, ref.x), (sols[0].lambda_raw, ref.lambda_raw), (sols[0].s, ref.s)]:
        ok, err = close(got, want)
        assert ok, err
    assert abs(sols[0].objective - ref.objective) <= RTOL * abs(ref.objective)
    assert [r.iter for r in sols[0].trace] == [int(i) for i in ref.trace[:, 0]]
    assert link_owners(p.m, world)[-1] == p.m


@pytest.mark.parametrize("world", [1, 2, 3])
def test_p2p_fused_epilogue_matches_oracle(world, restatement, oracle_mod, monkeypatch):
    # Fused mode (one GPU per rank in production: the "loads stored" wait in
    # every owner-epilogue CTA, the finalize in its last CTA, 2 NB + 1
    # launches per iteration).  Forced here with ranks sharing one GPU; the
    # grids of this small instance leave SMs free for every rank's kernels.
    import ctypes as C

    from paper_2509_10722_b200 import _lib
    from paper_2509_10722_b200.shard import p2p_local_group, run_ranks

    monkeypatch.setenv("NUMPMP_P2P_FUSED", "2")
    monkeypatch.setenv("NUMPMP_COL_BLOCKS", "2")
    p = _gen(1500, 3000, 6.0, 2, True, 23)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    ranks = p2p_local_group(p, cfg, world)
    L = _lib.lib()
    try:
        for s in ranks:
            assert L.numpmp_gpu_set_profiling(s.handle(), 1) == 0
        sols = run_ranks([s.solve for s in ranks])
        launches, iters = C.c_int64(), C.c_int64()
        k1, k2 = C.c_double(), C.c_double()
        assert L.numpmp_gpu_profile(ranks[0].handle(), C.byref(launches), C.byref(k1), C.byref(k2),
                                    C.byref(iters)) == 0
    finally:
        for s in ranks:
            s.close()
    # launches are counted per queued 32-iteration batch: 2 NB + 1 = 5 per
    # iteration fused (7 with the separate wait and finalize kernels)
    batches = -(-iters.value // 32)
    assert iters.value > 0 and launches.value % (32 * 5) == 0
    assert batches <= launches.value // (32 * 5) <= batches + 2
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    x = np.concatenate([s.x for s in sols])
    for s in sols:
        assert s.iterations == ref.iterations
        np.testing.assert_array_equal(s.lambda_raw, sols[0].lambda_raw)
    for got, want in [(x, ref.x), (sols[0].lambda_raw, ref.lambda_raw), (sols[0].s, ref.s)]:
        ok, err = close(got, want)
        assert ok, err


def test_p2p_exchange_repeated_and_warm_solves(restatement, oracle_mod):
    # the same ranks solving again (cold) and warm-started: each start state
    # must rebuild v on every rank, whatever the previous solve left there
    from paper_2509_10722_b200.shard import p2p_local_group, run_ranks

    p = _gen(1200, 2400, 5.0, 2, True, 41)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    ranks = p2p_local_group(p, cfg, 2)
    try:
        first = run_ranks([s.solve for s in ranks])
        again = run_ranks([s.solve for s in ranks])
        x0 = np.concatenate([s.x for s in first])
        warm = pmp.WarmStart(x0, first[0].lambda_raw, first[0].rho_final)
        warm_sols = run_ranks([lambda s=s: s.solve(warm) for s in ranks])
    finally:
        for s in ranks:
            s.close()
    for sols in (first, again):
        assert sols[0].iterations == ref.iterations
        ok, err = close(np.concatenate([s.x for s in sols]), ref.x)
        assert ok, err
    wref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg), warm=(warm.x0, warm.price, warm.rho))
    assert warm_sols[0].iterations == wref.iterations
    ok, err = close(np.concatenate([s.x for s in warm_sols]), wref.x)
    assert ok, err


def test_p2p_exchange_is_deterministic(monkeypatch):
    # rank-order sums: identical bytes on a rerun, whatever the arrival order
    from paper_2509_10722_b200.shard import p2p_local_group, run_ranks

    p = _gen(1500, 3000, 5.0, 2, True, 5)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    outs = []
    for _ in range(2):
        ranks = p2p_local_group(p, cfg, 3)
        try:
            outs.append(run_ranks([s.solve for s in ranks]))
        finally:
            for s in ranks:
                s.close()
    for a, b in zip(*outs):
        assert a.iterations == b.iterations
        np.testing.assert_array_equal(a.x, b.x)
        np.testing.assert_array_equal(a.lambda_raw, b.lambda_raw)


@pytest.mark.parametrize("K", [1, 10, 100])
def test_step_state_matches_oracle(K, restatement, oracle_mod):
    # state-level parity of step() on config A
    p = _gen(1000, 10000, 5.0, 0, False, 7)
    cfg = pmp.SolverConfig(rho0=1.0)
    a = oracle_mod.arrays_from(p)
    oc = ocfg(oracle_mod, cfg)
    ost = restatement.cold_state(a, oc)
    with pmp.PmpSolver(p, cfg) as s:
        st = s.cold_state()
        for _ in range(K):
            r, sn = s.step(st)
            ro, so, _ = restatement.step(a, oc, ost)
            assert abs(r - ro) <= RTOL * ro and abs(sn - so) <= RTOL * so
    for key in ("p", "z", "p_bar", "price"):
        ok, err = close(getattr(st, key), ost[key])
        assert ok, (key, err)
    assert st.iter == ost["iter"] == K


def test_warm_solve_matches_oracle(restatement, oracle_mod):
    # degrade workflow (config D shape, small): warm start from a prior solve
    base = _gen(500, 2000, 6.0, 2, True, 17)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1.0)
    with pmp.PmpSolver(base, cfg) as s:
        prior = s.solve()
    deg = pmp.degrade(base, 0.5, 0.5, 99)
    ratio = deg.capacities / base.capacities
    x0 = prior.x.copy()
    for j in range(deg.n):
        x0[j] *= min(1.0, float(np.min(ratio[deg.route(j)])))
        if deg.kinds[j] == 0 and not x0[j] > 0:
            x0[j] = 1e-8
    warm = pmp.WarmStart(x0, prior.lambda_raw / ratio, prior.rho_final / float(ratio.min()))
    with pmp.PmpSolver(deg, cfg) as s:
        sol = s.solve(warm)
    ref = restatement.solve(oracle_mod.arrays_from(deg), ocfg(oracle_mod, cfg), (warm.x0, warm.price, warm.rho))
    assert sol.iterations == ref.iterations
    ok, err = close(sol.x, ref.x)
    assert ok, err
    ok, err = close(sol.lambda_raw, ref.lambda_raw)
    assert ok, err


def test_termination_contract_post_hoc(restatement, oracle_mod):
    # acceptance.cpp criterion 4: residuals recomputed from the final state
    p = _gen(100, 50, 5.0, 2, True, 2)
    cfg = pmp.SolverConfig(eps_abs=1e-6)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
        st = s.final_state()
        prev_z = s.final_prev_z()
    a = oracle_mod.arrays_from(p)
    pbar = np.empty(p.m)
    pr, keep = restatement._prob(a)
    import ctypes

    restatement.L.oracle_link_averages(ctypes.byref(pr), oracle_mod._p(st.p), oracle_mod._p(pbar))
    r = math.sqrt(float(np.sum(a.link_counts * pbar * pbar)))
    sn = math.sqrt(float(np.sum((st.rho * (st.z - prev_z)) ** 2)))
    eps_tol = 1e-6 * math.sqrt(a.J)
    assert r < eps_tol and sn < eps_tol
    assert abs(r - sol.r_norm) <= 1e-9 * eps_tol and abs(sn - sol.s_norm) <= 1e-6 * eps_tol


def test_layout_bit_exact_with_reference(reference):
    # model.hpp:159-201: the device-built CSR against the reference layout
    for args in [(1000, 10000, 5.0, 0, ("constant", 1.0, 1.0), 7), (300, 150, 4.0, 2, ("uniform", 0.5, 1.5), 3)]:
        ra = reference.gen(*args).arrays()
        p = pmp.problem_from_arrays(ra.m, ra.n, ra.capacities, ra.weights, ra.kinds, ra.stream_offsets, ra.route_links)
        with pmp.PmpSolver(p) as s:
            lo, lt, lc = s.export_layout()
        np.testing.assert_array_equal(lo, ra.link_offsets)
        np.testing.assert_array_equal(lt, ra.link_terminals)
        np.testing.assert_array_equal(lc, ra.link_counts)


def test_layout_transit_unsorted_routes(reference):
    # config E shape (small): routes in travel order, not sorted
    rp = reference.gen_transit(12, 24, 5.0, 30, 40, 3, 24, 50.0, 4)
    ra = rp.arrays()
    p = pmp.problem_from_arrays(ra.m, ra.n, ra.capacities, ra.weights, ra.kinds, ra.stream_offsets, ra.route_links)
    with pmp.PmpSolver(p) as s:
        lo, lt, lc = s.export_layout()
    np.testing.assert_array_equal(lo, ra.link_offsets)
    np.testing.assert_array_equal(lt, ra.link_terminals)
    np.testing.assert_array_equal(lc, ra.link_counts)


def test_transit_solve_matches_reference(reference):
    rp = reference.gen_transit(12, 24, 5.0, 30, 40, 3, 24, 50.0, 4)
    ra = rp.arrays()
    p = pmp.problem_from_arrays(ra.m, ra.n, ra.capacities, ra.weights, ra.kinds, ra.stream_offsets, ra.route_links)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1.0, max_iters=3000)
    from oracle.oracle import Config

    ref = rp.solve(Config(eps_abs=1e-5, rho0=1.0, max_iters=3000))
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    assert sol.iterations == ref.iterations
    ok, err = close(sol.x, ref.x)
    assert ok, err


def test_runs_are_bit_identical():
    # determinism (parallel.hpp:54-76, test_solver.cpp:474-492): fixed-order device reductions
    p = _gen(2000, 4000, 6.0, 2, True, 11)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    with pmp.PmpSolver(p, cfg) as s:
        a = s.solve()
        b = s.solve()
    assert a.iterations == b.iterations
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.lambda_raw, b.lambda_raw)
    assert a.r_norm == b.r_norm and a.s_norm == b.s_norm


def test_extension_streams_rejected():
    p = pmp.problem_from_arrays(1, 1, [1.0], [1.0], [2], [0, 1], [0])
    with pytest.raises(pmp.SolverError):
        pmp.PmpSolver(p)


INVALID = [
    # (routes, kinds, weights, caps): model.hpp:76-155 rules, detected on the device
    ([[0, 0]], [0], [1.0], [1.0]),
    ([[]], [0], [1.0], [1.0]),
    ([[3]], [0], [1.0], [1.0]),
    ([[0]], [0], [1.0], [0.0, 1.0, 1.0]),
    ([[0]], [0], [0.0], [1.0]),
    ([[0]], [1], [-1.0], [1.0]),
    ([[0]], [0], [float("nan")], [1.0]),
    ([[0, 0], [5], [1, 1]] * 4, [0] * 12, [1.0] * 12, [1.0, -1.0]),
]


@pytest.mark.parametrize("case", INVALID)
def test_device_validation_raises_reference_message(case, reference):
    routes, kinds, weights, caps = case
    offs = np.cumsum([0] + [len(r) for r in routes]).astype(np.int64)
    rl = np.array([x for r in routes for x in r], np.int32)
    out = reference.build_problem(len(caps), len(routes), offs, rl, kinds, weights, caps)
    p = pmp.Problem(len(caps), len(routes), caps, weights, kinds, offs, rl)  # unvalidated
    with pytest.raises(pmp.ValidationError) as ei:
        pmp.PmpSolver(p)
    assert str(ei.value) == out[1]


def test_config_validation():
    p = single()
    for bad in [dict(eps_abs=0.0), dict(rho0=-1.0), dict(alpha=2.5), dict(mu=1.0), dict(gamma=1.0),
                dict(rho_update_interval=0), dict(max_iters=0), dict(trace_every=0), dict(threads=-1),
                dict(time_limit=-1.0)]:
        with pytest.raises(ValueError):
            pmp.PmpSolver(p, pmp.SolverConfig(**bad))


def test_cpp_dropin_binary():
    # include/numpmp/gpu_solver.hpp against the reference's own CPU
    # PmpSolver in one C++ binary (tests/cpp/test_dropin.cpp)
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("build/test_dropin not built (needs the reference headers at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASSED" in out.stdout


# ------------------------------------------------------------- config B / C
@pytest.mark.slow
def test_config_b_iterations_match_oracle(restatement, oracle_mod):
    # BASELINE.json configs[1]: 1M streams / 100k links, log utilities
    p = _gen(100000, 1000000, 10.0, 0, False, 7)
    cfg = pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0, max_iters=20)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert sol.iterations == ref.iterations == 20
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw)]:
        ok, err = close(got, want)
        assert ok, err
    for row, want in zip(sol.trace, ref.trace):
        assert abs(row.r_norm - want[1]) <= RTOL * want[1] and abs(row.s_norm - want[2]) <= RTOL * want[2]


@pytest.mark.slow
def test_config_c_first_iterations_match_oracle(restatement, oracle_mod):
    # BASELINE.json configs[2] at full size (100M nonzeros), K = 5 iterations
    p = _gen(1000000, 10000000, 10.0, 2, True, 7)
    cfg = pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0, max_iters=5, trace_every=1)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert sol.iterations == ref.iterations == 5
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw), (sol.s, ref.s)]:
        ok, err = close(got, want)
        assert ok, err
    assert len(sol.trace) == ref.trace.shape[0] == 5
    for row, want in zip(sol.trace, ref.trace):
        assert abs(row.r_norm - want[1]) <= RTOL * want[1] and abs(row.s_norm - want[2]) <= RTOL * want[2]
        assert abs(row.objective - want[4]) <= RTOL * abs(want[4])


@pytest.mark.slow
def test_config_c_full_solve_properties():
    # BASELINE.json configs[2] at full size: converged run is feasible within
    # tolerance and satisfies complementary slackness (test_solver.cpp:417-472)
    p = _gen(1000000, 10000000, 10.0, 2, True, 7)
    cfg = pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    assert sol.status == pmp.SolveStatus.Converged
    eps_tol = 1e-4 * math.sqrt(p.nnz + p.m)
    load = np.bincount(p.route_links, weights=np.repeat(sol.x, np.diff(p.stream_offsets)), minlength=p.m)
    viol = load + sol.s - p.capacities
    assert np.max(np.abs(viol)) <= 10.0 * eps_tol
    assert np.min(sol.x) >= -1e-4
    assert np.min(sol.lambda_) >= 0.0


def _config_f():
    # bench config F: B size + 100 hot links on ~10% of the streams (split rows)
    return pmp.gen_congested(pmp.GenSpec(m=100000, n=1000000, avg_links_per_stream=10.0, kind=pmp.GenKind.Mixed,
                                         weights=pmp.WeightDist.uniform(0.5, 1.5), seed=7), 0.001, 0.10)


@pytest.mark.slow
def test_config_f_first_iterations_match_oracle(restatement, oracle_mod):
    # the congested config at full size (2e7 nonzeros, hot rows of ~1e5 entries), K = 20 iterations
    p = _config_f()
    cfg = pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0, max_iters=20, trace_every=1)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert sol.iterations == ref.iterations == 20
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw), (sol.s, ref.s)]:
        ok, err = close(got, want)
        assert ok, err
    for row, want in zip(sol.trace, ref.trace):
        assert abs(row.r_norm - want[1]) <= RTOL * want[1] and abs(row.s_norm - want[2]) <= RTOL * want[2]


@pytest.mark.slow
def test_config_f_full_solve_properties():
    # converged congested run: feasible within tolerance, x >= 0, prices >= 0,
    # and bit-identical on a rerun (split-row pieces combine in a fixed order)
    p = _config_f()
    cfg = pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
        again = s.solve()
    assert sol.status == pmp.SolveStatus.Converged
    np.testing.assert_array_equal(sol.x, again.x)
    eps_tol = 1e-4 * math.sqrt(p.nnz + p.m)
    assert sol.r_norm < eps_tol and sol.s_norm < eps_tol
    load = np.bincount(p.route_links, weights=np.repeat(sol.x, np.diff(p.stream_offsets)), minlength=p.m)
    viol = np.abs(load + sol.s - p.capacities)
    # r^2 = sum_l (d_l + 1) pbar_l^2 bounds a link's load residual (d_l + 1) pbar_l by
    # sqrt(d_l + 1) r: the violation a converged run may leave grows with the degree
    deg = np.bincount(p.route_links, minlength=p.m)
    normal = deg <= 2 * p.nnz / p.m
    assert np.max(viol[normal]) <= 10.0 * eps_tol
    assert np.all(viol <= np.sqrt(deg + 1.0) * eps_tol)
    assert np.min(sol.x) >= -1e-4
    assert np.min(sol.lambda_) >= 0.0


def _ipc_rank(rank, world, port, q, fused=None):
    # one process per rank, all on cuda:0 (the box has one GPU): the real
    # CUDA IPC path of the exchange (export -> all_gather -> open), gloo for
    # the 64-byte handles
    import os

    if fused is not None:
        os.environ["NUMPMP_P2P_FUSED"] = fused

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2509_10722_b200 as pmp_
    from paper_2509_10722_b200.shard import ShardedPmpSolver

    p = _gen(1200, 2500, 5.0, 2, True, 3)
    cfg = pmp_.SolverConfig(eps_abs=1e-5, rho0=1000.0)

    def ipc_allgather(mine):
        out = [None] * world
        dist.all_gather_object(out, mine)
        return out

    s = ShardedPmpSolver(p, cfg, rank, world, device=0, exchange="p2p", ipc_allgather=ipc_allgather)
    sol = s.solve()
    s.close()
    q.put((rank, s.stream_begin, sol.x, sol.lambda_raw, sol.iterations))
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [None, "2"])
def test_p2p_exchange_over_cuda_ipc_processes(fused, restatement, oracle_mod):
    # fused "2": the one-GPU-per-rank owner epilogue (wait and finalize inside
    # it) forced across the two processes; they time-slice the GPU, so a
    # spinning epilogue only delays the other rank's kernels, and the
    # cross-process acquire / release protocol of the production path runs
    import socket

    import torch.multiprocessing as tmp

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_ipc_rank, args=(r, world, port, q, fused)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = _gen(1200, 2500, 5.0, 2, True, 3)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    x = np.concatenate([r[2] for r in sorted(res, key=lambda t: t[1])])
    assert all(r[4] == ref.iterations for r in res)
    for got, want in [(x, ref.x), (res[0][3], ref.lambda_raw)]:
        ok, err = close(got, want)
        assert ok, err


# ------------------------------------------------ warm-start recipes (warm.hpp)
def test_device_degrade_recipe_matches_reference(reference):
    # warm.hpp:25-57 on the device == the reference recipe, bit for bit; then
    # the warm re-solve matches the reference's warm re-solve
    case = (500, 2000, 6.0, 2, True, 17)
    base = _gen(*case)
    deg = pmp.degrade(base, 0.5, 0.5, 99)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1.0)
    with pmp.PmpSolver(base, cfg) as s:
        prior = s.solve()
    rb = reference.build_problem(base.m, base.n, base.stream_offsets, base.route_links, base.kinds, base.weights,
                                 base.capacities)
    rd = reference.build_problem(deg.m, deg.n, deg.stream_offsets, deg.route_links, deg.kinds, deg.weights,
                                 deg.capacities)

    class Prior:
        x, lambda_raw, rho_final = prior.x, prior.lambda_raw, prior.rho_final

    rx0, rprice, rrho = rb.warm_after_degrade(rd, Prior)
    with pmp.PmpSolver(deg, cfg) as s:
        w = s.warm_start_after_degrade(base, prior)
        sol = s.solve_prepared()
    np.testing.assert_array_equal(w.x0, rx0)
    np.testing.assert_array_equal(w.price, rprice)
    assert w.rho == rrho
    import oracle.oracle as o

    ref = rd.solve(o.Config(eps_abs=1e-5, rho0=1.0), warm=(rx0, rprice, rrho))
    assert sol.iterations == ref.iterations
    ok, err = close(sol.x, ref.x)
    assert ok, err


def test_device_prune_recipe_matches_reference(reference):
    # warm.hpp:62-94: loads summed in the reference's order, path prices in
    # route order: the recipe is bit-exact; the warm re-solve agrees
    case = (500, 2000, 4.0, 2, True, 23)
    base = _gen(*case)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1.0)
    with pmp.PmpSolver(base, cfg) as s:
        prior = s.solve()
    pruned, pmap = pmp.fail_and_prune(base, 0.2, 4)
    rb = reference.build_problem(base.m, base.n, base.stream_offsets, base.route_links, base.kinds, base.weights,
                                 base.capacities)
    rpr = rb.fail_and_prune(0.2, 4)

    class Prior:
        x, lambda_raw, rho_final = prior.x, prior.lambda_raw, prior.rho_final

    rx0, rprice, rrho = rpr.warm_after_prune(Prior, base.n, base.m)
    with pmp.PmpSolver(pruned, cfg) as s:
        w = s.warm_start_after_prune(pmap, prior)
        sol = s.solve_prepared()
    np.testing.assert_array_equal(w.x0, rx0)
    np.testing.assert_array_equal(w.price, rprice)
    assert w.rho == rrho
    import oracle.oracle as o

    ref = rpr.solve(o.Config(eps_abs=1e-5, rho0=1.0), warm=(rx0, rprice, rrho))
    assert sol.iterations == ref.iterations
    ok, err = close(sol.x, ref.x)
    assert ok, err


def test_device_path_prices_bit_exact():
    # transit.hpp:290-302 in route order
    p, _ = pmp.gen_transit(pmp.TransitSpec(12, 24, 5.0, 40, 30, 3, 6, 50.0, 2))
    lam = np.random.default_rng(0).uniform(0.0, 2.0, p.m)
    with pmp.PmpSolver(p, pmp.SolverConfig()) as s:
        pi = s.path_prices(lam)
    want = np.zeros(p.n)
    for j in range(p.n):  # plain left-to-right adds (Python's sum() compensates since 3.12)
        t = 0.0
        for l in p.route(j):
            t += float(lam[l])
        want[j] = t
    np.testing.assert_array_equal(pi, want)



def test_transit_report_from_device_solve(reference, tmp_path):
    # solve on the device, path prices on the device, the
    # report (transit.hpp:342-374) and both CSVs byte-identical to the
    # reference's on the same solution
    args = (12, 24, 5.0, 30, 40, 3, 24, 50.0, 4)
    p, meta = pmp.gen_transit(pmp.TransitSpec(*args), with_meta=True)
    rp = reference.gen_transit(*args)
    with pmp.PmpSolver(p, pmp.SolverConfig(eps_abs=1e-5, rho0=1.0, max_iters=3000, trace_every=7)) as s:
        sol = s.solve()
        pi = s.path_prices(sol.lambda_)
        n_rows = 0
        for od in range(len(meta.od_origin)):
            t0 = int(meta.stream_t0[meta.stream_od == od][0])
            rows = pmp.transit_report(p, sol.x, sol.lambda_, meta, od, t0, solver=s)
            assert [r.pi for r in rows] == [pi[r.stream] for r in rows]
            stream, rpi, hats = rp.transit_report(sol.x, sol.lambda_, od, t0, str(tmp_path / "ref.csv"))
            assert [r.stream for r in rows] == stream.tolist() and [r.pi for r in rows] == rpi.tolist()
            assert [r.lambda_hat for r in rows] == [h.tolist() for h in hats]
            pmp.write_transit_report_csv(rows, str(tmp_path / "mine.csv"))
            assert (tmp_path / "mine.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
            n_rows += len(rows)
    assert n_rows > 0 and sol.status == pmp.SolveStatus.Converged
    from oracle.oracle import ref_write_trace_csv

    pmp.write_trace_csv(sol.trace, str(tmp_path / "t_mine.csv"))
    t = sol.trace
    ref_write_trace_csv(reference, str(tmp_path / "t_ref.csv"), [r.iter for r in t], [r.r_norm for r in t],
                        [r.s_norm for r in t], [r.rho for r in t], [r.objective for r in t])
    assert (tmp_path / "t_mine.csv").read_bytes() == (tmp_path / "t_ref.csv").read_bytes()
    assert len(t) > 2

# ------------------------------------------- skew, ragged routes, edge shapes
def _ragged_problem():
    # one stream over every link (a 700-link route spans several staging
    # rounds of its tile), single-link routes, and links nobody uses
    rng = np.random.default_rng(5)
    m = 700
    routes = [list(range(m))]
    for j in range(1, 2000):
        k = 1 if j % 3 == 0 else int(rng.integers(2, 9))
        routes.append(sorted(rng.choice(600, size=k, replace=False).tolist()))  # links 600..699: only stream 0
    S = pmp.Stream
    streams = [S(j, pmp.StreamKind.Log if j % 2 else pmp.StreamKind.Linear, "", float(rng.uniform(0.5, 1.5)), r)
               for j, r in enumerate(routes)]
    return pmp.build_problem(streams, rng.uniform(0.5, 1.5, m).tolist())


SHAPE_CASES = {
    # hot links: 10 links in ~10% of the streams each (rows of ~2000 entries:
    # more than 32 segments, split over several warp units)
    "congested": lambda: pmp.gen_congested(pmp.GenSpec(m=2000, n=20000, avg_links_per_stream=4.0,
                                                       kind=pmp.GenKind.Mixed,
                                                       weights=pmp.WeightDist.uniform(0.5, 1.5), seed=13),
                                           0.005, 0.10),
    "ragged": _ragged_problem,
    # every stream on one link: a single row of n entries
    "one_link": lambda: pmp.build_problem([pmp.Stream(j, pmp.StreamKind.Log, "", 1.0 + 0.001 * j, [0])
                                           for j in range(5000)], [3.0]),
}


@pytest.mark.parametrize("shape", sorted(SHAPE_CASES))
@pytest.mark.parametrize("blocks", [1, 3])
def test_skewed_and_ragged_shapes_match_oracle(shape, blocks, restatement, oracle_mod, monkeypatch):
    monkeypatch.setenv("NUMPMP_COL_BLOCKS", str(blocks))
    p = SHAPE_CASES[shape]()
    cfg = (pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0, max_iters=20000) if shape == "congested"
           else pmp.SolverConfig(eps_abs=1e-5, rho0=1.0, max_iters=20000))
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert ref.error is None
    assert sol.iterations == ref.iterations and int(sol.status) == ref.status
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw), (sol.s, ref.s)]:
        ok, err = close(got, want)
        assert ok, err
    assert abs(sol.objective - ref.objective) <= RTOL * abs(ref.objective)


def _hot_problem():
    # hot rows of ~3000-6000 entries (split over 6-12 warp units) next to short rows
    return pmp.gen_congested(pmp.GenSpec(m=3000, n=30000, avg_links_per_stream=5.0, kind=pmp.GenKind.Mixed,
                                         weights=pmp.WeightDist.uniform(0.5, 1.5), seed=23), 0.004, 0.15)


@pytest.mark.parametrize("blocks", [1, 2])
def test_split_rows_deterministic_and_p2p(blocks, restatement, oracle_mod, monkeypatch):
    # split rows combine their pieces in unit order: identical bytes on a
    # rerun whatever warp finishes last, in the single-device engine and in
    # the peer-memory sharded engine (LP_P2P)
    from paper_2509_10722_b200.shard import p2p_local_group, run_ranks

    monkeypatch.setenv("NUMPMP_COL_BLOCKS", str(blocks))
    p = _hot_problem()
    assert np.bincount(p.route_links, minlength=p.m).max() > 32 * 16 * blocks
    cfg = pmp.SolverConfig(eps_abs=1e-4, rho0=1000.0, max_iters=20000)
    with pmp.PmpSolver(p, cfg) as s:
        a = s.solve()
        b = s.solve()
    assert a.iterations == b.iterations
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.lambda_raw, b.lambda_raw)
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert a.iterations == ref.iterations
    for got, want in [(a.x, ref.x), (a.lambda_raw, ref.lambda_raw)]:
        ok, err = close(got, want)
        assert ok, err
    ranks = p2p_local_group(p, cfg, 2)
    try:
        sols = run_ranks([r.solve for r in ranks])
        again = run_ranks([r.solve for r in ranks])
    finally:
        for r in ranks:
            r.close()
    assert sols[0].iterations == ref.iterations
    ok, err = close(np.concatenate([q.x for q in sols]), ref.x)
    assert ok, err
    np.testing.assert_array_equal(np.concatenate([q.x for q in sols]), np.concatenate([q.x for q in again]))


@pytest.mark.parametrize("row_mode_max", ["0", "100000"])
@pytest.mark.parametrize("blocks", [1, 3])
def test_link_pass_row_and_unit_modes_match_oracle(row_mode_max, blocks, restatement, oracle_mod, monkeypatch):
    # the link pass's two forms (lane per row / warp units of segments) on the
    # same problem: every block forced into one of them
    monkeypatch.setenv("NUMPMP_ROW_MODE_MAX", row_mode_max)
    monkeypatch.setenv("NUMPMP_COL_BLOCKS", str(blocks))
    p = _gen(3000, 2000, 6.0, 2, True, 19)
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=1000.0)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert sol.iterations == ref.iterations
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw), (sol.s, ref.s)]:
        ok, err = close(got, want)
        assert ok, err


@pytest.mark.parametrize("pair_tau,tile_q", [("0", "2"), ("100", "2"), ("100", "4")])
def test_stream_pass_tiles_and_pair_tiles_match_oracle(pair_tau, tile_q, restatement, oracle_mod, monkeypatch):
    # the stream pass on 32-stream tiles and on multi-route tiles (2 or 4
    # routes per lane), forced; transit-like short routes and a ragged tail
    monkeypatch.setenv("NUMPMP_PAIR_TILE_TAU", pair_tau)
    monkeypatch.setenv("NUMPMP_TILE_Q", tile_q)
    monkeypatch.setenv("NUMPMP_COL_BLOCKS", "2")
    p, _ = pmp.gen_transit(pmp.TransitSpec(12, 24, 5.0, 40, 30, 3, 6, 50.0, 2))
    cfg = pmp.SolverConfig(eps_abs=1e-5, rho0=10.0)
    with pmp.PmpSolver(p, cfg) as s:
        sol = s.solve()
    ref = restatement.solve(oracle_mod.arrays_from(p), ocfg(oracle_mod, cfg))
    assert sol.iterations == ref.iterations
    for got, want in [(sol.x, ref.x), (sol.lambda_raw, ref.lambda_raw)]:
        ok, err = close(got, want)
        assert ok, err
