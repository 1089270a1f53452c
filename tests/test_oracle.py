"""CPU tests of the oracle (the parity checker): the C restatement against
the reference itself (oracle/_ref) and against the committed golden
fixtures and the frozen values of the reference's own GoogleTest suites
(proj/tests/test_solver.cpp, test_prox.cpp).  Bit-exact throughout: the
restatement performs the reference's operations in the reference's order.
"""
import ctypes
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_case(oracle_mod, name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    a = oracle_mod.Arrays(int(z["m"]), int(z["n"]), z["capacities"], z["weights"], z["kinds"],
                          z["stream_offsets"], z["terminal_link"], z["link_offsets"], z["link_terminals"],
                          z["link_counts"])
    c = z["cfg"]
    cfg = oracle_mod.Config(eps_abs=c[0], rho0=c[1], alpha=c[2], mu=c[3], gamma=c[4], time_limit=c[5],
                            rho_update_interval=int(c[6]), max_iters=int(c[7]), trace_every=int(c[8]))
    return a, cfg, z


CASES = ["bipartite", "config_a", "mixed_small", "transit_small", "degraded_warm"]


@pytest.mark.parametrize("name", CASES)
def test_restatement_reproduces_golden_fixture(name, oracle_mod, restatement):
    a, cfg, z = load_case(oracle_mod, name)
    warm = None
    if name == "degraded_warm":
        w = np.load(os.path.join(GOLDEN, "degraded_warm_start.npz"))
        warm = (w["x0"], w["price"], float(w["rho"][0]))
    res = restatement.solve(a, cfg, warm)
    assert res.error is None
    assert res.iterations == int(z["ints"][1]) and res.status == int(z["ints"][0])
    np.testing.assert_array_equal(res.x, z["x"])
    np.testing.assert_array_equal(res.s, z["s"])
    np.testing.assert_array_equal(res.lambda_, z["lam"])
    np.testing.assert_array_equal(res.lambda_raw, z["lam_raw"])
    np.testing.assert_array_equal([res.objective, res.r_norm, res.s_norm, res.rho_final], z["scalars"])
    np.testing.assert_array_equal(res.trace, z["trace"])
    np.testing.assert_array_equal(res.final_z, z["final_z"])
    np.testing.assert_array_equal(res.final_p, z["final_p"])
    np.testing.assert_array_equal(res.final_prev_z, z["final_prev_z"])


@pytest.mark.parametrize("name", CASES)
def test_restatement_layout_matches_golden(name, oracle_mod, restatement):
    a, cfg, z = load_case(oracle_mod, name)
    tl, lo, lt, lc = restatement.build_layout(a.m, a.n, a.stream_offsets, a.route_links)
    np.testing.assert_array_equal(tl, z["terminal_link"])
    np.testing.assert_array_equal(lo, z["link_offsets"])
    np.testing.assert_array_equal(lt, z["link_terminals"])
    np.testing.assert_array_equal(lc, z["link_counts"])


@pytest.mark.parametrize("args", [
    (300, 150, 4.0, 2, ("uniform", 0.5, 1.5), 3, 1.0),
    (40, 20, 4.0, 2, ("constant", 1.0, 1.0), 9, 1.0),
    (2000, 4000, 6.0, 2, ("uniform", 0.5, 1.5), 11, 1000.0),
])
def test_restatement_matches_reference_solve(args, oracle_mod, restatement, reference):
    *g, rho0 = args
    rp = reference.gen(*g)
    cfg = oracle_mod.Config(eps_abs=1e-6, rho0=rho0, max_iters=5000)
    r1 = rp.solve(cfg, final_state=True)
    r2 = restatement.solve(rp.arrays(), cfg)
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(r1.x, r2.x)
    np.testing.assert_array_equal(r1.lambda_raw, r2.lambda_raw)
    np.testing.assert_array_equal(r1.trace, r2.trace)
    np.testing.assert_array_equal(r1.final_prev_z, r2.final_prev_z)


def test_restatement_matches_reference_steps(oracle_mod, restatement, reference):
    # StepResidualsMatchFreeFunction instance (test_solver.cpp:245-262)
    rp = reference.gen(40, 20, 4.0, 2, ("constant", 1.0, 1.0), 9)
    cfg = oracle_mod.Config()
    a = rp.arrays()
    st = restatement.cold_state(a, cfg)
    ref_st, rs = rp.steps(cfg, 20)
    for i in range(20):
        r, s, _ = restatement.step(a, cfg, st)
        assert (r, s) == (rs[i, 0], rs[i, 1])
    for k in ("p", "z", "p_bar", "price"):
        np.testing.assert_array_equal(st[k], ref_st[k])


# --------------------------------------------- frozen values of the reference tests
def test_prox_closed_forms(restatement):
    # test_prox.cpp:22-51
    assert abs(restatement.prox_log(2.0, 1.0, 1.0, 2) - (2.0 + math.sqrt(12.0)) / 4.0) <= 1e-12
    assert abs(restatement.prox_log(0.0, 1.0, 4.0, 1) - 0.5) <= 1e-12
    assert restatement.prox_log(-1e8, 1e-6, 1.0, 1) > 0.0
    assert restatement.prox_log(-1e12, 1.0, 10.0, 20) > 0.0
    assert restatement.prox_log(1e12, 1e-9, 0.1, 3) > 0.0
    assert restatement.prox_linear_nonneg(-2.0, 0.0, 1.0, 2) == 0.0
    assert restatement.prox_linear_nonneg(6.0, 3.0, 1.0, 2) == 4.5


def test_prox_matches_reference_on_random_draws(restatement, reference):
    rng = np.random.default_rng(2024)
    for _ in range(500):
        tau = int(rng.integers(1, 13))
        w, rho = rng.uniform(0.1, 5.0), rng.uniform(0.2, 5.0)
        z = float(rng.uniform(-5, 5) * tau)
        assert restatement.prox_log(z, w, rho, tau) == reference.prox_log(z, w, rho, tau)
        assert restatement.prox_linear_nonneg(z, w, rho, tau) == reference.prox_linear_nonneg(z, w, rho, tau)


def _single(oracle_mod, restatement, caps=(1.0,), routes=((0,),), kinds=(0,), weights=(1.0,)):
    offs = np.cumsum([0] + [len(r) for r in routes]).astype(np.int64)
    rl = np.concatenate([np.array(r, np.int32) for r in routes])
    tl, lo, lt, lc = restatement.build_layout(len(caps), len(routes), offs, rl)
    return oracle_mod.Arrays(len(caps), len(routes), np.array(caps, float), np.array(weights, float),
                             np.array(kinds, np.uint8), offs, tl, lo, lt, lc)


def test_first_iteration_from_zero_state(oracle_mod, restatement):
    # test_solver.cpp:110-124 (EXPECT_DOUBLE_EQ)
    a = _single(oracle_mod, restatement)
    cfg = oracle_mod.Config(alpha=1.0, rho0=1.0, rho_update_interval=1000000)
    st = restatement.cold_state(a, cfg)
    restatement.step(a, cfg, st)
    assert st["iter"] == 1
    assert list(st["p"]) == [1.0, 0.0] and list(st["p_bar"]) == [0.5]
    assert list(st["z"]) == [0.5, -0.5] and list(st["price"]) == [0.5]


@pytest.mark.parametrize("rho0", [1.0, 2.0])
def test_alpha1_matches_plain_transcription_bit_exact(rho0, oracle_mod, restatement):
    # test_solver.cpp:126-146 (ASSERT_EQ, 100 iterations)
    a = _single(oracle_mod, restatement, caps=(1.0, 1.0, 1.0), routes=((0,), (1, 2), (1,)), kinds=(0, 0, 0),
                weights=(1.0, 1.0, 1.0))
    cfg = oracle_mod.Config(alpha=1.0, rho0=rho0, rho_update_interval=1000000)
    st = restatement.cold_state(a, cfg)
    J = a.J
    pp, uu, pbar, arg = np.zeros(J), np.zeros(J), np.zeros(a.m), np.zeros(J)
    pr, keep = restatement._prob(a)
    for _ in range(100):
        restatement.step(a, cfg, st)
        restatement.L.oracle_plain_step(ctypes.byref(pr), ctypes.c_double(rho0),
                                        *[oracle_mod._p(v) for v in (pp, uu, pbar, arg)])
        np.testing.assert_array_equal(st["p"], pp)
        np.testing.assert_array_equal(st["price"][a.terminal_link], rho0 * uu)


@pytest.mark.parametrize("alpha", [1.0, 1.6])
def test_fixed_point_is_stationary(alpha, oracle_mod, restatement):
    # test_solver.cpp:148-171
    a = _single(oracle_mod, restatement)
    cfg = oracle_mod.Config(alpha=alpha, rho_update_interval=1000000)
    st = dict(p=np.array([1.0, -1.0]), z=np.array([1.0, -1.0]), p_bar=np.array([0.0]), price=np.array([1.0]),
              rho=1.0, iter=0)
    r, s, _ = restatement.step(a, cfg, st)
    np.testing.assert_allclose(st["p"], [1.0, -1.0], atol=1e-14)
    np.testing.assert_allclose(st["z"], [1.0, -1.0], atol=1e-14)
    assert abs(r) <= 1e-14 and abs(s) <= 1e-14


def test_link_averages_examples(oracle_mod, restatement):
    # test_solver.cpp:188-221
    a = _single(oracle_mod, restatement, caps=(1.0, 1.0, 1.0), routes=((0,), (1, 2), (1,)), kinds=(0, 0, 0),
                weights=(1.0, 1.0, 1.0))
    pr, keep = restatement._prob(a)
    flows = np.zeros(a.J)
    flows[1], flows[3], flows[a.nnz + 1] = 1.0, 2.0, -3.0
    pbar = np.zeros(a.m)
    restatement.L.oracle_link_averages(ctypes.byref(pr), oracle_mod._p(flows), oracle_mod._p(pbar))
    assert pbar[1] == 0.0
    flows[:] = 0.0
    flows[a.nnz + 2] = -1.0
    restatement.L.oracle_link_averages(ctypes.byref(pr), oracle_mod._p(flows), oracle_mod._p(pbar))
    assert pbar[2] == -0.5


def test_warm_start_slack_flows(oracle_mod, restatement):
    # test_solver.cpp:352-368
    a = _single(oracle_mod, restatement, caps=(1.0, 1.0, 1.0), routes=((0,), (1, 2), (1,)), kinds=(0, 0, 0),
                weights=(1.0, 1.0, 1.0))
    st = restatement.warm_state(a, oracle_mod.Config(), np.array([0.25, 0.5, 0.75]), None, 1.0)
    assert list(st["p"][a.nnz:]) == [-0.25, -1.0, -0.5]
    np.testing.assert_array_equal(st["z"], st["p"] - st["p_bar"][a.terminal_link])


def test_non_finite_reports_iteration(oracle_mod, restatement):
    # test_solver.cpp:173-186
    a = _single(oracle_mod, restatement, weights=(1e308,))
    res = restatement.solve(a, oracle_mod.Config(rho0=1e-8))
    assert res.error is not None and "iteration 1" in res.error


def test_max_iters_status(oracle_mod, restatement):
    # test_solver.cpp:384-393
    a = _single(oracle_mod, restatement, caps=(1.0, 1.0, 1.0), routes=((0,), (1, 2), (1,)), kinds=(0, 0, 0),
                weights=(1.0, 1.0, 1.0))
    res = restatement.solve(a, oracle_mod.Config(max_iters=3, eps_abs=1e-12))
    assert res.status == 1 and res.iterations == 3


def test_bipartite_fixture_solution(oracle_mod):
    # test_solver.cpp:98-108 / test_oracle.cpp:63-76: x = (1, .5, .5), lambda = (1, 2, 0)
    _, _, z = load_case(oracle_mod, "bipartite")
    np.testing.assert_allclose(z["x"], [1.0, 0.5, 0.5], rtol=1e-4)
    np.testing.assert_allclose(z["lam"], [1.0, 2.0, 0.0], atol=1e-3)


def test_config_a_iteration_count(oracle_mod):
    # config A at rho0 = 1000, eps 1e-4 -> 423 iterations
    _, _, z = load_case(oracle_mod, "config_a")
    assert int(z["ints"][1]) == 423 and int(z["ints"][0]) == 0
