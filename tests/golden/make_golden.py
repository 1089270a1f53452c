"""Generate tests/golden/*.npz from the reference itself (oracle/_ref, the
unmodified numpmp headers compiled by oracle/Makefile).  Run here, where
/root/reference exists; the fixtures are committed so the CPU tests and the
GPU box (which has no /root/reference) can check against them.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as o  # noqa: E402


def save_case(name, rp, cfg, warm=None):
    a = rp.arrays()
    res = rp.solve(cfg, warm=warm, final_state=True)
    assert res.error is None, res.error
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"),
        m=a.m, n=a.n, capacities=a.capacities, weights=a.weights, kinds=a.kinds,
        stream_offsets=a.stream_offsets, terminal_link=a.terminal_link, link_offsets=a.link_offsets,
        link_terminals=a.link_terminals, link_counts=a.link_counts,
        cfg=np.array([cfg.eps_abs, cfg.rho0, cfg.alpha, cfg.mu, cfg.gamma, cfg.time_limit,
                      cfg.rho_update_interval, cfg.max_iters, cfg.trace_every], np.float64),
        x=res.x, s=res.s, lam=res.lambda_, lam_raw=res.lambda_raw,
        scalars=np.array([res.objective, res.r_norm, res.s_norm, res.rho_final], np.float64),
        ints=np.array([res.status, res.iterations], np.int64), trace=res.trace,
        final_p=res.final_p, final_z=res.final_z, final_pbar=res.final_pbar, final_price=res.final_price,
        final_prev_z=res.final_prev_z,
    )
    print(name, a.m, a.n, a.nnz, res.iterations, res.status)


def main():
    ref = o.Reference()
    # bipartite fixture (test_solver.cpp:15-20)
    fx = ref.build_problem(3, 3, [0, 1, 3, 4], [0, 1, 2, 1], [0, 0, 0], [1.0, 1.0, 1.0], [1.0, 1.0, 1.0])
    save_case("bipartite", fx, o.Config(eps_abs=1e-7))
    # config A (BASELINE configs[0]), rho0 = 1000, eps 1e-4
    save_case("config_a", ref.gen(1000, 10000, 5.0, 0, ("constant", 1.0, 1.0), 7), o.Config(eps_abs=1e-4, rho0=1000.0))
    # mixed log/linear with uniform weights (ConvergedRunsAreFeasible shape)
    save_case("mixed_small", ref.gen(100, 50, 5.0, 2, ("uniform", 0.5, 1.5), 1), o.Config(eps_abs=1e-6))
    # time-expanded transit (config E shape, small)
    save_case("transit_small", ref.gen_transit(12, 24, 5.0, 30, 40, 3, 24, 50.0, 4),
              o.Config(eps_abs=1e-5, max_iters=3000))
    # degraded warm start (config D workflow, warm.hpp:25-55)
    base = ref.gen(500, 2000, 6.0, 2, ("uniform", 0.5, 1.5), 17)
    prior = base.solve(o.Config(eps_abs=1e-5))
    deg = base.degrade(0.5, 0.5, 99)
    warm = base.warm_after_degrade(deg, prior)
    save_case("degraded_warm", deg, o.Config(eps_abs=1e-5), warm=warm)
    np.savez_compressed(os.path.join(HERE, "degraded_warm_start.npz"), x0=warm[0], price=warm[1],
                        rho=np.array([warm[2]]))


if __name__ == "__main__":
    main()
