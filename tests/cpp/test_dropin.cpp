// tests/cpp/test_dropin.cpp -- integration test of the C++ drop-in
// (include/numpmp/gpu_solver.hpp): the reference's own CPU PmpSolver and
// numpmp::gpu::PmpSolver run side by side on the same numpmp::Problem,
// built by the reference's own generators.  Built here (it needs the
// reference headers) by __graft_entry__.build(); run on the GPU box by
// tests/test_gpu_parity.py::test_cpp_dropin_binary.  Prints one PASS/FAIL
// line per check and exits non-zero on any failure.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "numpmp/gen.hpp"
#include "numpmp/gpu_solver.hpp"
#include "numpmp/solver.hpp"
#include "numpmp/warm.hpp"

using namespace numpmp;

static int g_fail = 0;
static void check(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++g_fail;
}

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double err = 0.0, scale = 1e-12;
  for (std::size_t i = 0; i < b.size(); ++i) {
    err = std::max(err, std::fabs(a[i] - b[i]));
    scale = std::max(scale, std::fabs(b[i]));
  }
  return err / scale;
}

int main() {
  // test_solver.cpp:110-124 through the drop-in
  {
    Problem p = build_problem({Stream{0, StreamKind::Log, "", 1.0, {0}}}, {1.0});
    SolverConfig cfg;
    cfg.alpha = 1.0;
    cfg.rho_update_interval = 1000000;
    gpu::PmpSolver s(p, cfg);
    SolverState st = s.cold_state();
    s.step(st);
    check(st.iter == 1 && std::fabs(st.p[0] - 1.0) < 1e-15 && std::fabs(st.p_bar[0] - 0.5) < 1e-15 &&
              std::fabs(st.z[1] + 0.5) < 1e-15 && std::fabs(st.price[0] - 0.5) < 1e-15,
          "FirstIterationFromZeroState");
  }
  // exceptions of the reference API
  {
    Problem p = build_problem({Stream{0, StreamKind::Log, "", 1.0, {0}}}, {1.0});
    SolverConfig bad;
    bad.alpha = 3.0;
    bool threw = false;
    try {
      gpu::PmpSolver s(p, bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(threw, "invalid config -> std::invalid_argument");
    Problem q = build_problem({Stream{0, StreamKind::Log, "", 1e308, {0}}}, {1.0});
    SolverConfig c2;
    c2.rho0 = 1e-8;
    threw = false;
    try {
      gpu::PmpSolver s(q, c2);
      s.solve();
    } catch (const SolverError& e) {
      threw = std::string(e.what()).find("iteration 1") != std::string::npos;
    }
    check(threw, "NonFiniteStateReportsIterationNumber -> SolverError");
  }
  // reference CPU engine vs drop-in on generated instances
  struct Case {
    const char* name;
    GenSpec spec;
    double eps, rho0;
  };
  std::vector<Case> cases;
  {
    GenSpec a;
    a.m = 1000;
    a.n = 10000;
    a.avg_links_per_stream = 5.0;
    a.seed = 7;
    cases.push_back({"config A rho0=1000", a, 1e-4, 1000.0});
    cases.push_back({"config A rho0=1", a, 1e-4, 1.0});
    GenSpec b;
    b.m = 2000;
    b.n = 4000;
    b.avg_links_per_stream = 6.0;
    b.kind = GenKind::Mixed;
    b.weights = WeightDist::uniform(0.5, 1.5);
    b.seed = 11;
    cases.push_back({"mixed 2000x4000", b, 1e-5, 1000.0});
  }
  for (const Case& c : cases) {
    Problem p = gen_uncongested(c.spec);
    SolverConfig cfg;
    cfg.eps_abs = c.eps;
    cfg.rho0 = c.rho0;
    PmpSolver cpu(p, cfg);
    Solution a = cpu.solve();
    gpu::PmpSolver dev(p, cfg);
    Solution b = dev.solve();
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s: iterations %lld vs %lld, x rel %.2e, price rel %.2e, obj rel %.2e",
                  c.name, (long long)a.iterations, (long long)b.iterations, max_rel(b.x, a.x),
                  max_rel(b.lambda_raw, a.lambda_raw),
                  std::fabs(b.objective - a.objective) / std::fabs(a.objective));
    check(a.iterations == b.iterations && a.status == b.status && max_rel(b.x, a.x) <= 1e-6 &&
              max_rel(b.lambda_raw, a.lambda_raw) <= 1e-6 &&
              std::fabs(b.objective - a.objective) <= 1e-6 * std::fabs(a.objective) &&
              a.trace.size() == b.trace.size(),
          buf);
    // acceptance.cpp criterion 4 on the drop-in's final state
    SolverState st = dev.final_state();
    compute_link_averages(st.p, p.layout, 1, st.p_bar);
    SolverState prev = st;
    prev.z = dev.final_prev_z();
    auto [r, s] = residuals(st, prev, p.layout);
    const double tol = cfg.eps_abs * std::sqrt(double(p.layout.total_terminals));
    std::snprintf(buf, sizeof buf, "%s: post-hoc r %.3e s %.3e < %.3e (reported %.3e %.3e)", c.name, r, s,
                  tol, b.r_norm, b.s_norm);
    check(r < tol && s < tol && std::fabs(r - b.r_norm) <= 1e-9 * tol &&
              std::fabs(s - b.s_norm) <= 1e-6 * tol,
          buf);
  }
  // warm start after degradation (warm.hpp:25-55)
  {
    GenSpec g;
    g.m = 2000;
    g.n = 1000;
    g.avg_links_per_stream = 10.0;
    g.seed = 101;
    Problem base = gen_uncongested(g);
    SolverConfig cfg;
    cfg.eps_abs = 1e-5;
    gpu::PmpSolver s0(base, cfg);
    Solution sol0 = s0.solve();
    Problem deg = degrade(base, 0.25, 0.5, 102);
    WarmStart w = warm_start_after_degrade(base, deg, sol0);
    PmpSolver cpu(deg, cfg);
    Solution a = cpu.solve(w);
    gpu::PmpSolver dev(deg, cfg);
    Solution b = dev.solve(w);
    Solution cold = dev.solve();
    char buf[200];
    std::snprintf(buf, sizeof buf, "degrade warm start: iterations cpu %lld gpu %lld (cold %lld), x rel %.2e",
                  (long long)a.iterations, (long long)b.iterations, (long long)cold.iterations,
                  max_rel(b.x, a.x));
    check(a.iterations == b.iterations && max_rel(b.x, a.x) <= 1e-6 && 2 * b.iterations <= cold.iterations,
          buf);
    // the same recipe on the device: bit-identical WarmStart, same re-solve
    WarmStart wd = dev.warm_start_after_degrade(base, sol0);
    Solution c = dev.solve_prepared();
    std::snprintf(buf, sizeof buf, "device degrade recipe: x0/price/rho bit-identical %d, iterations %lld",
                  int(wd.x0 == w.x0 && wd.price == w.price && wd.rho == w.rho), (long long)c.iterations);
    check(wd.x0 == w.x0 && wd.price == w.price && wd.rho == w.rho && c.iterations == a.iterations, buf);
  }
  {  // warm.hpp:62-94 after link failures, host recipe vs device recipe
    GenSpec spec;
    spec.m = 300;
    spec.n = 900;
    spec.avg_links_per_stream = 4.0;
    spec.kind = GenKind::Mixed;
    spec.seed = 31;
    Problem base = gen_uncongested(spec);
    SolverConfig cfg;
    cfg.eps_abs = 1e-5;
    gpu::PmpSolver s0(base, cfg);
    Solution sol0 = s0.solve();
    auto [pruned, map] = fail_and_prune(base, 0.2, 6);
    WarmStart w = warm_start_after_prune(pruned, map, sol0);
    gpu::PmpSolver dev(pruned, cfg);
    WarmStart wd = dev.warm_start_after_prune(map, sol0);
    Solution c = dev.solve_prepared();
    PmpSolver cpu(pruned, cfg);
    Solution a = cpu.solve(w);
    char buf[200];
    std::snprintf(buf, sizeof buf, "device prune recipe: bit-identical %d, iterations cpu %lld gpu %lld, x rel %.2e",
                  int(wd.x0 == w.x0 && wd.price == w.price && wd.rho == w.rho), (long long)a.iterations,
                  (long long)c.iterations, max_rel(c.x, a.x));
    check(wd.x0 == w.x0 && wd.price == w.price && wd.rho == w.rho && a.iterations == c.iterations &&
              max_rel(c.x, a.x) <= 1e-6,
          buf);
  }
  {  // StepResidualsMatchFreeFunction (test_solver.cpp:245-262): step() ==
     // the drop-in's residuals() bit for bit; the reference's host
     // residuals() on the same downloaded states within 1e-12 relative
    GenSpec spec;
    spec.m = 40;
    spec.n = 20;
    spec.avg_links_per_stream = 4.0;
    spec.kind = GenKind::Mixed;
    spec.seed = 9;
    Problem p = gen_uncongested(spec);
    gpu::PmpSolver solver(p, SolverConfig{});
    const gpu::PmpSolver& cs = solver;  // every member the reference declares const, through a const&
    SolverState st = cs.cold_state();
    bool bit = true, close = true;
    for (int iter = 0; iter < 20; ++iter) {
      SolverState prev = st;
      auto [r, s] = solver.step(st);
      auto [r_dev, s_dev] = cs.residuals(st, prev);
      auto [r_host, s_host] = residuals(st, prev, p.layout);
      bit = bit && r == r_dev && s == s_dev;
      close = close && std::fabs(r - r_host) <= 1e-12 * std::max(1.0, r_host) &&
              std::fabs(s - s_host) <= 1e-12 * std::max(1.0, s_host);
    }
    check(bit, "step() == residuals(after, before) bit for bit (20 steps)");
    check(close, "step() == host residuals() within 1e-12 (20 steps)");
    // groups() is the reference's partition (model.hpp:255-286)
    const auto& g = cs.groups();
    const auto ref_g = group_streams(p);
    bool same = g.size() == ref_g.size();
    for (std::size_t i = 0; same && i < g.size(); ++i)
      same = g[i].tau == ref_g[i].tau && g[i].kind == ref_g[i].kind && g[i].members == ref_g[i].members &&
             g[i].terminal_links == ref_g[i].terminal_links;
    check(same && cs.problem().n == p.n && cs.config().alpha == SolverConfig{}.alpha, "const accessors, groups()");
    WarmStart w;
    w.x0.assign(static_cast<std::size_t>(p.n), 1.0);
    const SolverState ws = cs.warm_state(w);
    PmpSolver cpu(p, SolverConfig{});
    const SolverState wr = cpu.warm_state(w);
    check(max_rel(ws.z, wr.z) <= 1e-12 && max_rel(ws.p_bar, wr.p_bar) <= 1e-12, "warm_state() const");
    solver.solve();
    const SolverState& fs = cs.final_state();
    const std::vector<double>& fz = cs.final_prev_z();
    check(fs.z.size() == fz.size() && fs.iter > 0, "final_state() / final_prev_z() const");
  }
  {  // multi-device drop-in: two stream shards with the peer-memory exchange
     // (both on device 0 here: one host thread per rank, as with 2 GPUs)
    GenSpec b;
    b.m = 2000;
    b.n = 4000;
    b.avg_links_per_stream = 6.0;
    b.kind = GenKind::Mixed;
    b.weights = WeightDist::uniform(0.5, 1.5);
    b.seed = 11;
    Problem p = gen_uncongested(b);
    SolverConfig cfg;
    cfg.eps_abs = 1e-5;
    cfg.rho0 = 1000.0;
    PmpSolver cpu(p, cfg);
    Solution a = cpu.solve();
    for (int world : {2, 3}) {
      gpu::PmpSolver dev(p, cfg, nullptr, std::vector<int>(static_cast<std::size_t>(world), 0));
      Solution c = dev.solve();
      Solution c2 = dev.solve();  // repeated solves on the same sharded handles
      char buf[240];
      std::snprintf(buf, sizeof buf,
                    "sharded drop-in (%d ranks, p2p): iterations cpu %lld gpu %lld, x rel %.2e, price rel %.2e",
                    world, (long long)a.iterations, (long long)c.iterations, max_rel(c.x, a.x),
                    max_rel(c.lambda_raw, a.lambda_raw));
      check(a.iterations == c.iterations && a.status == c.status && max_rel(c.x, a.x) <= 1e-6 &&
                max_rel(c.lambda_raw, a.lambda_raw) <= 1e-6 && c2.x == c.x && c2.iterations == c.iterations &&
                dev.shard_bounds().size() == static_cast<std::size_t>(world) + 1,
            buf);
      bool threw = false;
      try {
        dev.cold_state();
      } catch (const std::logic_error&) {
        threw = true;
      }
      check(threw, "sharded drop-in: terminal-space members throw std::logic_error");
      WarmStart w;
      w.x0 = a.x;
      w.price = a.lambda_raw;
      w.rho = a.rho_final;
      Solution d = dev.solve(w);
      std::snprintf(buf, sizeof buf, "sharded drop-in (%d ranks): warm start from the optimum, %lld iterations",
                    world, (long long)d.iterations);
      check(d.iterations <= 5 && d.status == SolveStatus::Converged, buf);
    }
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}
