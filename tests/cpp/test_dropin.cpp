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
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}
