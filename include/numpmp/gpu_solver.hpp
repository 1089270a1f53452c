// numpmp/gpu_solver.hpp -- header-only C++ drop-in for the reference's
// numpmp::PmpSolver (proj/include/numpmp/solver.hpp:265-519), backed by the
// B200 engine in libnumpmp_cuda.so through its C-ABI (numpmp_gpu.h).
//
// A maintainer switches a call site from the CPU engine to the GPU one by
// replacing `numpmp::PmpSolver` with `numpmp::gpu::PmpSolver`: the
// constructor, cold_state / warm_state / step / solve, final_state /
// final_prev_z, the SolverConfig / SolverState / Solution / WarmStart types
// and the exception classes are the reference's own (this header includes
// numpmp/solver.hpp from the reference's include directory).
//
// Differences, by design:
//  * extension utilities (host std::function callbacks, prox.hpp:61-67)
//    cannot run in a kernel: streams of kind Extension throw SolverError at
//    construction;
//  * step() moves the state to the device and back (the device keeps it in
//    the stream/link form of SURVEY.md Appendix A); solve() never leaves
//    the device until the solution is downloaded;
//  * results match the CPU engine within 1e-6 relative at equal iteration
//    counts, not bit for bit (different summation order).
#ifndef NUMPMP_GPU_SOLVER_HPP_
#define NUMPMP_GPU_SOLVER_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "numpmp/common.hpp"
#include "numpmp/gen.hpp"
#include "numpmp/model.hpp"
#include "numpmp/prox.hpp"
#include "numpmp/solver.hpp"
#include "numpmp_gpu.h"

namespace numpmp {
namespace gpu {

// Maps a C-ABI return code to the reference's exception types
// (common.hpp:11-43, solver.hpp:32-44).
inline void throw_on_error(int rc, const numpmp_gpu* h) {
  if (rc == NUMPMP_OK) return;
  const std::string msg = numpmp_gpu_last_error(h);
  switch (rc) {
    case NUMPMP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case NUMPMP_VALIDATION_ERROR: throw ValidationError(msg);
    case NUMPMP_SOLVER_ERROR: throw SolverError(msg);
    case NUMPMP_DOMAIN_ERROR: throw std::domain_error(msg);
    default: throw std::runtime_error("numpmp gpu: " + msg);
  }
}

inline numpmp_config to_c(const SolverConfig& c) {
  numpmp_config o{};
  o.eps_abs = c.eps_abs;
  o.rho0 = c.rho0;
  o.alpha = c.alpha;
  o.mu = c.mu;
  o.gamma = c.gamma;
  o.time_limit = c.time_limit;
  o.rho_update_interval = c.rho_update_interval;
  o.max_iters = c.max_iters;
  o.trace_every = c.trace_every;
  o.threads = c.threads;
  return o;
}

class PmpSolver {
 public:
  explicit PmpSolver(const Problem& problem, SolverConfig config = {},
                     const ExtensionRegistry* extensions = nullptr, int device = 0)
      : prob_(problem), cfg_(config) {
    (void)extensions;  // extension streams are rejected by the device engine
    const std::size_t n = static_cast<std::size_t>(problem.n);
    weights_.resize(n);
    kinds_.resize(n);
    for (std::size_t j = 0; j < problem.streams.size() && j < n; ++j) {
      weights_[j] = problem.streams[j].weight;
      kinds_[j] = static_cast<std::uint8_t>(problem.streams[j].kind);
    }
    numpmp_problem_view v{};
    v.m = problem.m;
    v.n = problem.n;
    v.nnz = problem.layout.nnz;
    v.capacities = problem.capacities.data();
    v.weights = weights_.data();
    v.kinds = kinds_.data();
    v.stream_offsets = problem.layout.stream_offsets.data();
    v.route_links = problem.layout.terminal_link.data();  // [0, nnz): routes
    if (problem.layout.stream_offsets.size() != n + 1)
      throw ValidationError("invalid problem: layout missing (use build_problem)");
    const numpmp_config c = to_c(cfg_);
    throw_on_error(numpmp_gpu_create(&v, &c, device, &h_), nullptr);
  }
  ~PmpSolver() { numpmp_gpu_destroy(h_); }
  PmpSolver(const PmpSolver&) = delete;
  PmpSolver& operator=(const PmpSolver&) = delete;

  const Problem& problem() const { return prob_; }
  const SolverConfig& config() const { return cfg_; }

  SolverState cold_state() {
    throw_on_error(numpmp_gpu_set_cold(h_), h_);
    return download(false).first;
  }

  SolverState warm_state(const WarmStart& warm) {
    set_warm(warm);
    return download(false).first;
  }

  // One iteration; returns (r_norm, s_norm) of the new state.
  std::pair<double, double> step(SolverState& st) {
    throw_on_error(numpmp_gpu_set_state(h_, st.p.data(), st.z.data(), st.p_bar.data(),
                                        st.price.data(), st.rho, st.iter),
                   h_);
    double r = 0.0, s = 0.0;
    throw_on_error(numpmp_gpu_step(h_, &r, &s), h_);
    st = download(false).first;
    return {r, s};
  }

  Solution solve() {
    throw_on_error(numpmp_gpu_set_cold(h_), h_);
    return run();
  }

  Solution solve(const WarmStart& warm) {
    set_warm(warm);
    return run();
  }

  // warm.hpp:25-57 warm_start_after_degrade, computed on the device for this
  // solver's (degraded) problem; `before` is the problem `prior` solved.
  // The warm state is applied: solve_prepared() continues from it.  Returns
  // the recipe's WarmStart (bit-identical to the reference function).
  WarmStart warm_start_after_degrade(const Problem& before, const Solution& prior) {
    if (before.m != prob_.m || before.n != prob_.n)
      throw std::invalid_argument("degrade warm start: problems differ in structure");
    WarmStart w;
    w.x0.resize(static_cast<std::size_t>(prob_.n));
    w.price.resize(static_cast<std::size_t>(prob_.m));
    throw_on_error(numpmp_gpu_warm_after_degrade(h_, before.capacities.data(), prior.x.data(),
                                                 prior.lambda_raw.data(), prior.rho_final,
                                                 w.x0.data(), w.price.data(), &w.rho),
                   h_);
    return w;
  }

  // warm.hpp:62-94 warm_start_after_prune on the device (this solver holds
  // the pruned problem); the PruneMap projection is a host gather.
  WarmStart warm_start_after_prune(const PruneMap& map, const Solution& prior) {
    const std::vector<double> x0 = map.project_streams(prior.x);
    const std::vector<double> price = map.project_links(prior.lambda_raw);
    if (std::int64_t(x0.size()) != prob_.n || std::int64_t(price.size()) != prob_.m)
      throw std::invalid_argument("prune warm start: map does not fit problem");
    WarmStart w;
    w.x0.resize(x0.size());
    w.price.resize(price.size());
    throw_on_error(numpmp_gpu_warm_after_prune(h_, x0.data(), price.data(), prior.rho_final,
                                               w.x0.data(), w.price.data(), &w.rho),
                   h_);
    return w;
  }

  // run() from the state the last warm-start recipe applied.
  Solution solve_prepared() { return run(); }

  // transit.hpp:290-302 path_prices on the device (route order).
  std::vector<double> path_prices(const std::vector<double>& lambda) {
    if (std::int64_t(lambda.size()) != prob_.m)
      throw std::invalid_argument("path_prices: lambda length mismatch");
    std::vector<double> pi(static_cast<std::size_t>(prob_.n));
    throw_on_error(numpmp_gpu_path_prices(h_, lambda.data(), pi.data()), h_);
    return pi;
  }

  const SolverState& final_state() {
    materialize_final();
    return final_state_;
  }
  const std::vector<double>& final_prev_z() {
    materialize_final();
    return final_prev_z_;
  }

 private:
  void set_warm(const WarmStart& warm) {
    if (std::int64_t(warm.x0.size()) != prob_.n)
      throw std::invalid_argument("warm start: x0 length does not match n");
    if (!warm.price.empty() && std::int64_t(warm.price.size()) != prob_.m)
      throw std::invalid_argument("warm start: price length mismatch");
    throw_on_error(numpmp_gpu_set_warm(h_, warm.x0.data(),
                                       warm.price.empty() ? nullptr : warm.price.data(), warm.rho),
                   h_);
  }

  std::pair<SolverState, std::vector<double>> download(bool with_prev_z) {
    const std::size_t J = static_cast<std::size_t>(prob_.layout.total_terminals);
    SolverState st;
    st.p.resize(J);
    st.z.resize(J);
    st.p_bar.resize(static_cast<std::size_t>(prob_.m));
    st.price.resize(static_cast<std::size_t>(prob_.m));
    std::vector<double> prev;
    if (with_prev_z) prev.resize(J);
    throw_on_error(numpmp_gpu_get_state(h_, st.p.data(), st.z.data(), st.p_bar.data(),
                                        st.price.data(), &st.rho, &st.iter,
                                        with_prev_z ? prev.data() : nullptr),
                   h_);
    return {std::move(st), std::move(prev)};
  }

  Solution run() {
    Solution sol;
    sol.x.resize(static_cast<std::size_t>(prob_.n));
    sol.s.resize(static_cast<std::size_t>(prob_.m));
    sol.lambda.resize(static_cast<std::size_t>(prob_.m));
    sol.lambda_raw.resize(static_cast<std::size_t>(prob_.m));
    const std::int64_t cap = cfg_.max_iters / cfg_.trace_every + 2;
    std::vector<numpmp_trace_row> rows(static_cast<std::size_t>(cap));
    numpmp_solution_info info{};
    have_final_ = false;
    throw_on_error(numpmp_gpu_run(h_, sol.x.data(), sol.s.data(), sol.lambda.data(),
                                  sol.lambda_raw.data(), &info, rows.data(), cap),
                   h_);
    sol.objective = info.objective;
    sol.status = info.status == NUMPMP_CONVERGED  ? SolveStatus::Converged
                 : info.status == NUMPMP_TIMELIMIT ? SolveStatus::TimeLimit
                                                    : SolveStatus::MaxIters;
    sol.iterations = info.iterations;
    sol.r_norm = info.r_norm;
    sol.s_norm = info.s_norm;
    sol.rho_final = info.rho_final;
    for (std::int64_t i = 0; i < info.trace_len && i < cap; ++i) {
      const numpmp_trace_row& r = rows[static_cast<std::size_t>(i)];
      sol.trace.push_back(TraceRecord{r.iter, r.r_norm, r.s_norm, r.rho, r.objective});
    }
    return sol;
  }

  void materialize_final() {
    if (have_final_) return;
    auto pr = download(true);
    final_state_ = std::move(pr.first);
    final_prev_z_ = std::move(pr.second);
    have_final_ = true;
  }

  const Problem& prob_;
  SolverConfig cfg_;
  std::vector<double> weights_;
  std::vector<std::uint8_t> kinds_;
  numpmp_gpu* h_ = nullptr;
  bool have_final_ = false;
  SolverState final_state_;
  std::vector<double> final_prev_z_;
};

}  // namespace gpu
}  // namespace numpmp

#endif  // NUMPMP_GPU_SOLVER_HPP_
