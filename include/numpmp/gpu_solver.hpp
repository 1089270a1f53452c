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
//    counts, not bit for bit (different summation order);
//  * residuals(state, prev) is a member (the device reduction step() uses,
//    so step() == residuals(after, before) bit for bit, as solver.hpp:316-318
//    promises for the reference's free function);
//  * multi-GPU: PmpSolver(problem, cfg, ext, devices) with devices.size() > 1
//    shards the streams over the devices (nnz-balanced contiguous ranges,
//    one host thread per device, the fused peer-memory exchange of
//    numpmp_gpu_create_p2p); solve() / solve(warm) / groups() / accessors
//    work on it, the terminal-space members (cold_state, warm_state, step,
//    final_state, final_prev_z, residuals) are single-device only and throw
//    std::logic_error on a sharded solver.
#ifndef NUMPMP_GPU_SOLVER_HPP_
#define NUMPMP_GPU_SOLVER_HPP_

#include <algorithm>
#include <cstdint>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
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

// Runs fn(q) for q < count, one host thread each (the sharded engine's
// collective calls are made by every rank concurrently); rethrows the first
// exception after the join.
inline void for_each_rank(std::size_t count, const std::function<void(std::size_t)>& fn) {
  if (count == 1) {
    fn(0);
    return;
  }
  std::vector<std::exception_ptr> errs(count);
  std::vector<std::thread> ts;
  ts.reserve(count);
  for (std::size_t q = 0; q < count; ++q)
    ts.emplace_back([&, q] {
      try {
        fn(q);
      } catch (...) {
        errs[q] = std::current_exception();
      }
    });
  for (auto& t : ts) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

class PmpSolver {
 public:
  explicit PmpSolver(const Problem& problem, SolverConfig config = {},
                     const ExtensionRegistry* extensions = nullptr, int device = 0)
      : PmpSolver(problem, config, extensions, std::vector<int>{device}) {}

  // devices.size() > 1: one stream shard per device (see the file comment).
  PmpSolver(const Problem& problem, SolverConfig config, const ExtensionRegistry* extensions,
            std::vector<int> devices)
      : prob_(problem), cfg_(config), devices_(std::move(devices)) {
    (void)extensions;  // extension streams are rejected by the device engine
    if (devices_.empty()) throw std::invalid_argument("PmpSolver: no devices");
    const std::size_t n = static_cast<std::size_t>(problem.n);
    if (problem.layout.stream_offsets.size() != n + 1)
      throw ValidationError("invalid problem: layout missing (use build_problem)");
    weights_.resize(n);
    kinds_.resize(n);
    for (std::size_t j = 0; j < problem.streams.size() && j < n; ++j) {
      weights_[j] = problem.streams[j].weight;
      kinds_[j] = static_cast<std::uint8_t>(problem.streams[j].kind);
    }
    const numpmp_config c = to_c(cfg_);
    const std::size_t world = devices_.size();
    if (world == 1) {
      numpmp_problem_view v = view(0, problem.n, nullptr);
      throw_on_error(numpmp_gpu_create(&v, &c, devices_[0], &h_), nullptr);
      hs_.assign(1, h_);
      bounds_ = {0, problem.n};
      return;
    }
    // nnz-balanced contiguous stream ranges (shard.py shard_bounds)
    const auto& so = problem.layout.stream_offsets;
    const std::int64_t nnz = problem.layout.nnz;
    bounds_.assign(world + 1, 0);
    bounds_[world] = problem.n;
    for (std::size_t q = 1; q < world; ++q) {
      const std::int64_t target = static_cast<std::int64_t>(q) * nnz / static_cast<std::int64_t>(world);
      bounds_[q] = std::lower_bound(so.begin(), so.end(), target) - so.begin();
      bounds_[q] = std::max(bounds_[q - 1], std::min<std::int64_t>(bounds_[q], problem.n));
    }
    hs_.assign(world, nullptr);
    local_offsets_.resize(world);
    try {
      for (std::size_t q = 0; q < world; ++q) {
        const std::int64_t j0 = bounds_[q], j1 = bounds_[q + 1];
        local_offsets_[q].resize(static_cast<std::size_t>(j1 - j0) + 1);
        for (std::int64_t j = j0; j <= j1; ++j)
          local_offsets_[q][static_cast<std::size_t>(j - j0)] = so[static_cast<std::size_t>(j)] - so[static_cast<std::size_t>(j0)];
        numpmp_problem_view v = view(j0, j1, local_offsets_[q].data());
        throw_on_error(numpmp_gpu_create_p2p(&v, &c, devices_[q], static_cast<int>(q), static_cast<int>(world), j0,
                                             problem.n, &hs_[q]),
                       nullptr);
      }
      throw_on_error(numpmp_gpu_p2p_connect_local(hs_.data(), static_cast<int>(world)), nullptr);
      for_each_rank(world, [&](std::size_t q) { throw_on_error(numpmp_gpu_p2p_start(hs_[q]), hs_[q]); });
    } catch (...) {
      for (numpmp_gpu* hq : hs_) numpmp_gpu_destroy(hq);
      throw;
    }
    h_ = hs_[0];
  }
  ~PmpSolver() {
    for (numpmp_gpu* hq : hs_) numpmp_gpu_destroy(hq);
  }
  PmpSolver(const PmpSolver&) = delete;
  PmpSolver& operator=(const PmpSolver&) = delete;

  const Problem& problem() const { return prob_; }
  const SolverConfig& config() const { return cfg_; }
  // solver.hpp:291: the reference's own partition (model.hpp:255-286),
  // computed on first use; the device engine itself does not batch by group.
  const std::vector<TypeGroup>& groups() const {
    if (!have_groups_) {
      groups_ = group_streams(prob_);
      have_groups_ = true;
    }
    return groups_;
  }
  const std::vector<int>& devices() const { return devices_; }
  // stream range [shard_bounds()[q], shard_bounds()[q+1]) lives on devices()[q]
  const std::vector<std::int64_t>& shard_bounds() const { return bounds_; }

  SolverState cold_state() const {
    single("cold_state");
    throw_on_error(numpmp_gpu_set_cold(h_), h_);
    return download(false).first;
  }

  SolverState warm_state(const WarmStart& warm) const {
    single("warm_state");
    set_warm(warm);
    return download(false).first;
  }

  // One iteration; returns (r_norm, s_norm) of the new state, bit-identical
  // to residuals(after, before) below.  A state this solver issued (cold /
  // warm / stepped, unmodified) is kept on the device as is.
  std::pair<double, double> step(SolverState& st) {
    single("step");
    throw_on_error(numpmp_gpu_set_state(h_, st.p.data(), st.z.data(), st.p_bar.data(),
                                        st.price.data(), st.rho, st.iter),
                   h_);
    double r = 0.0, s = 0.0;
    throw_on_error(numpmp_gpu_step(h_, &r, &s), h_);
    st = download(false).first;
    return {r, s};
  }

  // residuals(state, prev, layout) (solver.hpp:139-154) with the device
  // reduction step() uses.
  std::pair<double, double> residuals(const SolverState& state, const SolverState& prev) const {
    single("residuals");
    const std::size_t J = static_cast<std::size_t>(prob_.layout.total_terminals);
    if (state.z.size() != J || prev.z.size() != J ||
        state.p_bar.size() != static_cast<std::size_t>(prob_.m))
      throw std::invalid_argument("residuals: state does not fit the problem");
    double r = 0.0, s = 0.0;
    throw_on_error(numpmp_gpu_residuals(h_, state.p_bar.data(), state.z.data(), prev.z.data(), state.rho,
                                        &r, &s),
                   h_);
    return {r, s};
  }

  Solution solve() {
    for_each_rank(hs_.size(), [&](std::size_t q) { throw_on_error(numpmp_gpu_set_cold(hs_[q]), hs_[q]); });
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
    single("warm_start_after_degrade");
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
    single("warm_start_after_prune");
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
  std::vector<double> path_prices(const std::vector<double>& lambda) const {
    single("path_prices");
    if (std::int64_t(lambda.size()) != prob_.m)
      throw std::invalid_argument("path_prices: lambda length mismatch");
    std::vector<double> pi(static_cast<std::size_t>(prob_.n));
    throw_on_error(numpmp_gpu_path_prices(h_, lambda.data(), pi.data()), h_);
    return pi;
  }

  const SolverState& final_state() const {
    materialize_final();
    return final_state_;
  }
  const std::vector<double>& final_prev_z() const {
    materialize_final();
    return final_prev_z_;
  }

 private:
  numpmp_problem_view view(std::int64_t j0, std::int64_t j1, const std::int64_t* offsets) const {
    const auto& so = prob_.layout.stream_offsets;
    numpmp_problem_view v{};
    v.m = prob_.m;
    v.n = j1 - j0;
    v.nnz = so[static_cast<std::size_t>(j1)] - so[static_cast<std::size_t>(j0)];
    v.capacities = prob_.capacities.data();
    v.weights = weights_.data() + j0;
    v.kinds = kinds_.data() + j0;
    v.stream_offsets = offsets ? offsets : so.data();
    v.route_links = prob_.layout.terminal_link.data() + so[static_cast<std::size_t>(j0)];  // [0, nnz): routes
    return v;
  }

  void single(const char* what) const {
    if (hs_.size() != 1)
      throw std::logic_error(std::string("PmpSolver::") + what + " is single-device only (sharded solver)");
  }

  void set_warm(const WarmStart& warm) const {
    if (std::int64_t(warm.x0.size()) != prob_.n)
      throw std::invalid_argument("warm start: x0 length does not match n");
    if (!warm.price.empty() && std::int64_t(warm.price.size()) != prob_.m)
      throw std::invalid_argument("warm start: price length mismatch");
    for_each_rank(hs_.size(), [&](std::size_t q) {
      throw_on_error(numpmp_gpu_set_warm(hs_[q], warm.x0.data() + bounds_[q],
                                         warm.price.empty() ? nullptr : warm.price.data(), warm.rho),
                     hs_[q]);
    });
  }

  std::pair<SolverState, std::vector<double>> download(bool with_prev_z) const {
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
    const std::size_t world = hs_.size();
    Solution sol;
    sol.x.resize(static_cast<std::size_t>(prob_.n));
    sol.s.resize(static_cast<std::size_t>(prob_.m));
    sol.lambda.resize(static_cast<std::size_t>(prob_.m));
    sol.lambda_raw.resize(static_cast<std::size_t>(prob_.m));
    const std::int64_t cap = cfg_.max_iters / cfg_.trace_every + 2;
    std::vector<numpmp_trace_row> rows(static_cast<std::size_t>(cap));
    std::vector<numpmp_solution_info> infos(world);
    have_final_ = false;
    // every rank: its x shard; link vectors and scalars are identical on
    // every rank, rank 0's are kept
    for_each_rank(world, [&](std::size_t q) {
      const bool r0 = q == 0;
      throw_on_error(numpmp_gpu_run(hs_[q], sol.x.data() + bounds_[q], r0 ? sol.s.data() : nullptr,
                                    r0 ? sol.lambda.data() : nullptr, r0 ? sol.lambda_raw.data() : nullptr,
                                    &infos[q], r0 ? rows.data() : nullptr, r0 ? cap : 0),
                     hs_[q]);
    });
    const numpmp_solution_info& info = infos[0];
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

  void materialize_final() const {
    single("final_state");
    if (have_final_) return;
    auto pr = download(true);
    final_state_ = std::move(pr.first);
    final_prev_z_ = std::move(pr.second);
    have_final_ = true;
  }

  const Problem& prob_;
  SolverConfig cfg_;
  std::vector<int> devices_;
  std::vector<double> weights_;
  std::vector<std::uint8_t> kinds_;
  std::vector<std::int64_t> bounds_;                      // world + 1 stream boundaries
  std::vector<std::vector<std::int64_t>> local_offsets_;  // rebased stream offsets per shard
  std::vector<numpmp_gpu*> hs_;                           // one handle per device
  numpmp_gpu* h_ = nullptr;                               // hs_[0]
  mutable bool have_final_ = false;
  mutable SolverState final_state_;
  mutable std::vector<double> final_prev_z_;
  mutable bool have_groups_ = false;
  mutable std::vector<TypeGroup> groups_;
};

}  // namespace gpu
}  // namespace numpmp

#endif  // NUMPMP_GPU_SOLVER_HPP_
