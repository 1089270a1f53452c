// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference numpmp headers
// (/root/reference/proj/include, included read-only at compile time by
// oracle/Makefile; no reference source is copied into this repo).  Built to
// oracle/_ref/libnumpmp_ref.so, it lets the Python tests and bench.py's
// reference arm call the reference's own generators and its own
// PmpSolver (solver.hpp:265-519) on the same inputs as the GPU path.
//
// numpmp.hpp / oracle.hpp are NOT included: they pull in Eigen, which is
// absent here.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "numpmp/common.hpp"
#include "numpmp/gen.hpp"
#include "numpmp/io.hpp"
#include "numpmp/model.hpp"
#include "numpmp/parallel.hpp"
#include "numpmp/prox.hpp"
#include "numpmp/solver.hpp"
#include "numpmp/transit.hpp"
#include "numpmp/warm.hpp"

using namespace numpmp;

namespace {

struct RefProblem {
  Problem p;
  TransitMetadata meta;  // filled for transit instances only
  std::vector<std::int32_t> prune_link_map;
  std::vector<std::int64_t> prune_stream_map;
};

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ValidationError*>(&e)) return 2;
  if (dynamic_cast<const SolverError*>(&e)) return 3;
  if (dynamic_cast<const std::domain_error*>(&e)) return 4;
  if (dynamic_cast<const GenError*>(&e)) return 5;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  return 9;
}

SolverConfig to_cfg(const double* d, const std::int64_t* i) {
  // d = {eps_abs, rho0, alpha, mu, gamma, time_limit}
  // i = {rho_update_interval, max_iters, trace_every, threads}
  SolverConfig c;
  c.eps_abs = d[0];
  c.rho0 = d[1];
  c.alpha = d[2];
  c.mu = d[3];
  c.gamma = d[4];
  c.time_limit = d[5];
  c.rho_update_interval = i[0];
  c.max_iters = i[1];
  c.trace_every = i[2];
  c.threads = static_cast<int>(i[3]);
  return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* h) { delete static_cast<RefProblem*>(h); }

// io.hpp:126-279 (encoding: 0 auto, 1 text, 2 binary)
int ref_write_problem(void* h, const char* path, int encoding) {
  try {
    write_problem(static_cast<RefProblem*>(h)->p, path,
                  encoding == 1 ? ProblemEncoding::Text
                                : (encoding == 2 ? ProblemEncoding::Binary : ProblemEncoding::Auto));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int ref_read_problem(const char* path, void** out) {
  try {
    auto* r = new RefProblem();
    try {
      r->p = read_problem(path);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// gen.hpp:91-97 / 103-128.  kind: 0 log, 1 linear, 2 mixed;
// wkind: 0 constant(wa), 1 uniform(wa, wb).  congested != 0 -> gen_congested.
int ref_gen(std::int64_t m, std::int64_t n, double avg, int kind, int wkind,
            double wa, double wb, std::uint64_t seed, int congested,
            double hot_link_fraction, double hot_stream_fraction, void** out) {
  try {
    GenSpec s;
    s.m = m;
    s.n = n;
    s.avg_links_per_stream = avg;
    s.kind = kind == 0 ? GenKind::Log : (kind == 1 ? GenKind::Linear : GenKind::Mixed);
    s.weights = wkind == 0 ? WeightDist::constant(wa) : WeightDist::uniform(wa, wb);
    s.seed = seed;
    auto* r = new RefProblem();
    r->p = congested ? gen_congested(s, hot_link_fraction, hot_stream_fraction)
                     : gen_uncongested(s);
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// transit.hpp:152-287
int ref_gen_transit(std::int32_t stations, std::int32_t time_bins, double bin_minutes,
                    std::int64_t spatial_edges, std::int64_t od_pairs,
                    std::int32_t routes_per_od, std::int32_t departures_per_route,
                    double seats, std::uint64_t seed, void** out,
                    std::int64_t* dropped) {
  try {
    TransitSpec s;
    s.stations = stations;
    s.time_bins = time_bins;
    s.bin_minutes = bin_minutes;
    s.spatial_edges = spatial_edges;
    s.od_pairs = od_pairs;
    s.routes_per_od = routes_per_od;
    s.departures_per_route = departures_per_route;
    s.seats = seats;
    s.seed = seed;
    auto* r = new RefProblem();
    auto pr = gen_transit(s);
    r->p = std::move(pr.first);
    r->meta = std::move(pr.second);
    *dropped = r->meta.dropped_streams;
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// gen.hpp:132-143
int ref_degrade(void* h, double p_degrade, double factor, std::uint64_t seed, void** out) {
  try {
    auto* r = new RefProblem();
    r->p = degrade(static_cast<RefProblem*>(h)->p, p_degrade, factor, seed);
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// gen.hpp:181-222; the prune map is kept on the new handle.
int ref_fail_and_prune(void* h, double p_fail, std::uint64_t seed, void** out) {
  try {
    auto* r = new RefProblem();
    auto pr = fail_and_prune(static_cast<RefProblem*>(h)->p, p_fail, seed);
    r->p = std::move(pr.first);
    r->prune_link_map = pr.second.link_map;
    r->prune_stream_map = pr.second.stream_map;
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_prune_maps(void* h, std::int32_t* link_map, std::int64_t* stream_map) {
  auto* r = static_cast<RefProblem*>(h);
  std::memcpy(link_map, r->prune_link_map.data(), r->prune_link_map.size() * 4);
  std::memcpy(stream_map, r->prune_stream_map.data(), r->prune_stream_map.size() * 8);
}

// model.hpp:222-241 from flat arrays (routes concatenated by offsets).
int ref_build_problem(std::int64_t n, std::int64_t m, const std::int64_t* offsets,
                      const std::int32_t* routes, const std::uint8_t* kinds,
                      const double* weights, const double* capacities, void** out) {
  try {
    std::vector<Stream> streams(static_cast<std::size_t>(n));
    for (std::int64_t j = 0; j < n; ++j) {
      Stream& s = streams[static_cast<std::size_t>(j)];
      s.id = j;
      s.kind = static_cast<StreamKind>(kinds[j]);
      s.weight = weights[j];
      s.route.assign(routes + offsets[j], routes + offsets[j + 1]);
    }
    std::vector<double> c(capacities, capacities + m);
    auto* r = new RefProblem();
    r->p = build_problem(std::move(streams), std::move(c));
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_sizes(void* h, std::int64_t* m, std::int64_t* n, std::int64_t* nnz) {
  const Problem& p = static_cast<RefProblem*>(h)->p;
  *m = p.m;
  *n = p.n;
  *nnz = p.layout.nnz;
}

// Problem + TerminalLayout as flat arrays (any pointer may be null).
void ref_export(void* h, double* capacities, double* weights, std::uint8_t* kinds,
                std::int64_t* stream_offsets, std::int32_t* terminal_link,
                std::int64_t* link_offsets, std::int64_t* link_terminals,
                std::int32_t* link_counts) {
  const Problem& p = static_cast<RefProblem*>(h)->p;
  const TerminalLayout& L = p.layout;
  if (capacities) std::memcpy(capacities, p.capacities.data(), 8 * p.m);
  for (std::int64_t j = 0; j < p.n; ++j) {
    const Stream& s = p.streams[static_cast<std::size_t>(j)];
    if (weights) weights[j] = s.weight;
    if (kinds) kinds[j] = static_cast<std::uint8_t>(s.kind);
  }
  if (stream_offsets) std::memcpy(stream_offsets, L.stream_offsets.data(), 8 * (p.n + 1));
  if (terminal_link) std::memcpy(terminal_link, L.terminal_link.data(), 4 * L.total_terminals);
  if (link_offsets) std::memcpy(link_offsets, L.link_offsets.data(), 8 * (p.m + 1));
  if (link_terminals) std::memcpy(link_terminals, L.link_terminals.data(), 8 * L.total_terminals);
  if (link_counts) std::memcpy(link_counts, L.link_counts.data(), 4 * p.m);
}

// PmpSolver::solve / solve(WarmStart) (solver.hpp:411-413).  warm_x0 null ->
// cold start.  Outputs: x[n], s[m], lambda[m], lambda_raw[m]; scal =
// {objective, r_norm, s_norm, rho_final, seconds}; ints = {status,
// iterations, trace_len}; trace rows as 5 doubles (iter, r, s, rho, obj).
// final_p/z/pbar/price/prev_z may be null.
int ref_solve(void* h, const double* cfgd, const std::int64_t* cfgi,
              const double* warm_x0, const double* warm_price, double warm_rho,
              double* x, double* s, double* lambda, double* lambda_raw, double* scal,
              std::int64_t* ints, double* trace, std::int64_t trace_cap,
              double* final_p, double* final_z, double* final_pbar,
              double* final_price, double* final_prev_z) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    PmpSolver solver(p, to_cfg(cfgd, cfgi));
    Solution sol;
    WarmStart warm;
    if (warm_x0) {
      warm.x0.assign(warm_x0, warm_x0 + p.n);
      if (warm_price) warm.price.assign(warm_price, warm_price + p.m);
      warm.rho = warm_rho;
    }
    const auto t0 = std::chrono::steady_clock::now();
    sol = warm_x0 ? solver.solve(warm) : solver.solve();
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(x, sol.x.data(), 8 * p.n);
    std::memcpy(s, sol.s.data(), 8 * p.m);
    std::memcpy(lambda, sol.lambda.data(), 8 * p.m);
    std::memcpy(lambda_raw, sol.lambda_raw.data(), 8 * p.m);
    scal[0] = sol.objective;
    scal[1] = sol.r_norm;
    scal[2] = sol.s_norm;
    scal[3] = sol.rho_final;
    scal[4] = secs;
    ints[0] = static_cast<std::int64_t>(sol.status);
    ints[1] = sol.iterations;
    ints[2] = static_cast<std::int64_t>(sol.trace.size());
    for (std::size_t k = 0; k < sol.trace.size() && std::int64_t(k) < trace_cap; ++k) {
      trace[5 * k + 0] = static_cast<double>(sol.trace[k].iter);
      trace[5 * k + 1] = sol.trace[k].r_norm;
      trace[5 * k + 2] = sol.trace[k].s_norm;
      trace[5 * k + 3] = sol.trace[k].rho;
      trace[5 * k + 4] = sol.trace[k].objective;
    }
    const SolverState& st = solver.final_state();
    const std::size_t J = static_cast<std::size_t>(p.layout.total_terminals);
    if (final_p) std::memcpy(final_p, st.p.data(), 8 * J);
    if (final_z) std::memcpy(final_z, st.z.data(), 8 * J);
    if (final_pbar) std::memcpy(final_pbar, st.p_bar.data(), 8 * p.m);
    if (final_price) std::memcpy(final_price, st.price.data(), 8 * p.m);
    if (final_prev_z) std::memcpy(final_prev_z, solver.final_prev_z().data(), 8 * J);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// PmpSolver::cold_state / warm_state then `k` calls of step()
// (solver.hpp:293-318); state arrays in/out when init == 2 (use given
// state), else init 0 = cold, 1 = warm from warm_x0/warm_price/warm_rho.
// rs receives (r, s) of every step (2*k doubles).
int ref_steps(void* h, const double* cfgd, const std::int64_t* cfgi, int init,
              const double* warm_x0, const double* warm_price, double warm_rho,
              std::int64_t k, double* p, double* z, double* pbar, double* price,
              double* rho, std::int64_t* iter, double* rs) {
  try {
    const Problem& prob = static_cast<RefProblem*>(h)->p;
    PmpSolver solver(prob, to_cfg(cfgd, cfgi));
    const std::size_t J = static_cast<std::size_t>(prob.layout.total_terminals);
    SolverState st;
    if (init == 0) {
      st = solver.cold_state();
    } else if (init == 1) {
      WarmStart warm;
      warm.x0.assign(warm_x0, warm_x0 + prob.n);
      if (warm_price) warm.price.assign(warm_price, warm_price + prob.m);
      warm.rho = warm_rho;
      st = solver.warm_state(warm);
    } else {
      st.p.assign(p, p + J);
      st.z.assign(z, z + J);
      st.p_bar.assign(pbar, pbar + prob.m);
      st.price.assign(price, price + prob.m);
      st.rho = *rho;
      st.iter = *iter;
    }
    for (std::int64_t i = 0; i < k; ++i) {
      auto [r, s] = solver.step(st);
      rs[2 * i] = r;
      rs[2 * i + 1] = s;
    }
    std::memcpy(p, st.p.data(), 8 * J);
    std::memcpy(z, st.z.data(), 8 * J);
    std::memcpy(pbar, st.p_bar.data(), 8 * prob.m);
    std::memcpy(price, st.price.data(), 8 * prob.m);
    *rho = st.rho;
    *iter = st.iter;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU baseline: the reference's own per-iteration work, timed.  Runs the
// body of PmpSolver::run's loop (solver.hpp:450-476: the prev-z copy, step,
// termination check, rho update) for `iters` iterations from the cold state
// with `threads` host threads, returning wall seconds of the loop only.
int ref_time_iterations(void* h, const double* cfgd, const std::int64_t* cfgi,
                        std::int64_t iters, double* seconds, double* last_rs) {
  try {
    const Problem& prob = static_cast<RefProblem*>(h)->p;
    SolverConfig cfg = to_cfg(cfgd, cfgi);
    PmpSolver solver(prob, cfg);
    SolverState st = solver.cold_state();
    std::vector<double> prev_z;
    double r = 0.0, s = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (std::int64_t it = 1; it <= iters; ++it) {
      prev_z = st.z;
      auto rs = solver.step(st);
      r = rs.first;
      s = rs.second;
      if (check_termination(r, s, prob.layout, solver.config())) break;
      if (it % cfg.rho_update_interval == 0) update_rho(st, r, s, solver.config());
    }
    *seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    last_rs[0] = r;
    last_rs[1] = s;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// warm.hpp:25-55; before/after handles, prior solution arrays.
int ref_warm_after_degrade(void* before, void* after, const double* prior_x,
                           const double* prior_lambda_raw, double prior_rho_final,
                           double* x0, double* price, double* rho) {
  try {
    const Problem& b = static_cast<RefProblem*>(before)->p;
    const Problem& a = static_cast<RefProblem*>(after)->p;
    Solution prior;
    prior.x.assign(prior_x, prior_x + b.n);
    prior.lambda_raw.assign(prior_lambda_raw, prior_lambda_raw + b.m);
    prior.rho_final = prior_rho_final;
    WarmStart w = warm_start_after_degrade(b, a, prior);
    std::memcpy(x0, w.x0.data(), 8 * a.n);
    std::memcpy(price, w.price.data(), 8 * a.m);
    *rho = w.rho;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// warm.hpp:60-94; `pruned` carries the prune map from ref_fail_and_prune.
int ref_warm_after_prune(void* pruned, const double* prior_x, std::int64_t prior_n,
                         const double* prior_lambda_raw, std::int64_t prior_m,
                         double prior_rho_final, double* x0, double* price,
                         double* rho) {
  try {
    auto* r = static_cast<RefProblem*>(pruned);
    PruneMap map;
    map.link_map = r->prune_link_map;
    map.stream_map = r->prune_stream_map;
    Solution prior;
    prior.x.assign(prior_x, prior_x + prior_n);
    prior.lambda_raw.assign(prior_lambda_raw, prior_lambda_raw + prior_m);
    prior.rho_final = prior_rho_final;
    WarmStart w = warm_start_after_prune(r->p, map, prior);
    std::memcpy(x0, w.x0.data(), 8 * r->p.n);
    std::memcpy(price, w.price.data(), 8 * r->p.m);
    *rho = w.rho;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Persistent CPU-baseline session: one PmpSolver constructed once (as a user
// would), with cfg.max_iters = the sample size; every ref_bench_solve call is
// the stock PmpSolver::solve() (solver.hpp:411 -> cold_state, run 441-508,
// post-processing), timed with steady_clock around solve() only.
struct RefBench {
  PmpSolver solver;
  RefBench(const Problem& p, const SolverConfig& c) : solver(p, c) {}
};

int ref_bench_open(void* h, const double* cfgd, const std::int64_t* cfgi, void** out) {
  try {
    *out = new RefBench(static_cast<RefProblem*>(h)->p, to_cfg(cfgd, cfgi));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ints = {status, iterations}; rs = {r_norm, s_norm}
int ref_bench_solve(void* bh, double* seconds, std::int64_t* ints, double* rs) {
  try {
    auto* b = static_cast<RefBench*>(bh);
    const auto t0 = std::chrono::steady_clock::now();
    const Solution sol = b->solver.solve();
    *seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ints[0] = static_cast<std::int64_t>(sol.status);
    ints[1] = sol.iterations;
    rs[0] = sol.r_norm;
    rs[1] = sol.s_norm;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// group_streams (model.hpp:255-286) flattened: per group tau, kind, member
// count; members concatenated in group order.  Call with null arrays first
// for the sizes.
void ref_groups(void* h, std::int64_t* ngroups, std::int64_t* nmembers, std::int32_t* tau,
                std::int32_t* kind, std::int64_t* count, std::int64_t* members) {
  const auto gs = group_streams(static_cast<RefProblem*>(h)->p);
  *ngroups = static_cast<std::int64_t>(gs.size());
  std::int64_t k = 0;
  for (std::size_t g = 0; g < gs.size(); ++g) {
    if (tau) tau[g] = gs[g].tau;
    if (kind) kind[g] = static_cast<std::int32_t>(gs[g].kind);
    if (count) count[g] = static_cast<std::int64_t>(gs[g].members.size());
    for (std::int64_t j : gs[g].members) {
      if (members) members[k] = j;
      ++k;
    }
  }
  *nmembers = k;
}

void ref_bench_close(void* bh) { delete static_cast<RefBench*>(bh); }

// prox.hpp scalars, for the prox golden vectors.
double ref_prox_log(double z, double w, double rho, std::int64_t tau) {
  return prox_log_scalar(z, w, rho, tau);
}
double ref_prox_linear_nonneg(double z, double w, double rho, std::int64_t tau) {
  return prox_linear_nonneg_scalar(z, w, rho, tau);
}

// TransitMetadata::streams / ods (transit.hpp:35-57)
int ref_transit_meta(void* h, std::int64_t* n_ods, std::int32_t* od, std::int32_t* route,
                     std::int32_t* t0, std::int32_t* origin, std::int32_t* dest) {
  const TransitMetadata& m = static_cast<RefProblem*>(h)->meta;
  *n_ods = static_cast<std::int64_t>(m.ods.size());
  for (std::size_t j = 0; j < m.streams.size(); ++j) {
    if (od) od[j] = m.streams[j].od;
    if (route) route[j] = m.streams[j].route;
    if (t0) t0[j] = m.streams[j].t0;
  }
  for (std::size_t q = 0; q < m.ods.size(); ++q) {
    if (origin) origin[q] = m.ods[q].origin;
    if (dest) dest[q] = m.ods[q].dest;
  }
  return 0;
}

// io.hpp:393-404
int ref_write_trace_csv(const char* path, std::int64_t rows, const std::int64_t* iter,
                        const double* r, const double* s, const double* rho, const double* obj) {
  try {
    ConvergenceTrace t;
    for (std::int64_t i = 0; i < rows; ++i) {
      TraceRecord rec;
      rec.iter = iter[i];
      rec.r_norm = r[i];
      rec.s_norm = s[i];
      rec.rho = rho[i];
      rec.objective = obj[i];
      t.push_back(rec);
    }
    write_trace_csv(t, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// transit.hpp:340-374; the rows flattened (stream, pi, lambda_hat) and the
// CSV the reference CLI writes for them (tools/numpmp.cpp:333-342 formatting)
int ref_transit_report(void* h, const double* x, const double* lam, std::int32_t od, std::int32_t t0,
                       const char* csv_path, std::int64_t* nrows, std::int64_t* stream, double* pi,
                       std::int64_t* hat_len, double* hats, std::int64_t hat_cap) {
  try {
    RefProblem* r = static_cast<RefProblem*>(h);
    std::vector<double> xv(x, x + r->p.n), lv(lam, lam + r->p.m);
    auto rows = transit_report(r->p, xv, lv, r->meta, od, t0);
    *nrows = static_cast<std::int64_t>(rows.size());
    std::int64_t k = 0;
    std::ofstream out(csv_path);
    out << "stream,od,route,t0,x,pi,lambda_hat_path\n";
    for (std::size_t i = 0; i < rows.size(); ++i) {
      const auto& row = rows[i];
      stream[i] = row.stream;
      pi[i] = row.pi;
      hat_len[i] = static_cast<std::int64_t>(row.lambda_hat.size());
      for (double v : row.lambda_hat)
        if (k < hat_cap) hats[k++] = v;
      out << row.stream << ',' << row.od << ',' << row.route << ',' << row.t0 << ',' << row.x << ','
          << row.pi << ',' << '"';
      for (std::size_t q = 0; q < row.lambda_hat.size(); ++q) {
        if (q) out << ' ';
        out << row.lambda_hat[q];
      }
      out << '"' << '\n';
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// io.hpp:444-540
int ref_write_transit_metadata(void* h, const char* path) {
  try {
    write_transit_metadata(static_cast<RefProblem*>(h)->meta, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int ref_check_transit_metadata(const char* path) {  // read_transit_metadata; 0 or the IoError
  try {
    (void)read_transit_metadata(path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
