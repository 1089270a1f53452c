/*
 * oracle/pmp_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference numpmp PMP engine in its native
 * terminal space, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker.  It is never linked into, called by, or
 * shipped with the product path (paper_2509_10722_b200/).
 *
 * Everything below follows the reference operation-for-operation so that
 * results are bit-identical to the reference compiled without -march
 * (no FMA contraction; build with -ffp-contract=off):
 *   build_layout          model.hpp:159-201
 *   prox_log_scalar       prox.hpp:31-40
 *   prox_linear_nonneg    prox.hpp:44-56
 *   deterministic_sum     parallel.hpp:57-76 (8192-wide chunks, in order)
 *   compute_link_averages solver.hpp:110-126
 *   PmpSolver::step       solver.hpp:318-409
 *   PmpSolver::run        solver.hpp:441-508
 *   check_termination     solver.hpp:157-163
 *   update_rho            solver.hpp:168-174
 *   current_objective     solver.hpp:420-439
 *   warm_start_from       solver.hpp:218-259 (+ warm_state 305-314)
 *
 * Parity is pinned: tests/test_oracle.py checks this file against the
 * reference itself (oracle/_ref, compiled from /root/reference headers by
 * oracle/Makefile) and against the golden vectors of the reference's own
 * GoogleTest suites (tests/golden/).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "pmp_oracle.h"

#define KREDUCE_CHUNK 8192 /* parallel.hpp:57 */

static void set_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    strncpy(err, msg, (size_t)errlen - 1);
    err[errlen - 1] = 0;
  }
}

/* model.hpp:159-201 -- terminals stream-major, then one slack per link;
 * link-major CSR built by a counting sort so each link's terminals are in
 * ascending terminal order with the slack last. */
int oracle_build_layout(int64_t n, int64_t m, const int64_t* stream_offsets,
                        const int32_t* route_links, int32_t* terminal_link,
                        int64_t* link_offsets, int64_t* link_terminals,
                        int32_t* link_counts) {
  const int64_t nnz = stream_offsets[n];
  const int64_t J = nnz + m;
  for (int64_t t = 0; t < nnz; ++t) terminal_link[t] = route_links[t];
  for (int64_t l = 0; l < m; ++l) terminal_link[nnz + l] = (int32_t)l;
  for (int64_t l = 0; l < m; ++l) link_counts[l] = 0;
  for (int64_t t = 0; t < J; ++t) ++link_counts[terminal_link[t]];
  link_offsets[0] = 0;
  for (int64_t l = 0; l < m; ++l)
    link_offsets[l + 1] = link_offsets[l] + link_counts[l];
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  if (!cursor) return -1;
  for (int64_t l = 0; l < m; ++l) cursor[l] = link_offsets[l];
  for (int64_t t = 0; t < J; ++t) link_terminals[cursor[terminal_link[t]]++] = t;
  free(cursor);
  return 0;
}

/* prox.hpp:31-40 */
double oracle_prox_log(double z_sum, double w, double rho, int64_t tau) {
  const double d = 4.0 * w * (double)tau / rho;
  if (z_sum >= 0.0)
    return (z_sum + sqrt(z_sum * z_sum + d)) / (2.0 * (double)tau);
  return d / (2.0 * (double)tau * (sqrt(z_sum * z_sum + d) - z_sum));
}

/* prox.hpp:44-56 (prox_linear_scalar, then the clamp of the nonneg variant) */
double oracle_prox_linear_nonneg(double z_sum, double w, double rho,
                                 int64_t tau) {
  const double x = (z_sum + w / rho) / (double)tau;
  return (x < 0.0) ? 0.0 : x; /* std::max(x, 0.0), NaN and -0.0 kept */
}

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* solver.hpp:110-126 */
void oracle_link_averages(const oracle_problem* P, const double* p,
                          double* p_bar) {
  for (int64_t l = 0; l < P->m; ++l) {
    double acc = 0.0;
    for (int64_t k = P->link_offsets[l]; k < P->link_offsets[l + 1]; ++k)
      acc += p[P->link_terminals[k]];
    p_bar[l] = acc / P->link_counts[l];
  }
}

/* solver.hpp:318-409; x_out (length n) receives the stream rates (x_buf_). */
void oracle_step(const oracle_problem* P, const oracle_config* cfg,
                 oracle_state* st, double* u_buf, double* x_out, double* r_norm,
                 double* s_norm) {
  const int64_t m = P->m, n = P->n, nnz = P->nnz, J = nnz + m;
  const double rho = st->rho;
  const double alpha = cfg->alpha;
  for (int64_t l = 0; l < m; ++l) u_buf[l] = st->price[l] / rho;

  /* Stream prox updates (solver.hpp:332-366).  Each stream writes only its
   * own terminals, so the type-group order does not affect results. */
  for (int64_t j = 0; j < n; ++j) {
    const int64_t off = P->stream_offsets[j];
    const int64_t tau = P->stream_offsets[j + 1] - off;
    double z_sum = 0.0;
    for (int64_t i = 0; i < tau; ++i) {
      const int64_t t = off + i;
      z_sum += st->z[t] - u_buf[P->terminal_link[t]];
    }
    const double w = P->weights[j];
    double x = (P->kinds[j] == 0) ? oracle_prox_log(z_sum, w, rho, tau)
                                  : oracle_prox_linear_nonneg(z_sum, w, rho, tau);
    x_out[j] = x;
    for (int64_t i = 0; i < tau; ++i) st->p[off + i] = x;
  }
  /* slack projection (solver.hpp:368-376) */
  for (int64_t l = 0; l < m; ++l) {
    const int64_t t = nnz + l;
    const double v = st->z[t] - u_buf[l];
    st->p[t] = dmax(v, -P->capacities[l]);
  }
  oracle_link_averages(P, st->p, st->p_bar);

  /* r^2 = deterministic_sum over m (solver.hpp:379-384, parallel.hpp:57-76) */
  double r2 = 0.0;
  for (int64_t c0 = 0; c0 < m; c0 += KREDUCE_CHUNK) {
    const int64_t c1 = c0 + KREDUCE_CHUNK < m ? c0 + KREDUCE_CHUNK : m;
    double acc = 0.0;
    for (int64_t l = c0; l < c1; ++l) {
      const double v = st->p_bar[l];
      acc += (double)P->link_counts[l] * v * v;
    }
    r2 += acc;
  }
  /* z update + s^2 (solver.hpp:388-399) */
  double s2 = 0.0;
  for (int64_t c0 = 0; c0 < J; c0 += KREDUCE_CHUNK) {
    const int64_t c1 = c0 + KREDUCE_CHUNK < J ? c0 + KREDUCE_CHUNK : J;
    double acc = 0.0;
    for (int64_t t = c0; t < c1; ++t) {
      const double z_old = st->z[t];
      const double z_new =
          alpha * (st->p[t] - st->p_bar[P->terminal_link[t]]) + (1.0 - alpha) * z_old;
      st->z[t] = z_new;
      const double d = rho * (z_new - z_old);
      acc += d * d;
    }
    s2 += acc;
  }
  /* price update (solver.hpp:401-405) */
  for (int64_t l = 0; l < m; ++l) st->price[l] += rho * (alpha * st->p_bar[l]);
  st->iter += 1;
  *r_norm = sqrt(r2);
  *s_norm = sqrt(s2);
}

/* solver.hpp:420-439 (log / linear only; extension utilities are out of scope) */
double oracle_objective(const oracle_problem* P, const double* x) {
  double total = 0.0;
  for (int64_t j = 0; j < P->n; ++j) {
    if (P->kinds[j] == 0)
      total += P->weights[j] * log(x[j]);
    else
      total += P->weights[j] * x[j];
  }
  return total;
}

/* solver.hpp:218-259 + 305-314. Returns 0, or 1 (invalid_argument) /
 * 4 (domain_error) with a message. */
int oracle_warm_state(const oracle_problem* P, const oracle_config* cfg,
                      const double* x0, const double* price0, double rho,
                      oracle_state* st, char* err, int errlen) {
  const int64_t m = P->m, n = P->n, nnz = P->nnz, J = nnz + m;
  for (int64_t j = 0; j < n; ++j)
    if (P->kinds[j] == 0 && !(x0[j] > 0.0)) {
      char buf[128];
      snprintf(buf, sizeof buf, "warm start: log stream %lld needs a positive rate",
               (long long)j);
      set_err(err, errlen, buf);
      return 4;
    }
  st->rho = rho > 0.0 ? rho : cfg->rho0;
  st->iter = 0;
  double* load = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  for (int64_t j = 0; j < n; ++j) {
    const double xj = x0[j];
    for (int64_t t = P->stream_offsets[j]; t < P->stream_offsets[j + 1]; ++t) {
      st->p[t] = xj;
      load[P->terminal_link[t]] += xj;
    }
  }
  for (int64_t l = 0; l < m; ++l) {
    const double slack = dmax(P->capacities[l] - load[l], 0.0);
    st->p[nnz + l] = slack - P->capacities[l];
  }
  free(load);
  oracle_link_averages(P, st->p, st->p_bar);
  for (int64_t t = 0; t < J; ++t) st->z[t] = st->p[t] - st->p_bar[P->terminal_link[t]];
  for (int64_t l = 0; l < m; ++l) st->price[l] = price0 ? price0[l] : 0.0;
  return 0;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* solver.hpp:441-508.  st holds the start state (cold or warm) on entry and
 * the final state on exit; prev_z (nullable, length J) receives
 * final_prev_z_.  Returns 0 or 3 (SolverError, message in err). */
int oracle_run(const oracle_problem* P, const oracle_config* cfg,
               oracle_state* st, double* prev_z, oracle_solution* sol,
               oracle_trace_row* trace, int64_t trace_cap, char* err,
               int errlen) {
  const int64_t m = P->m, n = P->n, J = P->nnz + m;
  const double start = now_seconds();
  double* u_buf = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double* x_buf = sol->x; /* x_buf_, clamped in place at the end */
  for (int64_t j = 0; j < n; ++j) x_buf[j] = 0.0;
  sol->status = ORACLE_MAXITERS;
  sol->trace_len = 0;
  double r_norm = 0.0, s_norm = 0.0;
  const double eps_tol = cfg->eps_abs * sqrt((double)J);
  int rc = 0;
  for (int64_t iter = 1; iter <= cfg->max_iters; ++iter) {
    if (prev_z) memcpy(prev_z, st->z, sizeof(double) * (size_t)J);
    oracle_step(P, cfg, st, u_buf, x_buf, &r_norm, &s_norm);
    if (!isfinite(r_norm) || !isfinite(s_norm)) {
      char buf[96];
      snprintf(buf, sizeof buf, "non-finite state at iteration %lld", (long long)iter);
      set_err(err, errlen, buf);
      rc = 3;
      goto done;
    }
    if (r_norm < eps_tol && s_norm < eps_tol) {
      sol->status = ORACLE_CONVERGED;
      break;
    }
    if (iter % cfg->trace_every == 0 && sol->trace_len < trace_cap) {
      oracle_trace_row* row = &trace[sol->trace_len++];
      row->iter = iter;
      row->r_norm = r_norm;
      row->s_norm = s_norm;
      row->rho = st->rho;
      row->objective = oracle_objective(P, x_buf);
    }
    if (cfg->time_limit > 0.0 && now_seconds() - start > cfg->time_limit) {
      sol->status = ORACLE_TIMELIMIT;
      break;
    }
    if (iter % cfg->rho_update_interval == 0) {
      if (r_norm > cfg->mu * s_norm)
        st->rho *= cfg->gamma;
      else if (s_norm > cfg->mu * r_norm)
        st->rho /= cfg->gamma;
    }
  }
  if ((sol->trace_len == 0 || trace[sol->trace_len - 1].iter != st->iter) &&
      sol->trace_len < trace_cap) {
    oracle_trace_row* row = &trace[sol->trace_len++];
    row->iter = st->iter;
    row->r_norm = r_norm;
    row->s_norm = s_norm;
    row->rho = st->rho;
    row->objective = oracle_objective(P, x_buf);
  }
  sol->iterations = st->iter;
  sol->r_norm = r_norm;
  sol->s_norm = s_norm;
  sol->rho_final = st->rho;
  for (int64_t j = 0; j < n; ++j)
    if (x_buf[j] < 0.0 && -x_buf[j] < cfg->eps_abs) x_buf[j] = 0.0;
  {
    double* load = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    for (int64_t j = 0; j < n; ++j)
      for (int64_t t = P->stream_offsets[j]; t < P->stream_offsets[j + 1]; ++t)
        load[P->terminal_link[t]] += x_buf[j];
    for (int64_t l = 0; l < m; ++l) sol->s[l] = dmax(P->capacities[l] - load[l], 0.0);
    free(load);
  }
  for (int64_t l = 0; l < m; ++l) {
    sol->lambda[l] = dmax(st->price[l], 0.0);
    sol->lambda_raw[l] = st->price[l];
  }
  sol->objective = oracle_objective(P, x_buf);
done:
  free(u_buf);
  return rc;
}

/* Plain per-terminal recursion of test_solver.cpp:25-60 / acceptance.cpp
 * criterion 7 (alpha = 1, fixed rho): p <- prox(p - pbar - u), u += pbar.
 * Used to pin the alpha = 1 reduction. */
void oracle_plain_step(const oracle_problem* P, double rho, double* p, double* u,
                       double* p_bar, double* arg) {
  const int64_t m = P->m, n = P->n, nnz = P->nnz, J = nnz + m;
  for (int64_t t = 0; t < J; ++t) arg[t] = p[t] - p_bar[P->terminal_link[t]] - u[t];
  for (int64_t j = 0; j < n; ++j) {
    const int64_t off = P->stream_offsets[j];
    const int64_t tau = P->stream_offsets[j + 1] - off;
    double z_sum = 0.0;
    for (int64_t i = 0; i < tau; ++i) z_sum += arg[off + i];
    const double x = (P->kinds[j] == 0)
                         ? oracle_prox_log(z_sum, P->weights[j], rho, tau)
                         : oracle_prox_linear_nonneg(z_sum, P->weights[j], rho, tau);
    for (int64_t i = 0; i < tau; ++i) p[off + i] = x;
  }
  for (int64_t l = 0; l < m; ++l) p[nnz + l] = dmax(arg[nnz + l], -P->capacities[l]);
  oracle_link_averages(P, p, p_bar);
  for (int64_t t = 0; t < J; ++t) u[t] += p_bar[P->terminal_link[t]];
}
