/*
 * oracle/pmp_oracle.h -- TEST INFRASTRUCTURE ONLY.  C restatement of the
 * reference numpmp engine (see pmp_oracle.c for the file:line map).
 */
#ifndef PMP_ORACLE_H_
#define PMP_ORACLE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The reference Problem + TerminalLayout (model.hpp:47-65) as flat arrays. */
typedef struct {
  int64_t m, n, nnz;
  const double* capacities;     /* m */
  const double* weights;        /* n */
  const uint8_t* kinds;         /* n: 0 = log, 1 = linear (model.hpp:18) */
  const int64_t* stream_offsets;/* n+1 */
  const int32_t* terminal_link; /* J = nnz + m */
  const int64_t* link_offsets;  /* m+1 */
  const int64_t* link_terminals;/* J */
  const int32_t* link_counts;   /* m */
} oracle_problem;

/* SolverConfig (solver.hpp:19-30), threads omitted (results are
 * thread-count invariant, parallel.hpp:54-56). */
typedef struct {
  double eps_abs, rho0, alpha, mu, gamma, time_limit;
  int64_t rho_update_interval, max_iters, trace_every;
} oracle_config;

/* SolverState (solver.hpp:51-62): caller-owned arrays. */
typedef struct {
  double* p;      /* J */
  double* z;      /* J */
  double* p_bar;  /* m */
  double* price;  /* m */
  double rho;
  int64_t iter;
} oracle_state;

typedef struct {
  int64_t iter;
  double r_norm, s_norm, rho, objective;
} oracle_trace_row;

enum { ORACLE_CONVERGED = 0, ORACLE_MAXITERS = 1, ORACLE_TIMELIMIT = 2 };

/* Solution (solver.hpp:85-97): caller-owned arrays x[n], s[m], lambda[m],
 * lambda_raw[m]. */
typedef struct {
  double* x;
  double* s;
  double* lambda;
  double* lambda_raw;
  double objective;
  int32_t status;
  int64_t iterations;
  double r_norm, s_norm, rho_final;
  int64_t trace_len;
} oracle_solution;

int oracle_build_layout(int64_t n, int64_t m, const int64_t* stream_offsets,
                        const int32_t* route_links, int32_t* terminal_link,
                        int64_t* link_offsets, int64_t* link_terminals,
                        int32_t* link_counts);
double oracle_prox_log(double z_sum, double w, double rho, int64_t tau);
double oracle_prox_linear_nonneg(double z_sum, double w, double rho, int64_t tau);
void oracle_link_averages(const oracle_problem* P, const double* p, double* p_bar);
void oracle_step(const oracle_problem* P, const oracle_config* cfg,
                 oracle_state* st, double* u_buf, double* x_out, double* r_norm,
                 double* s_norm);
double oracle_objective(const oracle_problem* P, const double* x);
int oracle_warm_state(const oracle_problem* P, const oracle_config* cfg,
                      const double* x0, const double* price0, double rho,
                      oracle_state* st, char* err, int errlen);
int oracle_run(const oracle_problem* P, const oracle_config* cfg,
               oracle_state* st, double* prev_z, oracle_solution* sol,
               oracle_trace_row* trace, int64_t trace_cap, char* err, int errlen);
void oracle_plain_step(const oracle_problem* P, double rho, double* p, double* u,
                       double* p_bar, double* arg);

#ifdef __cplusplus
}
#endif
#endif
