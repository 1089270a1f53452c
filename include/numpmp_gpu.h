/*
 * numpmp_gpu.h -- C-ABI of libnumpmp_cuda.so, the B200 (sm_100a) PMP/ADMM
 * engine that replaces the reference's CPU PmpSolver hot path.
 *
 * The reference (numpmp, header-only C++20) has no C-ABI; its boundary is
 * the C++ class numpmp::PmpSolver (proj/include/numpmp/solver.hpp:265-519).
 * Each entry point below replaces one member of that class; the header-only
 * C++ drop-in include/numpmp/gpu_solver.hpp wraps them back into the
 * reference's own signatures and exception types.
 *
 * Conventions: plain pointers and sizes, caller-owned host buffers, no
 * torch/CUDA types.  A handle copies the problem to the device at create and
 * never keeps host pointers.  A handle is not thread-safe (one owner, as the
 * reference's PmpSolver, solver.hpp:510-518).  Every function returns a
 * numpmp_status code; the message of the last failure is available from
 * numpmp_gpu_last_error().
 */
#ifndef NUMPMP_GPU_H_
#define NUMPMP_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes, 1:1 with the reference's exception types (common.hpp:11-43,
 * solver.hpp:32-44, 218-227). */
typedef enum {
  NUMPMP_OK = 0,
  NUMPMP_INVALID_ARGUMENT = 1, /* std::invalid_argument               */
  NUMPMP_VALIDATION_ERROR = 2, /* numpmp::ValidationError             */
  NUMPMP_SOLVER_ERROR = 3,     /* numpmp::SolverError (non-finite ...)*/
  NUMPMP_DOMAIN_ERROR = 4,     /* std::domain_error                   */
  NUMPMP_CUDA_ERROR = 10,
  NUMPMP_NCCL_ERROR = 11
} numpmp_status;

/* SolveStatus (solver.hpp:74). */
enum { NUMPMP_CONVERGED = 0, NUMPMP_MAXITERS = 1, NUMPMP_TIMELIMIT = 2 };

/* StreamKind (model.hpp:18).  Extension utilities are rejected with
 * NUMPMP_SOLVER_ERROR: their prox is a host std::function callback
 * (prox.hpp:61-67) that cannot run in a kernel. */
enum { NUMPMP_KIND_LOG = 0, NUMPMP_KIND_LINEAR = 1, NUMPMP_KIND_EXTENSION = 2 };

/* Problem + TerminalLayout view (model.hpp:32-65).  route_links is the
 * stream-major incidence, i.e. TerminalLayout::terminal_link[0:nnz)
 * (model.hpp:51, 171-177), stream_offsets is TerminalLayout::stream_offsets
 * (model.hpp:50).  The link-major CSR (link_offsets / link_terminals,
 * model.hpp:52-54, 187-199) is built on the device. */
typedef struct {
  int64_t m;                     /* links                       */
  int64_t n;                     /* traffic streams             */
  int64_t nnz;                   /* = stream_offsets[n]         */
  const double* capacities;      /* m                           */
  const double* weights;         /* n                           */
  const uint8_t* kinds;          /* n  (NUMPMP_KIND_*)          */
  const int64_t* stream_offsets; /* n+1                         */
  const int32_t* route_links;    /* nnz                         */
} numpmp_problem_view;

/* SolverConfig (solver.hpp:19-30).  threads has no GPU meaning and is
 * validated only. */
typedef struct {
  double eps_abs;
  double rho0;
  double alpha;
  double mu;
  double gamma;
  double time_limit; /* wall seconds on the device clock; 0 disables */
  int64_t rho_update_interval;
  int64_t max_iters;
  int64_t trace_every;
  int32_t threads;
  int32_t _pad;
} numpmp_config;

/* TraceRecord (solver.hpp:64-70). */
typedef struct {
  int64_t iter;
  double r_norm;
  double s_norm;
  double rho;
  double objective;
} numpmp_trace_row;

/* Solution scalars (solver.hpp:85-97); the vectors are separate outputs. */
typedef struct {
  double objective;
  double r_norm;
  double s_norm;
  double rho_final;
  int64_t iterations;
  int32_t status; /* NUMPMP_CONVERGED / MAXITERS / TIMELIMIT */
  int32_t _pad;
  int64_t trace_len;
} numpmp_solution_info;

typedef struct numpmp_gpu numpmp_gpu; /* opaque; one per solver object */

/* Replaces PmpSolver::PmpSolver (solver.hpp:267-287): validate_config
 * (solver.hpp:32-44 -> NUMPMP_INVALID_ARGUMENT), validate (model.hpp:76-155
 * -> NUMPMP_VALIDATION_ERROR), extension streams -> NUMPMP_SOLVER_ERROR.
 * Uploads the problem to `device` and builds the link-major CSR there. */
int numpmp_gpu_create(const numpmp_problem_view* problem, const numpmp_config* config,
                      int device, numpmp_gpu** out);

/* Sharded variant for one process per GPU (multi-GPU):
 * the view holds this rank's contiguous stream range [stream_begin,
 * stream_begin + view->n) of a problem with `n_total` streams; link state
 * is replicated and the per-link partial loads are summed with an NCCL
 * all-reduce over NVLink.  nccl_id is the 128-byte ncclUniqueId produced by
 * numpmp_gpu_nccl_unique_id on rank 0 and broadcast by the caller. */
int numpmp_gpu_create_sharded(const numpmp_problem_view* shard, const numpmp_config* config,
                              int device, int rank, int world, const void* nccl_id,
                              int64_t stream_begin, int64_t n_total, numpmp_gpu** out);
int numpmp_gpu_nccl_unique_id(void* out128);

/* Sharded variant with the fused peer-memory exchange (the default for
 * multi-GPU runs; pmp_p2p.cuh): links are owned in contiguous ranges, the
 * link pass stores every row's partial load straight into the owner's HBM
 * over NVLink, each owner runs the link epilogue for its links and stores
 * v into every rank's HBM; two system-scope barriers per iteration, no
 * NCCL kernel in the loop.  Setup, all collective over the ranks:
 *   numpmp_gpu_create_p2p  -> numpmp_gpu_p2p_export (64-byte CUDA IPC
 *   handle of the exchange region; the caller all-gathers them) ->
 *   numpmp_gpu_p2p_connect (rank-ordered world x 64 bytes) ->
 *   numpmp_gpu_p2p_start (global link degrees / nnz through the exchange).
 * numpmp_gpu_p2p_connect_local wires `world` handles of one process instead
 * (one GPU, or several with peer access); each handle must then be driven
 * by its own host thread, as each rank by its own process.
 * Every later call that runs iterations or collectives (set_warm, step,
 * run, run_device) is collective too. */
int numpmp_gpu_create_p2p(const numpmp_problem_view* shard, const numpmp_config* config,
                          int device, int rank, int world, int64_t stream_begin, int64_t n_total,
                          numpmp_gpu** out);
int numpmp_gpu_p2p_export(numpmp_gpu* h, void* out64);
int numpmp_gpu_p2p_connect(numpmp_gpu* h, const void* handles);
int numpmp_gpu_p2p_connect_local(numpmp_gpu** handles, int world);
int numpmp_gpu_p2p_start(numpmp_gpu* h);

/* Replaces PmpSolver::cold_state (solver.hpp:293-303). */
int numpmp_gpu_set_cold(numpmp_gpu* h);

/* Replaces PmpSolver::warm_state + warm_start_from (solver.hpp:218-259,
 * 305-314).  price may be null (zero prices); rho <= 0 selects rho0.
 * x0 length n, price length m; log streams need x0 > 0 (NUMPMP_DOMAIN_ERROR). */
int numpmp_gpu_set_warm(numpmp_gpu* h, const double* x0, const double* price, double rho);

/* Warm-start recipes of warm.hpp computed on the device and applied with
 * warm_start_from (solver.hpp:218-259) without a host round trip.
 * numpmp_gpu_warm_after_degrade replaces warm_start_after_degrade
 * (warm.hpp:25-57): the handle holds the degraded problem; cap_before[m] is
 * the prior problem's capacities, prior_x[n] / prior_lambda_raw[m] /
 * prior_rho the prior Solution.  numpmp_gpu_warm_after_prune replaces
 * warm_start_after_prune (warm.hpp:62-94): the handle holds the pruned
 * problem; x0_proj[n] / price_proj[m] are the prior x and lambda_raw already
 * projected with PruneMap::project_streams / project_links (gen.hpp:146-178).
 * The optional outputs return the recipe's WarmStart (x0, price, rho). */
int numpmp_gpu_warm_after_degrade(numpmp_gpu* h, const double* cap_before, const double* prior_x,
                                  const double* prior_lambda_raw, double prior_rho, double* x0_out,
                                  double* price_out, double* rho_out);
int numpmp_gpu_warm_after_prune(numpmp_gpu* h, const double* x0_proj, const double* price_proj,
                                double prior_rho, double* x0_out, double* price_out, double* rho_out);

/* Replaces path_prices (transit.hpp:290-302): pi[n] = sum of lambda[m]
 * along each stream's route, in route order. */
int numpmp_gpu_path_prices(numpmp_gpu* h, const double* lambda, double* pi);

/* Loads an arbitrary reference SolverState (solver.hpp:51-62): p, z of
 * length J = nnz + m, p_bar and price of length m.  z must decompose as
 * z_t = A_j - B_l over the incidence (every cold, warm and stepped state
 * does); otherwise NUMPMP_INVALID_ARGUMENT.  The state the handle issued
 * last through numpmp_gpu_get_state (all four arrays), with nothing run
 * since, is recognised by a fingerprint and kept as is: no host
 * decomposition, no upload, and the device state stays bit-identical. */
int numpmp_gpu_set_state(numpmp_gpu* h, const double* p, const double* z, const double* p_bar,
                         const double* price, double rho, int64_t iter);

/* Materialises the current state in the reference's terminal space.  Any
 * output may be null.  prev_z (length J) is final_prev_z() of solver.hpp:417. */
int numpmp_gpu_get_state(numpmp_gpu* h, double* p, double* z, double* p_bar, double* price,
                         double* rho, int64_t* iter, double* prev_z);

/* Replaces PmpSolver::step (solver.hpp:316-409): one iteration with no
 * termination test, trace or rho balancing; returns (r_norm, s_norm) of
 * residuals(after, before) -- on single-device handles computed by exactly
 * the reduction numpmp_gpu_residuals runs, so the two agree bit for bit on
 * the states get_state returns (solver.hpp:316-318, test_solver.cpp:245-262).
 * A run's `done` flag is cleared first (step after run iterates). */
int numpmp_gpu_step(numpmp_gpu* h, double* r_norm, double* s_norm);

/* Replaces the free function residuals(state, prev, layout)
 * (solver.hpp:139-154): r = sqrt(sum_l |l| p_bar_l^2), s = sqrt(sum_t
 * (rho (z_t - prev_z_t))^2) over the handle's layout, as a fixed-order device
 * reduction.  p_bar[m], z[J], prev_z[J]; rho is the after-state's rho.
 * Single-device handles only. */
int numpmp_gpu_residuals(numpmp_gpu* h, const double* p_bar, const double* z, const double* prev_z,
                         double rho, double* r_norm, double* s_norm);

/* Replaces PmpSolver::run (solver.hpp:441-508) from the current state
 * (call set_cold / set_warm first; solve() == set_cold + run).  x[n],
 * s[m], lambda[m], lambda_raw[m] may be null; trace may be null. */
int numpmp_gpu_run(numpmp_gpu* h, double* x, double* s, double* lambda, double* lambda_raw,
                   numpmp_solution_info* info, numpmp_trace_row* trace, int64_t trace_cap);

/* Device-resident loop only (benchmarking): runs from the current state
 * and leaves the solution on the device; returns the iterations run and
 * the status. */
int numpmp_gpu_run_device(numpmp_gpu* h, numpmp_solution_info* info);

/* Layout export in the reference's TerminalLayout format (model.hpp:47-57),
 * rebuilt from the device CSR, for bit-exact parity checks.  Arrays:
 * link_offsets[m+1], link_terminals[J], link_counts[m]. */
int numpmp_gpu_export_layout(numpmp_gpu* h, int64_t* link_offsets, int64_t* link_terminals,
                             int32_t* link_counts);

/* Sizes of the handle's problem (this rank's shard for sharded handles). */
int numpmp_gpu_sizes(const numpmp_gpu* h, int64_t* m, int64_t* n, int64_t* nnz);

/* Kernel-level measurements of the last run: number of kernel launches
 * and accumulated device milliseconds per kernel class (events on the
 * launching stream; enabled by numpmp_gpu_set_profiling). */
int numpmp_gpu_set_profiling(numpmp_gpu* h, int enable);
int numpmp_gpu_profile(const numpmp_gpu* h, int64_t* launches, double* ms_stream_pass,
                       double* ms_link_pass, int64_t* iterations_timed);

/* Bytes moved host<->device since create (for e2e accounting). */
int numpmp_gpu_transfer_bytes(const numpmp_gpu* h, int64_t* h2d, int64_t* d2h);

/* Device time of the last run / run_device: CUDA events recorded on the
 * handle's stream before the first and after the last iteration batch. */
int numpmp_gpu_last_run_ms(const numpmp_gpu* h, double* ms);

/* Page-lock (cudaHostRegister) a caller buffer so problem uploads and
 * solution downloads run at full PCIe bandwidth; unpin before freeing. */
int numpmp_gpu_pin_host(void* ptr, int64_t bytes);
int numpmp_gpu_unpin_host(void* ptr);

const char* numpmp_gpu_last_error(const numpmp_gpu* h); /* h may be null */
void numpmp_gpu_destroy(numpmp_gpu* h);

#ifdef __cplusplus
}
#endif
#endif /* NUMPMP_GPU_H_ */
