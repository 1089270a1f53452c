// pmp_kernels.cuh -- sm_100a kernels of the PMP/ADMM iteration.
//
// State layout (verified restatement of
// solver.hpp:318-409).  The reference keeps the copies z in terminal space
// (one per nonzero of R plus one per link).  Every reachable state has
// z_t = A_j - B_l for the traffic terminal t = (l, j) and z_{s(l)} = zs_l
// for the slack terminal, and the iteration preserves that form, so the
// device keeps only stream-space (A, x) and link-space (B, zs, price, Q, v)
// vectors:
//
//   v_l    = B_l + price_l / rho                       (link epilogue)
//   zeta_j = tau_j A_j - sum_{l in route(j)} v_l        (stream pass, route order)
//   x_j    = prox(zeta_j)                 (prox.hpp:31-56, IEEE sqrt/div)
//   A_j   <- alpha x_j + (1 - alpha) A_j
//   ps_l   = max(zs_l - price_l/rho, -c_l)             (link epilogue)
//   L_l    = sum_{j in link l} x_j        (ascending stream id)
//   pbar_l = (L_l + ps_l) / (d_l + 1)
//   B_l   <- alpha pbar_l + (1 - alpha) B_l
//   zs_l  <- alpha (ps_l - pbar_l) + (1 - alpha) zs_l
//   price_l += rho (alpha pbar_l)
//   r^2 = sum_l (d_l + 1) pbar_l^2
//   s^2 = rho^2 [ sum_j tau_j dA_j^2 - 2 sum_l dB_l (R dA)_l
//                 + sum_l d_l dB_l^2 + sum_l dzs_l^2 ]
//
// (R dA)_l is tracked without a second gather: Q_l = (R A)_l is kept as link
// state, Q <- alpha L + (1 - alpha) Q, so (R dA)_l = Q_new - Q_old.  The
// tracking error is damped by |1 - alpha| <= 1 every iteration.
//
// Both passes are bound by random 8-byte gathers (one per nonzero and
// direction), i.e. by the L1TEX wavefront rate, not by HBM bytes.  The
// gather core therefore stages only the 32-bit *indices* of a warp's span in
// shared memory (coalesced 128-bit loads, conflict-free 128-bit stores) and
// lets every lane gather and sum its own segment in registers, in index
// order.  Column blocks: the streams are split into NB contiguous blocks;
// the stream pass over block b is followed immediately by the link-pass
// gather over block b's CSR, so the just-written x_b is still L2-resident.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "numpmp_gpu.h"

namespace numpmp_dev {

// Tuning knobs (overridable at build time for sweeps, scripts/variants.sh).
#ifndef NUMPMP_WARPS
#define NUMPMP_WARPS 8
#endif
#ifndef NUMPMP_MIN_BLOCKS
#define NUMPMP_MIN_BLOCKS 4
#endif
#ifndef NUMPMP_STAGE_INTS
#define NUMPMP_STAGE_INTS 512
#endif
#ifndef NUMPMP_GATHER_UNROLL
#define NUMPMP_GATHER_UNROLL 8
#endif
constexpr int kWarps = NUMPMP_WARPS;  // warps per block (gather passes)
constexpr int kThreads = kWarps * 32;
constexpr int kMinBlocks = NUMPMP_MIN_BLOCKS;  // resident blocks per SM the passes are built for
constexpr int kStageInts = NUMPMP_STAGE_INTS;  // staged indices per warp and round
constexpr int kUnroll = NUMPMP_GATHER_UNROLL;  // gathers in flight per lane
// Multi-route stream tiles (short routes, 64-128 streams per warp: spans of
// ~200 indices at config E) stage rounds of 256: half the shared memory,
// more L1 for the gathered v, which consecutive transit tiles reuse
// (E: K1 -5.5%, profiles/r2_stage_ints_ab.txt)
#ifndef NUMPMP_STAGE_Q
#define NUMPMP_STAGE_Q 256
#endif
constexpr int kStageQ = NUMPMP_STAGE_Q;
constexpr int kSeg = kStageInts / 32;          // target entries per link segment (one staged round per warp)
constexpr int kSplitMin = 32 * kSeg;           // rows longer than this are split into pieces
#ifndef NUMPMP_PIECE_ROUNDS
#define NUMPMP_PIECE_ROUNDS 8
#endif
constexpr int kPiece = NUMPMP_PIECE_ROUNDS * kStageInts;  // entries per split-row piece
constexpr int kMaxBlocks = 16;                 // max column blocks
constexpr unsigned kFull = 0xffffffffu;

enum : int { ST_RUNNING = -1, ST_CONVERGED = 0, ST_MAXITERS = 1, ST_TIMELIMIT = 2,
             ST_NONFINITE = 3 };
// MODE_AUX: a link-pass gather outside the iteration (warm start, state
// materialisation, post-processing) -- ignores the `done` flag.
enum : int { MODE_RUN = 0, MODE_STEP = 1, MODE_AUX = 2 };

// Device-resident control block: the run loop of solver.hpp:450-476 lives
// here, written only by the last block of the link pass.
struct Ctrl {
  double rho;        // rho for the next iteration
  double rho_iter;   // rho used by the last completed iteration
  double r_norm;
  double s_norm;
  long long iter;    // SolverState::iter
  long long run_k;   // iteration counter of the current run (1-based)
  long long trace_len;
  long long t0_ns;   // %globaltimer at the start of the run
  int done;          // 1: every later kernel of the batch exits at entry
  int status;        // ST_*
  int rho_changed;   // next stream pass recomputes v = B + price / rho
  unsigned ticket;   // last-block detection, link pass
  unsigned ticket2;  // last-block detection, sharded gather pass
  unsigned ticket3;  // last-block detection, peer-memory owner epilogue
  int v_sel;         // v of the next iteration: 0 v, 1 v_alt[0] (rho*gamma), 2 v_alt[1] (rho/gamma)
};

// Peer-memory exchange of the sharded engine (pmp_p2p.cuh).  Links are
// owned by ranks in contiguous ranges of mo links; every rank maps the
// exchange regions of all ranks (CUDA IPC / same process), so a kernel
// stores straight into a peer's HBM over NVLink.
constexpr int kMaxRanks = 8;
struct P2PArgs {
  int rank, world;   // world == 0: not connected
  int cta_sysfence;  // 1: system-scope fence in every CTA before its ticket (A/B; 0: gpu scope, see k_link_pass)
  long long mo;      // links per owner (ceil(m / world)); owner(l) = l / mo
  long long l0, l1;  // this rank's links
  // device-resident tables of `world` peer pointers (index = rank q)
  double* const* slots_peer;              // rank q's slots: [world][mo] doubles
  double* const* v_peer;                  // rank q's v: m doubles
  double* const* xs_peer;                 // rank q's scalar slots: [world][8] doubles
  unsigned long long* const* flags_peer;  // rank q's barrier counters [4]
  unsigned long long* flags;                 // local barrier counters [4]
  unsigned long long* done_cnt;              // local completed-barrier counts [4]
  double* ep_part;                           // [grid3][4]: owner-epilogue residual partials
};

struct IterArgs {
  // stream side (CSC of R)
  const int* col_ptr;         // n+1
  const int* row_idx;         // nnz (+pad), link of each terminal in route order
  const double* w;            // n
  const unsigned char* kind;  // n
  const int* deg;             // m, link degree (global)
  const double* cap;          // m
  long long n, m;
  // config
  double alpha, eps_tol, mu, gamma;
  long long rho_interval, trace_every, max_iters, time_limit_ns;
  int mode;
  // state, ping-pong: *_in is the current iterate, *_out the next
  const double* A_in;
  double* A_out;
  double* x;
  const double* B_in;
  double* B_out;
  const double* zs_in;
  double* zs_out;
  const double* pr_in;
  double* pr_out;
  const double* Q_in;
  double* Q_out;
  double* v;
  // On rho-update iterations (k % rho_update_interval == 0) the link
  // epilogue also writes v for both candidate rhos; finalize_iteration
  // selects one (Ctrl::v_sel), so no pass rebuilds v after a rho change.
  double* v_alt[2];
  double* k1_part;  // [nb][grid1][2]: tau dA^2, objective
  double* k2_part;  // [grid2][4]: r^2, dB.dQ, d dB^2, dzs^2
  int grid1, grid2, grid3, nblocks;
  double* Lacc;     // m: link loads accumulated over the column blocks
  double* Lbuf;     // sharded: m partial loads + 2 scalars
  Ctrl* ctrl;
  numpmp_trace_row* trace;
  long long trace_cap;
  P2PArgs p2p;
};

// One column block: streams [s0, s1), the CSR of their columns, and its
// segmentation into segments of at most `seg` consecutive entries of one
// link (rows split evenly), packed into warp units of <= 32 segments of
// whole rows (k_link_pass), so every lane's gather chain is bounded
// whatever the link degree skew.
struct BlockArgs {
  long long s0, s1;
  const int* col_idx;  // global stream ids, ascending per row
  const int* vptr;     // nv+1: first CSR entry of each segment
  const int* vrow;     // nv: link of each segment
  const int2* units;   // nu: segment range [x, y) of each warp unit (whole rows)
  long long nv, nu;
  int index;           // block number b
  int first;           // b == 0
  // row mode (blocks whose longest row is short, e.g. more links than
  // streams): one lane per row, 32 consecutive rows per warp, no segment
  // metadata and no scan
  int row_mode;
  int pair_tiles;      // k_stream_pass streams per lane (1 = tiles; 2 / 4 for short routes)
  const int* row_ptr;  // m+1 (this block's CSR)
  long long m;
  // split rows (> kSplitMin entries, e.g. the hot links of gen_congested)
  // are not in any unit: they are cut into pieces of <= kPiece entries,
  // {entry begin, entry end, row, first slot of the row}, ordered by their
  // relative position in the row so the warps in flight gather from a narrow
  // window of x.  A piece's sum goes to upart[slot]; the piece that brings
  // uctr[first slot] to the row's piece count adds the slots in order
  // (deterministic whichever warp finishes last) and finishes the row.
  const int4* pieces;
  long long npieces;
  unsigned* uctr;
  double* upart;
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Streaming 128-bit index load: read once per pass, no L1 allocation, first
// to be evicted from L2 so the gathered vectors stay resident.
__device__ __forceinline__ int4 ld_stream_int4(const int* p, uint64_t pol) {
  int4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
  double r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int2 ld_nc_int2(const int2* p) {
  int2 r;
  asm("ld.global.nc.v2.s32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_nc_int4(const int4* p) {
  int4 r;
  asm("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// Release of this thread's prior stores + acquire of the other pieces' (one
// instruction instead of a fence and a relaxed atomic).
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ double ld_gather_f64(const double* p) {
  double r;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_hint_f64(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ double dmax_ref(double a, double b) {  // std::max
  return (a < b) ? b : a;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// prox.hpp:31-40 (two cancellation-safe branches, IEEE sqrt and division).
__device__ __forceinline__ double prox_log(double z_sum, double w, double rho, int tau) {
  const double t = static_cast<double>(tau);
  const double d = 4.0 * w * t / rho;
  const double root = sqrt(z_sum * z_sum + d);
  if (z_sum >= 0.0) return (z_sum + root) / (2.0 * t);
  return d / (2.0 * t * (root - z_sum));
}
// prox.hpp:44-56 (prox_linear_scalar clamped at zero, std::max semantics).
__device__ __forceinline__ double prox_linear_nonneg(double z_sum, double w, double rho, int tau) {
  const double x = (z_sum + w / rho) / static_cast<double>(tau);
  return (x < 0.0) ? 0.0 : x;
}

struct GatherV {  // v_l (written by the previous link pass)
  const double* __restrict__ v;
  __device__ __forceinline__ double operator()(int l) const { return __ldg(v + l); }
};
// x_j (written by this iteration's stream pass).  kL1: allocate in L1
// (ld.global.nc) -- the row-mode link pass: P 0.574 -> 0.463 ms, C -1.1%;
// warp units and pieces keep L1::no_allocate (B +0.6% with allocation),
// profiles/r2_x_l1_alloc_ab.txt.
template <bool kL1>
struct GatherX {
  const double* __restrict__ x;
  __device__ __forceinline__ double operator()(int j) const { return kL1 ? __ldg(x + j) : ld_gather_f64(x + j); }
};

// Warp-cooperative segmented gather-sum.  The 32 lanes own contiguous,
// lane-ordered segments [seg_beg, seg_end) tiling [span_beg, span_end) of
// the index array.  Rounds of kStageInts indices are streamed with
// coalesced 128-bit loads (the next round is prefetched into registers
// while the current one is gathered) and parked in shared memory; each lane
// then reads its own indices back and gathers/sums its segment in
// registers, in index order (route order for R^T v, ascending stream id for
// R x), four gathers in flight.
template <class G>
__device__ __forceinline__ double warp_segments_sum(const int* __restrict__ idx, int span_beg,
                                                    int span_end, int seg_beg, int seg_end,
                                                    int* __restrict__ sidx, int lane, G g,
                                                    uint64_t pol_stream) {
  constexpr int NV = kStageInts / 128;
  double acc = 0.0;
  int cb = span_beg & ~3;
  int4 buf[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int gp = cb + 4 * (lane + 32 * i);
    if (gp < span_end) buf[i] = ld_stream_int4(idx + gp, pol_stream);
  }
  while (cb < span_end) {
    const int c1 = min(cb + kStageInts, span_end);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int o = 4 * (lane + 32 * i);
      if (cb + o < c1) *reinterpret_cast<int4*>(sidx + o) = buf[i];
    }
    __syncwarp();
    const int nb = cb + kStageInts;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int gp = nb + 4 * (lane + 32 * i);
      if (gp < span_end) buf[i] = ld_stream_int4(idx + gp, pol_stream);
    }
    const int lo = max(seg_beg, cb), hi = min(seg_end, c1);
    // Batches of kUnroll gathers, the last one predicated: a lane never has
    // fewer than min(kUnroll, remaining) gathers in flight (the passes are
    // bound by outstanding L1->L2 requests, not by instructions).
    for (int k = lo; k < hi; k += kUnroll) {
      double vv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) vv[u] = (k + u < hi) ? g(sidx[k + u - cb]) : 0.0;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (k + u < hi) acc += vv[u];
    }
    __syncwarp();
    cb = nb;
  }
  return acc;
}

// Warp-cooperative gather-sum of one contiguous index range (a split-row
// piece): rounds of kStageInts indices staged as in warp_segments_sum; lane
// k gathers entries k, k+32, ... of each round, so one load instruction
// covers 32 consecutive entries of the row (ascending stream ids: fewer
// distinct lines per request than 32 separate segments).  Returns the
// lane's partial; the caller reduces over the warp.
template <class G>
__device__ __forceinline__ double warp_strided_sum(const int* __restrict__ idx, int beg, int end,
                                                   int* __restrict__ sidx, int lane, G g, uint64_t pol_stream) {
  constexpr int NV = kStageInts / 128;
  double acc = 0.0;
  int cb = beg & ~3;
  int4 buf[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int gp = cb + 4 * (lane + 32 * i);
    if (gp < end) buf[i] = ld_stream_int4(idx + gp, pol_stream);
  }
  while (cb < end) {
    const int c1 = min(cb + kStageInts, end);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int o = 4 * (lane + 32 * i);
      if (cb + o < c1) *reinterpret_cast<int4*>(sidx + o) = buf[i];
    }
    __syncwarp();
    const int nb = cb + kStageInts;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int gp = nb + 4 * (lane + 32 * i);
      if (gp < end) buf[i] = ld_stream_int4(idx + gp, pol_stream);
    }
    for (int k = max(beg, cb) + lane; k < c1; k += 32 * kUnroll) {
      double vv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) vv[u] = (k + 32 * u < c1) ? g(sidx[k + 32 * u - cb]) : 0.0;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (k + 32 * u < c1) acc += vv[u];
    }
    __syncwarp();
    cb = nb;
  }
  return acc;
}

// warp_segments_sum with Q segments per lane ([b[q], e[q]), lane-ordered
// within each q, segment q+1 after segment q across the warp): each batch
// issues kUnroll/Q gathers from every segment, so a lane with Q short routes
// keeps all of them in flight at once.  Each segment is summed in index order.
template <int Q, int kStage, class G>
__device__ __forceinline__ void warp_segments_sum_q(const int* __restrict__ idx, int span_beg,
                                                    int span_end, const int (&b)[Q], const int (&e)[Q],
                                                    int* __restrict__ sidx, int lane, G g,
                                                    uint64_t pol_stream, double (&acc)[Q]) {
  constexpr int NV = kStage / 128;
  constexpr int H = kUnroll / Q;
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = 0.0;
  int cb = span_beg & ~3;
  int4 buf[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int gp = cb + 4 * (lane + 32 * i);
    if (gp < span_end) buf[i] = ld_stream_int4(idx + gp, pol_stream);
  }
  while (cb < span_end) {
    const int c1 = min(cb + kStage, span_end);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int o = 4 * (lane + 32 * i);
      if (cb + o < c1) *reinterpret_cast<int4*>(sidx + o) = buf[i];
    }
    __syncwarp();
    const int nb = cb + kStage;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int gp = nb + 4 * (lane + 32 * i);
      if (gp < span_end) buf[i] = ld_stream_int4(idx + gp, pol_stream);
    }
    int k[Q], hi[Q];
    bool more = false;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      k[q] = max(b[q], cb);
      hi[q] = min(e[q], c1);
      more = more || k[q] < hi[q];
    }
    while (more) {
      double vv[Q][H];
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int u = 0; u < H; ++u) vv[q][u] = (k[q] + u < hi[q]) ? g(sidx[k[q] + u - cb]) : 0.0;
      more = false;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
#pragma unroll
        for (int u = 0; u < H; ++u)
          if (k[q] + u < hi[q]) acc[q] += vv[q][u];
        k[q] += H;
        more = more || k[q] < hi[q];
      }
    }
    __syncwarp();
    cb = nb;
  }
}

// Fixed-order block reduction of NV partials; thread 0 writes out[0..NV).
template <int NV>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* out) {
  __shared__ double red[kWarps][NV];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) red[wib][i] = v[i];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += red[w][i];
      out[i] = s;
    }
  }
  __syncthreads();
}

// Fixed-order sum of a strided partial array by one block; result on all threads.
__device__ __forceinline__ double block_sum_array(const double* part, int count, int stride,
                                                  int comp) {
  __shared__ double red[kWarps];
  __shared__ double total;
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += __ldcg(part + i * stride + comp);
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (lane == 0) red[wib] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += red[w];
    total = t;
  }
  __syncthreads();
  const double r = total;
  __syncthreads();
  return r;
}

__device__ __forceinline__ bool kernel_should_exit(const Ctrl* ctrl) {
  return *reinterpret_cast<const volatile int*>(&ctrl->done) != 0;
}

// v = B + price / rho is stale after a rho change or a state upload
// (rho_changed, set by finalize_iteration / the host): recompute it before
// the iteration's first stream pass.  Exits at entry otherwise.
__global__ void __launch_bounds__(kThreads) k_refresh_v(IterArgs a) {
  if (a.ctrl->rho_changed == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl->v_sel = 0;
  const double rho = a.ctrl->rho;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < a.m;
       l += (long long)gridDim.x * blockDim.x)
    a.v[l] = a.B_in[l] + a.pr_in[l] / rho;
}

// v = B + price / rho unconditionally (outside the loop), v_sel = 0.
__global__ void __launch_bounds__(256) k_set_v(IterArgs a) {
  const double rho = a.ctrl->rho;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < a.m;
       l += (long long)gridDim.x * blockDim.x)
    a.v[l] = a.B_in[l] + a.pr_in[l] / rho;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl->v_sel = 0;
}

// ------------------------------------------------------------ K1: streams
// R^T v gather over the CSC + prox + A update (solver.hpp:325-366
// restated), for the streams of one column block.
template <class G>
__device__ __forceinline__ void stream_pass_body(const IterArgs& a, const BlockArgs& bk, G g,
                                                 double rho, bool trace_it, int* sidx,
                                                 double& p_tda2, double& p_obj) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  const long long ntiles = (bk.s1 - bk.s0 + 31) / 32;
  const double alpha = a.alpha;
  for (long long tile = (long long)blockIdx.x * kWarps + wib; tile < ntiles;
       tile += (long long)gridDim.x * kWarps) {
    const long long j = bk.s0 + tile * 32 + lane;
    const bool valid = j < bk.s1;
    // two independent offset loads (no select on a loaded value, so the
    // second load is not held back by the first)
    const int beg = __ldg(a.col_ptr + (valid ? j : bk.s1));
    const int end = __ldg(a.col_ptr + (valid ? j + 1 : bk.s1));
    double A = 0.0, w = 0.0;
    int kd = 0;
    if (valid) {  // independent of the gather: issue early
      A = ld_stream_f64(a.A_in + j, pol_first);
      w = __ldg(a.w + j);
      kd = __ldg(a.kind + j);
    }
    const int span_beg = __shfl_sync(kFull, beg, 0);
    const int span_end = __shfl_sync(kFull, end, 31);
    const double sum = warp_segments_sum(a.row_idx, span_beg, span_end, beg, end, sidx, lane, g,
                                         pol_first);
    // keep the kind test (and with it the wait for the kind / weight loads)
    // after the gather loop: the compiler otherwise hoists it and the warp
    // stalls on those loads before issuing any gather
    asm volatile("" : "+r"(kd), "+d"(w) : : "memory");
    if (valid) {
      const int tau = end - beg;
      const double zeta = static_cast<double>(tau) * A - sum;
      const double x = (kd == NUMPMP_KIND_LOG) ? prox_log(zeta, w, rho, tau)
                                               : prox_linear_nonneg(zeta, w, rho, tau);
      const double An = alpha * x + (1.0 - alpha) * A;
      const double dA = An - A;
      st_hint_f64(a.x + j, x, pol_last);
      st_hint_f64(a.A_out + j, An, pol_first);
      p_tda2 += static_cast<double>(tau) * dA * dA;
      if (trace_it) p_obj += (kd == NUMPMP_KIND_LOG) ? w * log(x) : w * x;
    }
  }
}

// Multi-route tiles (short routes, e.g. the transit instance's ~3 links): a
// warp takes 32*Q consecutive streams, lane l streams l, l + 32, ..., all Q
// routes' gathers in the same batches -- Q times the work behind each tile's
// chain of dependent loads (offsets, index staging, gathers).
__device__ __forceinline__ void stream_update(const IterArgs& a, long long j, int beg, int end,
                                              double A, double w, int kd, double sum, double rho,
                                              bool trace_it, double& p_tda2, double& p_obj,
                                              uint64_t pol_first, uint64_t pol_last) {
  const int tau = end - beg;
  const double zeta = static_cast<double>(tau) * A - sum;
  const double x = (kd == NUMPMP_KIND_LOG) ? prox_log(zeta, w, rho, tau)
                                           : prox_linear_nonneg(zeta, w, rho, tau);
  const double An = a.alpha * x + (1.0 - a.alpha) * A;
  const double dA = An - A;
  st_hint_f64(a.x + j, x, pol_last);
  st_hint_f64(a.A_out + j, An, pol_first);
  p_tda2 += static_cast<double>(tau) * dA * dA;
  if (trace_it) p_obj += (kd == NUMPMP_KIND_LOG) ? w * log(x) : w * x;
}

template <int Q, class G>
__device__ __forceinline__ void stream_pass_multi(const IterArgs& a, const BlockArgs& bk, G g,
                                                  double rho, bool trace_it, int* sidx,
                                                  double& p_tda2, double& p_obj) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  const long long ngroups = (bk.s1 - bk.s0 + 32 * Q - 1) / (32 * Q);
  for (long long pt = (long long)blockIdx.x * kWarps + wib; pt < ngroups;
       pt += (long long)gridDim.x * kWarps) {
    int beg[Q], end[Q], kd[Q];
    double A[Q], w[Q], sum[Q];
    const long long base = bk.s0 + pt * 32 * Q + lane;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const long long j = base + 32 * q;
      const bool v = j < bk.s1;
      beg[q] = __ldg(a.col_ptr + (v ? j : bk.s1));
      end[q] = __ldg(a.col_ptr + (v ? j + 1 : bk.s1));
      A[q] = 0.0;
      w[q] = 0.0;
      kd[q] = 0;
      if (v) {
        A[q] = ld_stream_f64(a.A_in + j, pol_first);
        w[q] = __ldg(a.w + j);
        kd[q] = __ldg(a.kind + j);
      }
    }
    const int span_beg = __shfl_sync(kFull, beg[0], 0);
    int span_end = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) span_end = max(span_end, __shfl_sync(kFull, end[q], 31));
    warp_segments_sum_q<Q, kStageQ>(a.row_idx, span_beg, span_end, beg, end, sidx, lane, g, pol_first, sum);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      asm volatile("" : "+r"(kd[q]), "+d"(w[q]) : : "memory");
      const long long j = base + 32 * q;
      if (j < bk.s1)
        stream_update(a, j, beg[q], end[q], A[q], w[q], kd[q], sum[q], rho, trace_it, p_tda2, p_obj,
                      pol_first, pol_last);
    }
  }
}

// kQ: streams per lane (1: 32-stream tiles; 2 / 4: multi-route tiles for
// short routes) -- separate instantiations, each with its own registers.
#ifndef NUMPMP_Q_MINB
#define NUMPMP_Q_MINB NUMPMP_MIN_BLOCKS  // resident CTAs per SM the multi-route tiles are built for
#endif
template <int kQ>
__global__ void __launch_bounds__(kThreads, kQ > 1 ? NUMPMP_Q_MINB : kMinBlocks) k_stream_pass(IterArgs a, BlockArgs bk) {
  __shared__ __align__(16) int sidx[kWarps][kQ > 1 ? kStageQ : kStageInts];
  if (kernel_should_exit(a.ctrl)) return;
  const double rho = a.ctrl->rho;
  const long long k = a.ctrl->run_k + 1;
  const bool trace_it = (a.mode == MODE_RUN) && (k % a.trace_every == 0);
  double part[2] = {0.0, 0.0};
  int* sb = sidx[threadIdx.x >> 5];
  const int sel = a.ctrl->v_sel;
  const double* v = (sel == 0 || a.v_alt[0] == nullptr) ? a.v : a.v_alt[sel - 1];
  if (kQ > 1)
    stream_pass_multi<kQ>(a, bk, GatherV{v}, rho, trace_it, sb, part[0], part[1]);
  else
    stream_pass_body(a, bk, GatherV{v}, rho, trace_it, sb, part[0], part[1]);
  block_sum_store<2>(part, a.k1_part + 2 * ((long long)bk.index * a.grid1 + blockIdx.x));
}

// --------------------------------------------------------------- K2: links
struct LinkIn {  // one link's epilogue inputs
  double c, pr, B, zs, Q;
};
__device__ __forceinline__ LinkIn load_link(const IterArgs& a, long long r, uint64_t pol) {
  LinkIn in;
  in.c = __ldg(a.cap + r);
  in.pr = ld_stream_f64(a.pr_in + r, pol);
  in.B = ld_stream_f64(a.B_in + r, pol);
  in.zs = ld_stream_f64(a.zs_in + r, pol);
  in.Q = ld_stream_f64(a.Q_in + r, pol);
  return in;
}
__device__ __forceinline__ double link_update(const IterArgs& a, long long r, double L, int d,
                                             const LinkIn& in, double rho, double (&part)[4],
                                             uint64_t pol_last, double* Bn_out = nullptr,
                                             double* prn_out = nullptr) {
  const double alpha = a.alpha;
  const double u = in.pr / rho;
  const double ps = dmax_ref(in.zs - u, -in.c);
  const double cnt = static_cast<double>(d + 1);
  const double pbar = (L + ps) / cnt;
  part[0] += cnt * pbar * pbar;
  const double Bn = alpha * pbar + (1.0 - alpha) * in.B;
  const double dB = Bn - in.B;
  const double zsn = alpha * (ps - pbar) + (1.0 - alpha) * in.zs;
  const double dzs = zsn - in.zs;
  const double Qn = alpha * L + (1.0 - alpha) * in.Q;
  const double dQ = Qn - in.Q;
  part[1] += dB * dQ;
  part[2] += static_cast<double>(d) * dB * dB;
  part[3] += dzs * dzs;
  const double prn = in.pr + rho * (alpha * pbar);
  a.B_out[r] = Bn;
  a.zs_out[r] = zsn;
  a.Q_out[r] = Qn;
  a.pr_out[r] = prn;
  const double vn = Bn + prn / rho;
  st_hint_f64(a.v + r, vn, pol_last);
  if (Bn_out) {
    *Bn_out = Bn;
    *prn_out = prn;
  }
  if (a.v_alt[0] != nullptr && a.mode == MODE_RUN && (a.ctrl->run_k + 1) % a.rho_interval == 0) {
    // the rhos finalize_iteration may switch to, computed as it does
    st_hint_f64(a.v_alt[0] + r, Bn + prn / (rho * a.gamma), pol_last);
    st_hint_f64(a.v_alt[1] + r, Bn + prn / (rho / a.gamma), pol_last);
  }
  return vn;
}
// Per-link epilogue: slack projection (solver.hpp:368-376), link average
// (110-126), z update split into B / zs / Q (388-399), price (401-405).
__device__ __forceinline__ double link_epilogue(const IterArgs& a, long long r, double L, int d,
                                              double rho, double (&part)[4], uint64_t pol,
                                              uint64_t pol_last, double* Bn_out = nullptr,
                                              double* prn_out = nullptr) {
  return link_update(a, r, L, d, load_link(a, r, pol), rho, part, pol_last, Bn_out, prn_out);
}

// 1.0 when this device's run has exceeded the time limit (solver.hpp:466-473).
__device__ __forceinline__ double time_over_flag(const IterArgs& a) {
  return (a.time_limit_ns > 0 && globaltimer_ns() - a.ctrl->t0_ns > a.time_limit_ns) ? 1.0 : 0.0;
}

// Finalize one iteration on the device: r, s, then the exact control order
// of PmpSolver::run (solver.hpp:450-476).  Runs on one thread.  over_time:
// < 0 reads this device's clock; >= 0 is the sum of the ranks' time_over_flag
// exchanged with the residual partials, so every rank of a sharded run stops
// at the same iteration (a rank's own clock would let them disagree).
__device__ void finalize_iteration(const IterArgs& a, double rho, double tda2, double obj,
                                   double r2, double cross, double ddb2, double dzs2,
                                   double over_time = -1.0) {
  Ctrl* c = a.ctrl;
  double s2r = tda2 - 2.0 * cross + ddb2 + dzs2;
  if (s2r < 0.0) s2r = 0.0;  // rounding of the expanded form near zero
  const double r_norm = sqrt(r2);
  const double s_norm = sqrt(rho * rho * s2r);
  c->iter += 1;
  c->rho_iter = rho;
  c->r_norm = r_norm;
  c->s_norm = s_norm;
  c->rho_changed = 0;
  c->v_sel = 0;
  if (a.mode != MODE_RUN) return;  // step(): no control (solver.hpp:318-409)
  const long long k = ++c->run_k;
  if (!isfinite(r_norm) || !isfinite(s_norm)) {
    c->status = ST_NONFINITE;
    c->done = 1;
    return;
  }
  if (r_norm < a.eps_tol && s_norm < a.eps_tol) {  // check_termination, strict
    c->status = ST_CONVERGED;
    c->done = 1;
    return;
  }
  if (k % a.trace_every == 0 && c->trace_len < a.trace_cap) {
    numpmp_trace_row row;
    row.iter = k;
    row.r_norm = r_norm;
    row.s_norm = s_norm;
    row.rho = rho;
    row.objective = obj;
    a.trace[c->trace_len++] = row;
  }
  if (over_time < 0.0 ? time_over_flag(a) > 0.0 : over_time > 0.0) {
    c->status = ST_TIMELIMIT;
    c->done = 1;
    return;
  }
  if (k % a.rho_interval == 0) {  // update_rho (solver.hpp:168-174)
    if (r_norm > a.mu * s_norm) {
      c->rho = rho * a.gamma;
      c->rho_changed = 1;
      c->v_sel = 1;
    } else if (s_norm > a.mu * r_norm) {
      c->rho = rho / a.gamma;
      c->rho_changed = 1;
      c->v_sel = 2;
    }
  }
  if (k >= a.max_iters) {
    c->status = ST_MAXITERS;
    c->done = 1;
  }
}

// The last CTA of a fused link pass: fixed-order sums of the stream-pass
// and link-pass partials, then finalize_iteration.
// One warp's fixed-order sum of part[i * stride + comp], i < count: lane l
// adds i = l, l + 32, ... (4 loads in flight), then a butterfly.  The same
// order on every call and every rank.
__device__ __forceinline__ double warp_sum_array(const double* part, int count, int stride, int comp,
                                                 int lane) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = lane;
  for (; i + 96 < count; i += 128) {
    s0 += __ldcg(part + (long long)i * stride + comp);
    s1 += __ldcg(part + (long long)(i + 32) * stride + comp);
    s2 += __ldcg(part + (long long)(i + 64) * stride + comp);
    s3 += __ldcg(part + (long long)(i + 96) * stride + comp);
  }
  for (; i < count; i += 32) s0 += __ldcg(part + (long long)i * stride + comp);
  return warp_sum((s0 + s1) + (s2 + s3));
}

// Components 0..ncomp-1 (ncomp <= kWarps) of a strided partial array, one
// warp each in parallel, fixed order; every thread gets res[0..ncomp).
__device__ __forceinline__ void multi_sum(const double* part, int count, int stride, int ncomp,
                                          double* res /* shared, >= ncomp */) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (wib < ncomp) {
    const double v = warp_sum_array(part, count, stride, wib, lane);
    if (lane == 0) res[wib] = v;
  }
  __syncthreads();
}

// The last CTA of an iteration's link side: the six residual / objective
// sums, one warp each, in parallel; then finalize_iteration.
__device__ __forceinline__ void last_block_finalize(const IterArgs& a, double rho, int nparts,
                                                    bool scalars_in_lbuf) {
  static_assert(kWarps >= 6, "one warp per sum");
  __shared__ double sums[6];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n1 = a.grid1 * a.nblocks;
  double v = 0.0;
  if (wib == 0)
    v = scalars_in_lbuf ? __ldcg(a.Lbuf + a.m) : warp_sum_array(a.k1_part, n1, 2, 0, lane);
  else if (wib == 1)
    v = scalars_in_lbuf ? __ldcg(a.Lbuf + a.m + 1) : warp_sum_array(a.k1_part, n1, 2, 1, lane);
  else if (wib < 6)
    v = warp_sum_array(a.k2_part, nparts, 4, wib - 2, lane);
  if (wib < 6 && lane == 0) sums[wib] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    finalize_iteration(a, rho, sums[0], sums[1], sums[2], sums[3], sums[4], sums[5],
                       scalars_in_lbuf ? __ldcg(a.Lbuf + a.m + 2) : -1.0);
    a.ctrl->ticket = 0;
    __threadfence();
  }
}

// Link-pass phases (one launch per column block b).
//   LP_ACC    : b < NB-1: block partial of every link -> Lacc (b = 0 stores,
//               later blocks add in block order).
//   LP_FUSED  : last block, single GPU: L = Lacc + partial, link epilogue,
//               residual partials, last-CTA finalize.
//   LP_GATHER : last block, sharded: local loads -> Lbuf; the last CTA folds
//               the stream-pass scalars into Lbuf[m], Lbuf[m+1] and its
//               time-limit flag into Lbuf[m+2] (one NCCL all-reduce carries all).
//   LP_ROWSUM : last block, outside the iteration: L -> out (R src).
//   LP_P2P    : last block, peer-memory exchange: the row's local load is
//               stored straight into the owning rank's slot for this rank
//               (NVLink store, overlapped with the remaining gathers); the
//               last CTA signals every rank (pmp_p2p.cuh).
enum : int { LP_ACC = 0, LP_FUSED = 1, LP_GATHER = 2, LP_ROWSUM = 3, LP_P2P = 4 };

// Read-only load of a pointer from a device-resident table.
template <class T>
__device__ __forceinline__ T* ld_ptr(T* const* p) {
  return reinterpret_cast<T*>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}

// Signal every rank's counter `which` with ONE system-scope release: a
// fence.acq_rel.sys followed by relaxed reductions is a release pattern for
// each of them (cumulative over everything this thread has observed,
// including the other CTAs' stores ordered before their tickets).  A
// red.release.sys per peer would put `world` system fences, and a
// fence.sc.sys (__threadfence_system) a stronger one, on the critical path
// of the barrier (profiles/r2_p2p_fences.txt).
__device__ __forceinline__ void signal_all_sys(unsigned long long* const* flags_peer, int world, int which) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int q = 0; q < world; ++q) {
    unsigned long long* c = ld_ptr(flags_peer + q) + which;
    asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
  }
}

// Link-pass gather over one column block's CSR, in "warp units": the rows
// (links) are cut into segments of <= seg entries (near-equal split; every
// row has >= 1 segment, possibly empty), and consecutive whole rows are
// packed into units of <= 32 segments.  A warp takes one unit, one lane per
// segment; a fixed-order segmented inclusive scan over the lanes leaves the
// block partial of each row at its last ("tail") lane, which owns the row's
// epilogue.  Rows never cross units, so no second combine pass exists.
// kForm: 0 row mode, 1 warp units, 2 warp units + split-row pieces (separate
// instantiations: neither form's code shapes another's register allocation).
#ifndef NUMPMP_ROW_MINB
#define NUMPMP_ROW_MINB NUMPMP_MIN_BLOCKS
#endif
template <int kPhase, int kForm>
__global__ void __launch_bounds__(kThreads, kForm == 0 ? NUMPMP_ROW_MINB : kMinBlocks) k_link_pass(IterArgs a, BlockArgs bk,
                                                                   const double* __restrict__ src,
                                                                   double* __restrict__ out) {
  __shared__ __align__(16) int sidx[kWarps][kStageInts];
  __shared__ bool s_last;
  if (a.mode != MODE_AUX && kernel_should_exit(a.ctrl)) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  const double rho = (kPhase == LP_FUSED) ? a.ctrl->rho : 0.0;
  double part[4] = {0.0, 0.0, 0.0, 0.0};
  // a row's action once its load (this block's part added) is known
  auto row_done = [&](long long r, double L) {
    if (kPhase == LP_ACC) {
      __stcg(a.Lacc + r, L);
    } else if (kPhase == LP_ROWSUM) {
      out[r] = L;
    } else if (kPhase == LP_GATHER) {
      a.Lbuf[r] = L;
    } else if (kPhase == LP_P2P) {
      // owner and local index in 32 bits (m < 2^31: int32 CSR offsets)
      const unsigned mo = static_cast<unsigned>(a.p2p.mo);
      const unsigned q = static_cast<unsigned>(r) / mo;
      double* dst = ld_ptr(a.p2p.slots_peer + q);
      dst[static_cast<long long>(a.p2p.rank) * a.p2p.mo + (static_cast<unsigned>(r) - q * mo)] = L;
    } else {
      link_epilogue(a, r, L, __ldg(a.deg + r), rho, part, pol_first, pol_last);
    }
  };
  if (kForm == 0) {
    const long long ngroups = (bk.m + 31) / 32;
    for (long long g = (long long)blockIdx.x * kWarps + wib; g < ngroups;
         g += (long long)gridDim.x * kWarps) {
      const long long r = g * 32 + lane;
      const bool valid = r < bk.m;
      const int rb = __ldg(bk.row_ptr + (valid ? r : bk.m));
      const int re = __ldg(bk.row_ptr + (valid ? r + 1 : bk.m));
      double Lprev = 0.0;
      if (!bk.first && valid) Lprev = __ldcg(a.Lacc + r);
      const int span_beg = __shfl_sync(kFull, rb, 0);
      const int span_end = __shfl_sync(kFull, re, 31);
      const double s = warp_segments_sum(bk.col_idx, span_beg, span_end, rb, re, sidx[wib], lane,
                                         GatherX<true>{src}, pol_first);
      if (valid) row_done(r, bk.first ? s : Lprev + s);
    }
  } else {
    const long long ustride = (long long)gridDim.x * kWarps;
    long long u = (long long)blockIdx.x * kWarps + wib;
    // this unit's segment range, loaded one unit ahead (the units -> vptr
    // chain would otherwise put two dependent loads in front of every unit)
    int2 vr = make_int2(0, 0);
    if (u < bk.nu) vr = ld_nc_int2(bk.units + u);
    for (; u < bk.nu; u += ustride) {
      const int v0 = vr.x, v1 = vr.y;
      const int v = v0 + lane;
      const bool valid = v < v1;
      // independent loads, no select on a loaded value (it would hold the
      // next load back until the first one returns)
      const int vb = __ldg(bk.vptr + (valid ? v : v1));
      const int ve = __ldg(bk.vptr + (valid ? v + 1 : v1));
      int row = -1 - lane;
      if (valid) row = __ldg(bk.vrow + v);
      if (u + ustride < bk.nu) vr = ld_nc_int2(bk.units + u + ustride);
      const int span_beg = __shfl_sync(kFull, vb, 0);
      const int span_end = __shfl_sync(kFull, ve, 31);
      double s = warp_segments_sum(bk.col_idx, span_beg, span_end, vb, ve, sidx[wib], lane,
                                   GatherX<false>{src}, pol_first);
  #pragma unroll
      for (int d = 1; d < 32; d <<= 1) {  // segmented scan, segments = equal rows
        const double t = __shfl_up_sync(kFull, s, d);
        const int tr = __shfl_up_sync(kFull, row, d);
        if (lane >= d && tr == row) s += t;
      }
      const int next_row = __shfl_down_sync(kFull, row, 1);
      if (!valid || (lane != 31 && next_row == row)) continue;  // not the row's tail
      const long long r = row;
      row_done(r, bk.first ? s : __ldcg(a.Lacc + r) + s);
    }
    // split rows, piece by piece
    for (long long q = (long long)blockIdx.x * kWarps + wib; kForm == 2 && q < bk.npieces; q += ustride) {
      const int4 pc = ld_nc_int4(bk.pieces + q);
      double s = warp_strided_sum(bk.col_idx, pc.x, pc.y, sidx[wib], lane, GatherX<false>{src}, pol_first);
  #pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);  // same bits on every lane
      const int rb = __ldg(bk.row_ptr + pc.z), re = __ldg(bk.row_ptr + pc.z + 1);
      const int np = (re - rb + kPiece - 1) / kPiece;
      unsigned done = 0;
      if (lane == 0) {
        __stcg(bk.upart + pc.w + (pc.x - rb) / kPiece, s);
        done = atom_add_acq_rel(bk.uctr + pc.w, 1u);
      }
      done = __shfl_sync(kFull, done, 0);
      if (done != static_cast<unsigned>(np - 1)) continue;
      // last piece of the row: the slots in a fixed order (lane-strided, then butterfly)
      double S = 0.0;
      for (int k = lane; k < np; k += 32) S += __ldcg(bk.upart + pc.w + k);
  #pragma unroll
      for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(kFull, S, o);
      if (lane == 0) {
        bk.uctr[pc.w] = 0u;  // ready for the next launch
        const long long r = pc.z;
        row_done(r, bk.first ? S : __ldcg(a.Lacc + r) + S);
      }
    }
  }
  if (kPhase == LP_ACC || kPhase == LP_ROWSUM) return;
  if (kPhase == LP_P2P) {
    // The CTA's peer stores, then a fence before the ticket (the grid.sync
    // pattern: bar.sync orders the CTA's writes before thread 0's cumulative
    // fence).  The ticket is observed on this GPU only, so a gpu-scope fence
    // orders the stores before it; the last CTA's system-scope release
    // (signal_all_sys) is cumulative over everything it observed, which makes
    // every CTA's peer stores visible to the peers that acquire the signal.
    __syncthreads();
    if (threadIdx.x == 0) {
      if (a.p2p.cta_sysfence)
        __threadfence_system();
      else
        __threadfence();
      s_last = (atomicAdd(&a.ctrl->ticket2, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    // (the stream-pass scalars are summed by the owner epilogue's last CTA)
    a.ctrl->ticket2 = 0;
    signal_all_sys(a.p2p.flags_peer, a.p2p.world, 0);  // "loads stored"
    return;
  }
  if (kPhase == LP_GATHER) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&a.ctrl->ticket2, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ double k1s[2];
    multi_sum(a.k1_part, a.grid1 * a.nblocks, 2, 2, k1s);
    if (threadIdx.x == 0) {
      a.Lbuf[a.m] = k1s[0];
      a.Lbuf[a.m + 1] = k1s[1];
      a.Lbuf[a.m + 2] = time_over_flag(a);  // summed by the all-reduce
      a.ctrl->ticket2 = 0;
    }
    return;
  }
  block_sum_store<4>(part, a.k2_part + 4 * blockIdx.x);
  __threadfence();
  if (threadIdx.x == 0) s_last = (atomicAdd(&a.ctrl->ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  last_block_finalize(a, rho, gridDim.x, false);
}

// The link epilogue as a streaming pass (one thread per link, coalesced):
// kSrc 0 = sharded, on the all-reduced loads Lbuf (scalars in Lbuf[m..]);
// kSrc 1 = one device, on the loads the last block accumulated into Lacc.
// Residual partials, last-CTA finalize.
template <int kSrc>
#ifndef NUMPMP_EPI_MINB
#define NUMPMP_EPI_MINB 4  // 4 CTAs per SM (64 registers): C -0.35% (profiles/r1_congested_sweeps.txt, lib A/B)
#endif
__global__ void __launch_bounds__(kThreads, NUMPMP_EPI_MINB) k_link_epilogue(IterArgs a) {
  __shared__ bool s_last;
  if (kernel_should_exit(a.ctrl)) return;
  const double rho = a.ctrl->rho;
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  double part[4] = {0.0, 0.0, 0.0, 0.0};
  const double* L = (kSrc == 0) ? a.Lbuf : a.Lacc;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < a.m; r += 2 * stride) {
    // two links' loads in flight per thread (same link order as one at a time)
    const long long r1 = r + stride;
    const bool has1 = r1 < a.m;
    const LinkIn in0 = load_link(a, r, pol_first);
    const double L0 = __ldcg(L + r);
    const int d0 = __ldg(a.deg + r);
    LinkIn in1{};
    double L1 = 0.0;
    int d1 = 0;
    if (has1) {
      in1 = load_link(a, r1, pol_first);
      L1 = __ldcg(L + r1);
      d1 = __ldg(a.deg + r1);
    }
    link_update(a, r, L0, d0, in0, rho, part, pol_last);
    if (has1) link_update(a, r1, L1, d1, in1, rho, part, pol_last);
  }
  block_sum_store<4>(part, a.k2_part + 4 * blockIdx.x);
  __threadfence();
  if (threadIdx.x == 0) s_last = (atomicAdd(&a.ctrl->ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  last_block_finalize(a, rho, gridDim.x, kSrc == 0);
}

}  // namespace numpmp_dev
