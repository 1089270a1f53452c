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
#define NUMPMP_GATHER_UNROLL 4
#endif
constexpr int kWarps = NUMPMP_WARPS;  // warps per block (gather passes)
constexpr int kThreads = kWarps * 32;
constexpr int kMinBlocks = NUMPMP_MIN_BLOCKS;  // resident blocks per SM the passes are built for
constexpr int kStageInts = NUMPMP_STAGE_INTS;  // staged indices per warp and round
constexpr int kUnroll = NUMPMP_GATHER_UNROLL;  // gathers in flight per lane
constexpr int kSeg = kStageInts / 32;          // target entries per link segment (one staged round per warp)
constexpr int kMaxBlocks = 16;                 // max column blocks
// Index ring (per warp): kRingPieces pieces of kPieceInts indices, each
// fetched by one TMA bulk copy and completed on its own mbarrier.
constexpr int kPieceInts = 128;
constexpr int kRingPieces = 8;
constexpr int kRingInts = kPieceInts * kRingPieces;
// An item (tile / unit) may use the ring if its index span, at the worst
// alignment, touches at most kRingPieces - 1 pieces (>= 1 piece of lookahead).
constexpr int kRingMaxSpan = kPieceInts * (kRingPieces - 2);
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
  int pad;
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
  double* k1_part;  // [nb][grid1][2]: tau dA^2, objective
  double* k2_part;  // [grid2][4]: r^2, dB.dQ, d dB^2, dzs^2
  int grid1, grid2, grid3, nblocks;
  double* Lacc;     // m: link loads accumulated over the column blocks
  double* Lbuf;     // sharded: m partial loads + 2 scalars
  Ctrl* ctrl;
  numpmp_trace_row* trace;
  long long trace_cap;
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
  const int* uptr;     // nu+1: first segment of each warp unit
  long long nv, nu;
  int index;           // block number b
  int first;           // b == 0
  // static per-warp work ranges (k_stream_pass: 32-stream tiles; k_link_pass:
  // warp units), balanced by index count; fb*: the range has an item too
  // long for the index ring and takes the direct staging path.
  const int* wr1;
  const unsigned char* fb1;
  const int* wr2;
  const unsigned char* fb2;
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
struct GatherBU {  // v_l recomputed after a rho change / state upload
  const double* __restrict__ B;
  const double* __restrict__ pr;
  double rho;
  __device__ __forceinline__ double operator()(int l) const {
    return __ldg(B + l) + __ldg(pr + l) / rho;
  }
};
struct GatherX {  // x_j (written by this iteration's stream pass)
  const double* __restrict__ x;
  __device__ __forceinline__ double operator()(int j) const { return ld_gather_f64(x + j); }
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
    int k = lo;
    for (; k + kUnroll <= hi; k += kUnroll) {
      int ii[kUnroll];
      double vv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) ii[u] = sidx[k + u - cb];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) vv[u] = g(ii[u]);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) acc += vv[u];
    }
    for (; k < hi; ++k) acc += g(sidx[k - cb]);
    __syncwarp();
    cb = nb;
  }
  return acc;
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

// ------------------------------------------------------- warp index ring
// A warp owns a static, contiguous range of work items whose index spans are
// contiguous and increasing (32-stream tiles of the CSC, or warp units of
// the CSR).  The range's index stream [start, end) is fetched into a ring of
// kRingPieces x kPieceInts ints in shared memory by TMA bulk copies
// (cp.async.bulk, one elected lane, completion on one mbarrier per piece),
// up to kRingPieces pieces ahead of the consumer.  The indices never pass
// through registers or the LSU on the way in, and the fetch of the next
// items' indices overlaps the gathers of the current one.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct WarpRing {
  uint32_t sbuf;  // shared-memory address of the ring
  uint32_t sbar;  // shared-memory address of the kRingPieces mbarriers
  const int* src;
  int base;       // absolute index of piece 0 (16-byte aligned)
  int npieces, issued, ready, released;

  __device__ __forceinline__ void init_barriers(int lane) {
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < kRingPieces; ++k)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar + 8 * k));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  __device__ __forceinline__ void start(const int* s, int first, int last, int lane) {
    src = s;
    base = first & ~3;
    npieces = last > first ? (last - base + kPieceInts - 1) / kPieceInts : 0;
    issued = ready = released = 0;
    top_up(lane);
  }
  __device__ __forceinline__ void issue(int k, int lane) {
    if (lane == 0) {
      const uint32_t b = sbar + 8 * (k & (kRingPieces - 1));
      const uint32_t dst = sbuf + 4 * kPieceInts * (k & (kRingPieces - 1));
      const int* g = src + base + static_cast<long long>(k) * kPieceInts;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                   "r"(kPieceInts * 4)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              dst),
          "l"(g), "r"(kPieceInts * 4), "r"(b)
          : "memory");
    }
  }
  __device__ __forceinline__ void top_up(int lane) {
    while (issued < npieces && issued < released + kRingPieces) {
      issue(issued, lane);
      ++issued;
    }
  }
  // Make every piece up to absolute position last-1 resident.
  __device__ __forceinline__ void acquire(int last) {
    const int ke = (last - 1 - base) / kPieceInts;
    if (ke >= issued) __trap();  // item longer than the ring: a host planning bug, never a hang
    while (ready <= ke) {
      const uint32_t b = sbar + 8 * (ready & (kRingPieces - 1));
      const uint32_t par = (ready / kRingPieces) & 1;
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(b), "r"(par)
            : "memory");
      ++ready;
    }
  }
  // The next item starts at absolute position pos: recycle the pieces
  // wholly below it (only pieces already waited on).
  __device__ __forceinline__ void release_below(int pos, int lane) {
    const int kn = min((pos - base) / kPieceInts, ready);
    if (kn > released) {
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      released = kn;
      top_up(lane);
    }
  }
  __device__ __forceinline__ int at(int p) const {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(sbuf + 4 * ((p - base) & (kRingInts - 1))));
    return v;
  }
};

// Sum of g over the ring positions [b, e), in index order, kUnroll in flight.
template <class G>
__device__ __forceinline__ double ring_segment_sum(const WarpRing& ring, int b, int e, G g) {
  double acc = 0.0;
  int k = b;
  for (; k + kUnroll <= e; k += kUnroll) {
    int ii[kUnroll];
    double vv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) ii[u] = ring.at(k + u);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) vv[u] = g(ii[u]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) acc += vv[u];
  }
  for (; k < e; ++k) acc += g(ring.at(k));
  return acc;
}

// ------------------------------------------------------------ K1: streams
// R^T v gather over the CSC + prox + A update (solver.hpp:325-366
// restated), for the streams of one column block.  A warp takes its static
// range of 32-stream tiles [tlo, thi), one lane per stream.

struct TileMeta {  // one lane's stream of a tile
  int beg, end, kd;
  double A, w;
  bool valid;
};
__device__ __forceinline__ TileMeta load_tile(const IterArgs& a, const BlockArgs& bk, long long t,
                                              int lane, uint64_t pol_first) {
  TileMeta m;
  const long long j = bk.s0 + 32 * t + lane;
  m.valid = j < bk.s1;
  m.beg = __ldg(a.col_ptr + (m.valid ? j : bk.s1));
  m.end = m.valid ? __ldg(a.col_ptr + j + 1) : m.beg;
  m.A = 0.0;
  m.w = 0.0;
  m.kd = 0;
  if (m.valid) {
    m.A = ld_stream_f64(a.A_in + j, pol_first);
    m.w = __ldg(a.w + j);
    m.kd = __ldg(a.kind + j);
  }
  return m;
}

__device__ __forceinline__ void stream_update(const IterArgs& a, long long j, const TileMeta& m,
                                              double sum, double rho, bool trace_it,
                                              double& p_tda2, double& p_obj, uint64_t pol_first,
                                              uint64_t pol_last) {
  const int tau = m.end - m.beg;
  const double zeta = static_cast<double>(tau) * m.A - sum;
  const double x = (m.kd == NUMPMP_KIND_LOG) ? prox_log(zeta, m.w, rho, tau)
                                             : prox_linear_nonneg(zeta, m.w, rho, tau);
  const double An = a.alpha * x + (1.0 - a.alpha) * m.A;
  const double dA = An - m.A;
  st_hint_f64(a.x + j, x, pol_last);
  st_hint_f64(a.A_out + j, An, pol_first);
  p_tda2 += static_cast<double>(tau) * dA * dA;
  if (trace_it) p_obj += (m.kd == NUMPMP_KIND_LOG) ? m.w * log(x) : m.w * x;
}

// Ring path: the tiles' indices arrive through the warp's TMA ring; the next
// tile's offsets are loaded while this tile gathers (the stream state is
// needed only after the gather, so it is issued at the tile's start).
template <class G>
__device__ __forceinline__ void stream_pass_ring(const IterArgs& a, const BlockArgs& bk, G g,
                                                 double rho, bool trace_it, WarpRing& ring,
                                                 int lane, int tlo, int thi, double& p_tda2,
                                                 double& p_obj) {
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  const long long jf = bk.s0 + 32LL * tlo, jl = min(bk.s0 + 32LL * thi, bk.s1);
  ring.start(a.row_idx, __ldg(a.col_ptr + jf), __ldg(a.col_ptr + jl), lane);
  long long j = jf + lane;
  int beg = __ldg(a.col_ptr + min(j, bk.s1));
  int end = (j < bk.s1) ? __ldg(a.col_ptr + j + 1) : beg;
  for (int t = tlo; t < thi; ++t, j += 32) {
    const bool valid = j < bk.s1;
    TileMeta cur;
    cur.valid = valid;
    cur.beg = beg;
    cur.end = end;
    cur.A = 0.0;
    cur.w = 0.0;
    cur.kd = 0;
    if (valid) {
      cur.A = ld_stream_f64(a.A_in + j, pol_first);
      cur.w = __ldg(a.w + j);
      cur.kd = __ldg(a.kind + j);
    }
    if (t + 1 < thi) {  // next tile's offsets
      const long long jn = j + 32;
      beg = __ldg(a.col_ptr + min(jn, bk.s1));
      end = (jn < bk.s1) ? __ldg(a.col_ptr + jn + 1) : beg;
    }
    const int span_beg = __shfl_sync(kFull, cur.beg, 0);
    const int span_end = __shfl_sync(kFull, cur.end, 31);
    double sum = 0.0;
    if (span_end > span_beg) {
      ring.acquire(span_end);
      sum = ring_segment_sum(ring, cur.beg, cur.end, g);
    }
    ring.release_below(span_end, lane);
    if (valid) stream_update(a, j, cur, sum, rho, trace_it, p_tda2, p_obj, pol_first, pol_last);
  }
}

// Direct path (a tile too long for the ring): indices staged through
// registers into shared memory, round by round (warp_segments_sum).
template <class G>
__device__ __forceinline__ void stream_pass_direct(const IterArgs& a, const BlockArgs& bk, G g,
                                                   double rho, bool trace_it, int* sidx, int lane,
                                                   int tlo, int thi, double& p_tda2,
                                                   double& p_obj) {
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  for (int t = tlo; t < thi; ++t) {
    const TileMeta cur = load_tile(a, bk, t, lane, pol_first);
    const int span_beg = __shfl_sync(kFull, cur.beg, 0);
    const int span_end = __shfl_sync(kFull, cur.end, 31);
    const double sum = warp_segments_sum(a.row_idx, span_beg, span_end, cur.beg, cur.end, sidx,
                                         lane, g, pol_first);
    if (cur.valid)
      stream_update(a, bk.s0 + 32LL * t + lane, cur, sum, rho, trace_it, p_tda2, p_obj, pol_first,
                    pol_last);
  }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) k_stream_pass(IterArgs a, BlockArgs bk) {
  __shared__ __align__(128) int sbuf[kWarps][kRingInts];
  __shared__ __align__(8) uint64_t sbar[kWarps][kRingPieces];
  if (kernel_should_exit(a.ctrl)) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const double rho = a.ctrl->rho;
  const bool rc = a.ctrl->rho_changed != 0;
  const long long k = a.ctrl->run_k + 1;
  const bool trace_it = (a.mode == MODE_RUN) && (k % a.trace_every == 0);
  double part[2] = {0.0, 0.0};
  const int gw = blockIdx.x * kWarps + wib;
  const int tlo = __ldg(bk.wr1 + gw), thi = __ldg(bk.wr1 + gw + 1);
  if (tlo < thi) {
    // v = B + price / rho is stale after a rho change or a state upload (one
    // iteration in rho_update_interval): that iteration gathers B and price
    // directly, on the staging path.
    if (rc) {
      stream_pass_direct(a, bk, GatherBU{a.B_in, a.pr_in, rho}, rho, trace_it, sbuf[wib], lane, tlo,
                         thi, part[0], part[1]);
    } else if (__ldg(bk.fb1 + gw)) {
      stream_pass_direct(a, bk, GatherV{a.v}, rho, trace_it, sbuf[wib], lane, tlo, thi, part[0],
                         part[1]);
    } else {
      WarpRing ring;
      ring.sbuf = smem_addr(sbuf[wib]);
      ring.sbar = smem_addr(sbar[wib]);
      ring.init_barriers(lane);
      stream_pass_ring(a, bk, GatherV{a.v}, rho, trace_it, ring, lane, tlo, thi, part[0], part[1]);
    }
  }
  block_sum_store<2>(part, a.k1_part + 2 * ((long long)bk.index * a.grid1 + blockIdx.x));
}

// --------------------------------------------------------------- K2: links
// Per-link epilogue: slack projection (solver.hpp:368-376), link average
// (110-126), z update split into B / zs / Q (388-399), price (401-405).
__device__ __forceinline__ void link_epilogue(const IterArgs& a, long long r, double L, int d,
                                              double rho, double (&part)[4], uint64_t pol,
                                              uint64_t pol_last) {
  const double alpha = a.alpha;
  const double c = __ldg(a.cap + r);
  const double pr = ld_stream_f64(a.pr_in + r, pol);
  const double B = ld_stream_f64(a.B_in + r, pol);
  const double zs = ld_stream_f64(a.zs_in + r, pol);
  const double Q = ld_stream_f64(a.Q_in + r, pol);
  const double u = pr / rho;
  const double ps = dmax_ref(zs - u, -c);
  const double cnt = static_cast<double>(d + 1);
  const double pbar = (L + ps) / cnt;
  part[0] += cnt * pbar * pbar;
  const double Bn = alpha * pbar + (1.0 - alpha) * B;
  const double dB = Bn - B;
  const double zsn = alpha * (ps - pbar) + (1.0 - alpha) * zs;
  const double dzs = zsn - zs;
  const double Qn = alpha * L + (1.0 - alpha) * Q;
  const double dQ = Qn - Q;
  part[1] += dB * dQ;
  part[2] += static_cast<double>(d) * dB * dB;
  part[3] += dzs * dzs;
  const double prn = pr + rho * (alpha * pbar);
  a.B_out[r] = Bn;
  a.zs_out[r] = zsn;
  a.Q_out[r] = Qn;
  a.pr_out[r] = prn;
  st_hint_f64(a.v + r, Bn + prn / rho, pol_last);
}

// Finalize one iteration on the device: r, s, then the exact control order
// of PmpSolver::run (solver.hpp:450-476).  Runs on one thread.
__device__ void finalize_iteration(const IterArgs& a, double rho, double tda2, double obj,
                                   double r2, double cross, double ddb2, double dzs2) {
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
  if (a.time_limit_ns > 0 && globaltimer_ns() - c->t0_ns > a.time_limit_ns) {
    c->status = ST_TIMELIMIT;
    c->done = 1;
    return;
  }
  if (k % a.rho_interval == 0) {  // update_rho (solver.hpp:168-174)
    if (r_norm > a.mu * s_norm) {
      c->rho = rho * a.gamma;
      c->rho_changed = 1;
    } else if (s_norm > a.mu * r_norm) {
      c->rho = rho / a.gamma;
      c->rho_changed = 1;
    }
  }
  if (k >= a.max_iters) {
    c->status = ST_MAXITERS;
    c->done = 1;
  }
}

// The last CTA of a fused link pass: fixed-order sums of the stream-pass
// and link-pass partials, then finalize_iteration.
__device__ __forceinline__ void last_block_finalize(const IterArgs& a, double rho, int nparts,
                                                    bool scalars_in_lbuf) {
  double tda2, obj;
  if (scalars_in_lbuf) {
    tda2 = __ldcg(a.Lbuf + a.m);
    obj = __ldcg(a.Lbuf + a.m + 1);
  } else {
    tda2 = block_sum_array(a.k1_part, a.grid1 * a.nblocks, 2, 0);
    obj = block_sum_array(a.k1_part, a.grid1 * a.nblocks, 2, 1);
  }
  const double r2 = block_sum_array(a.k2_part, nparts, 4, 0);
  const double cross = block_sum_array(a.k2_part, nparts, 4, 1);
  const double ddb2 = block_sum_array(a.k2_part, nparts, 4, 2);
  const double dzs2 = block_sum_array(a.k2_part, nparts, 4, 3);
  if (threadIdx.x == 0) {
    finalize_iteration(a, rho, tda2, obj, r2, cross, ddb2, dzs2);
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
//               the stream-pass scalars into Lbuf[m], Lbuf[m+1] (one NCCL
//               all-reduce carries both).
//   LP_ROWSUM : last block, outside the iteration: L -> out (R src).
enum : int { LP_ACC = 0, LP_FUSED = 1, LP_GATHER = 2, LP_ROWSUM = 3 };

// Link-pass gather over one column block's CSR, in "warp units": the rows
// (links) are cut into segments of <= seg entries (near-equal split; every
// row has >= 1 segment, possibly empty), and consecutive whole rows are
// packed into units of <= 32 segments.  A warp takes its static range of
// units, one lane per segment; a fixed-order segmented inclusive scan over
// the lanes leaves the block partial of each row at its last ("tail") lane,
// which owns the row's epilogue.  Rows never cross units, so no second
// combine pass exists.

struct UnitMeta {  // one lane's segment of a unit
  int vb, ve, row;
  bool valid;
};
// uptr values of units ubase.. are held one per lane in `up`.
__device__ __forceinline__ UnitMeta load_unit(const BlockArgs& bk, int up, int rel, int lane) {
  UnitMeta m;
  const int v0 = __shfl_sync(kFull, up, rel), v1 = __shfl_sync(kFull, up, rel + 1);
  const int v = v0 + lane;
  m.valid = v < v1;
  m.vb = __ldg(bk.vptr + (m.valid ? v : v1));
  m.ve = m.valid ? __ldg(bk.vptr + v + 1) : m.vb;
  m.row = m.valid ? __ldg(bk.vrow + v) : -1 - lane;
  return m;
}

// Segmented scan of the lanes' partials (segments = equal rows) and the
// row's action at its tail lane.  Lprev: the row's accumulated load of the
// earlier column blocks (prefetched; ignored for the first block).
template <int kPhase>
__device__ __forceinline__ void unit_finish(const IterArgs& a, const BlockArgs& bk, double s,
                                            const UnitMeta& m, double Lprev, double* out, int lane,
                                            double rho, double (&part)[4], uint64_t pol_first,
                                            uint64_t pol_last) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double t = __shfl_up_sync(kFull, s, d);
    const int tr = __shfl_up_sync(kFull, m.row, d);
    if (lane >= d && tr == m.row) s += t;
  }
  const int next_row = __shfl_down_sync(kFull, m.row, 1);
  if (!m.valid || (lane != 31 && next_row == m.row)) return;  // not the row's tail
  const long long r = m.row;
  const double L = bk.first ? s : Lprev + s;
  if (kPhase == LP_ACC) {
    __stcg(a.Lacc + r, L);
  } else if (kPhase == LP_ROWSUM) {
    out[r] = L;
  } else if (kPhase == LP_GATHER) {
    a.Lbuf[r] = L;
  } else {
    link_epilogue(a, r, L, __ldg(a.deg + r), rho, part, pol_first, pol_last);
  }
}

template <int kPhase>
__device__ __forceinline__ void link_pass_ring(const IterArgs& a, const BlockArgs& bk,
                                               const double* __restrict__ src, double* out,
                                               WarpRing& ring, int lane, int ulo, int uhi,
                                               double rho, double (&part)[4]) {
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  int ubase = ulo;
  int up = __ldg(bk.uptr + min(ubase + lane, uhi));
  const int sf = __shfl_sync(kFull, up, 0);
  ring.start(bk.col_idx, __ldg(bk.vptr + sf), __ldg(bk.vptr + __ldg(bk.uptr + uhi)), lane);
  UnitMeta cur = load_unit(bk, up, 0, lane);
  double Lcur = 0.0;
  if (!bk.first && cur.valid) Lcur = __ldcg(a.Lacc + cur.row);
  for (int u = ulo; u < uhi; ++u) {
    UnitMeta nxt;
    nxt.valid = false;
    nxt.row = -1 - lane;
    if (u + 1 < uhi) {
      if (u + 1 - ubase >= 31) {
        ubase = u + 1;
        up = __ldg(bk.uptr + min(ubase + lane, uhi));
      }
      nxt = load_unit(bk, up, u + 1 - ubase, lane);
    }
    const int span_beg = __shfl_sync(kFull, cur.vb, 0);
    const int span_end = __shfl_sync(kFull, cur.ve, 31);
    double s = 0.0;
    if (span_end > span_beg) {
      ring.acquire(span_end);
      s = ring_segment_sum(ring, cur.vb, cur.ve, GatherX{src});
    }
    ring.release_below(span_end, lane);
    double Lnxt = 0.0;
    if (!bk.first && nxt.valid) Lnxt = __ldcg(a.Lacc + nxt.row);
    unit_finish<kPhase>(a, bk, s, cur, Lcur, out, lane, rho, part, pol_first, pol_last);
    cur = nxt;
    Lcur = Lnxt;
  }
}

template <int kPhase>
__device__ __forceinline__ void link_pass_direct(const IterArgs& a, const BlockArgs& bk,
                                                 const double* __restrict__ src, double* out,
                                                 int* sidx, int lane, int ulo, int uhi, double rho,
                                                 double (&part)[4]) {
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  for (int u = ulo; u < uhi; ++u) {
    const int up = __ldg(bk.uptr + min(u + lane, uhi));
    const UnitMeta cur = load_unit(bk, up, 0, lane);
    const int span_beg = __shfl_sync(kFull, cur.vb, 0);
    const int span_end = __shfl_sync(kFull, cur.ve, 31);
    const double s = warp_segments_sum(bk.col_idx, span_beg, span_end, cur.vb, cur.ve, sidx, lane,
                                       GatherX{src}, pol_first);
    const double Lprev = (!bk.first && cur.valid) ? __ldcg(a.Lacc + cur.row) : 0.0;
    unit_finish<kPhase>(a, bk, s, cur, Lprev, out, lane, rho, part, pol_first, pol_last);
  }
}

template <int kPhase>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_link_pass(IterArgs a, BlockArgs bk,
                                                                   const double* __restrict__ src,
                                                                   double* __restrict__ out) {
  __shared__ __align__(128) int sbuf[kWarps][kRingInts];
  __shared__ __align__(8) uint64_t sbar[kWarps][kRingPieces];
  __shared__ bool s_last;
  if (a.mode != MODE_AUX && kernel_should_exit(a.ctrl)) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const double rho = (kPhase == LP_FUSED) ? a.ctrl->rho : 0.0;
  double part[4] = {0.0, 0.0, 0.0, 0.0};
  const int gw = blockIdx.x * kWarps + wib;
  const int ulo = __ldg(bk.wr2 + gw), uhi = __ldg(bk.wr2 + gw + 1);
  if (ulo < uhi) {
    if (__ldg(bk.fb2 + gw)) {
      link_pass_direct<kPhase>(a, bk, src, out, sbuf[wib], lane, ulo, uhi, rho, part);
    } else {
      WarpRing ring;
      ring.sbuf = smem_addr(sbuf[wib]);
      ring.sbar = smem_addr(sbar[wib]);
      ring.init_barriers(lane);
      link_pass_ring<kPhase>(a, bk, src, out, ring, lane, ulo, uhi, rho, part);
    }
  }
  if (kPhase == LP_ACC || kPhase == LP_ROWSUM) return;
  if (kPhase == LP_GATHER) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&a.ctrl->ticket2, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const double tda2 = block_sum_array(a.k1_part, a.grid1 * a.nblocks, 2, 0);
    const double obj = block_sum_array(a.k1_part, a.grid1 * a.nblocks, 2, 1);
    if (threadIdx.x == 0) {
      a.Lbuf[a.m] = tda2;
      a.Lbuf[a.m + 1] = obj;
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

// Sharded: the replicated link epilogue on the all-reduced loads Lbuf (one
// thread per link), residual partials, last-CTA finalize.
__global__ void __launch_bounds__(kThreads) k_link_epilogue(IterArgs a) {
  __shared__ bool s_last;
  if (kernel_should_exit(a.ctrl)) return;
  const double rho = a.ctrl->rho;
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  double part[4] = {0.0, 0.0, 0.0, 0.0};
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < a.m;
       r += (long long)gridDim.x * blockDim.x)
    link_epilogue(a, r, __ldcg(a.Lbuf + r), __ldg(a.deg + r), rho, part, pol_first, pol_last);
  block_sum_store<4>(part, a.k2_part + 4 * blockIdx.x);
  __threadfence();
  if (threadIdx.x == 0) s_last = (atomicAdd(&a.ctrl->ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  last_block_finalize(a, rho, gridDim.x, true);
}

}  // namespace numpmp_dev
