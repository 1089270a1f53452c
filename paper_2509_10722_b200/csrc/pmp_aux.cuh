// pmp_aux.cuh -- setup / state-materialisation / post-processing kernels.
// None of these run inside the iteration loop.
#pragma once

#include "pmp_kernels.cuh"

namespace numpmp_dev {

// Model validation on the device (the rules of model.hpp:76-135): one
// counter per rule; any nonzero count sends the caller to the host
// validator, which produces the reference's exact message.
//   bad[0] capacity, bad[1] empty route / offsets, bad[2] link out of range,
//   bad[3] duplicate link, bad[4] weight, bad[5] kind
__global__ void k_validate(const long long* __restrict__ off, const int* __restrict__ links,
                           const double* __restrict__ w, const unsigned char* __restrict__ kind,
                           const double* __restrict__ cap, long long n, long long m,
                           unsigned long long* __restrict__ bad) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  for (long long l = tid; l < m; l += stride) {
    const double v = cap[l];
    if (!(v > 0.0) || !isfinite(v)) ++c[0];
  }
  for (long long j = tid; j < n; j += stride) {
    const long long b = off[j], e = off[j + 1];
    if (e <= b) ++c[1];
    // range check + strictly-increasing check in one pass (generated and
    // most real routes are sorted); only an unsorted route pays the
    // quadratic duplicate search.  Counts are flags: any nonzero count sends
    // the caller to the host validator for the exact message.
    bool sorted = true;
    int prev = -1;
    for (long long t = b; t < e; ++t) {
      const int l = links[t];
      if (l < 0 || l >= m) ++c[2];
      if (l <= prev) sorted = false;
      prev = l;
    }
    if (!sorted)
      for (long long t = b; t < e; ++t) {
        const int l = links[t];
        for (long long u = b; u < t; ++u)
          if (links[u] == l) {
            ++c[3];
            break;
          }
      }
    const double wj = w[j];
    const int k = kind[j];
    if (!isfinite(wj) || (k == NUMPMP_KIND_LOG && !(wj > 0.0)) || (k != NUMPMP_KIND_LOG && wj < 0.0))
      ++c[4];
    if (k >= NUMPMP_KIND_EXTENSION) ++c[5];  // extension (or unknown) utility
  }
#pragma unroll
  for (int i = 0; i < 6; ++i)
    if (c[i]) atomicAdd(bad + i, c[i]);
}

// int64 stream offsets -> int32 CSC column pointer (nnz < 2^31 checked on host).
__global__ void k_offsets_to_i32(const long long* __restrict__ in, int* __restrict__ out,
                                 long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = static_cast<int>(in[i]);
}

// terminal -> (global) stream map for the streams col_ptr[0..n) (absolute
// terminal ids), and the terminal iota used as sort values.
__global__ void k_terminal_stream(const int* __restrict__ col_ptr, long long n, long long s0,
                                  int* __restrict__ t2s) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const int b = col_ptr[j], e = col_ptr[j + 1];
    for (int t = b; t < e; ++t) t2s[t] = static_cast<int>(s0 + j);
  }
}
__global__ void k_iota(int* __restrict__ out, long long count, long long base) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = static_cast<int>(base + i);
}
__global__ void k_add_degree(const int* __restrict__ row_ptr, long long m, int* __restrict__ deg) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x)
    deg[l] += row_ptr[l + 1] - row_ptr[l];
}
// Row pointer from the link-sorted keys: row_ptr[l] = first k with key >= l.
__global__ void k_row_ptr_from_sorted(const int* __restrict__ keys, long long nnz, long long m,
                                      int* __restrict__ row_ptr) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int cur = (k < nnz) ? keys[k] : static_cast<int>(m);
    const int prev = (k > 0) ? keys[k - 1] : -1;
    for (int l = prev + 1; l <= cur; ++l) row_ptr[l] = static_cast<int>(k);
  }
}
__global__ void k_gather_i32(const int* __restrict__ src, const int* __restrict__ idx,
                             int* __restrict__ out, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}
__global__ void k_degree(const int* __restrict__ row_ptr, long long m, int* __restrict__ deg) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x)
    deg[l] = row_ptr[l + 1] - row_ptr[l];
}

// Column-block segmentation of the link-major CSR (k_link_pass): link l
// with d entries in the block gets max(1, ceil(d / seg)) segments of
// near-equal size.  nseg[l] -> (exclusive scan) row_vstart; then each link
// writes its segments' CSR starts and its id.
__global__ void k_seg_count(const int* __restrict__ row_ptr, long long m, int seg,
                            int* __restrict__ nseg) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    const int d = row_ptr[l + 1] - row_ptr[l];
    nseg[l] = max(1, (d + seg - 1) / seg);
  }
}
__global__ void k_seg_fill(const int* __restrict__ row_ptr, const int* __restrict__ row_vstart,
                           long long m, int* __restrict__ vptr, int* __restrict__ vrow) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    const int b = row_ptr[l], d = row_ptr[l + 1] - b;
    const int v0 = row_vstart[l], ns = row_vstart[l + 1] - v0;
    for (int s = 0; s < ns; ++s) {
      vptr[v0 + s] = b + static_cast<int>((static_cast<long long>(s) * d) / ns);
      vrow[v0 + s] = static_cast<int>(l);
    }
    if (l == m - 1) vptr[v0 + ns] = b + d;
  }
}
__global__ void k_max_degree(const int* __restrict__ row_ptr, long long m, int* __restrict__ out) {
  int mx = 0;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x)
    mx = max(mx, row_ptr[l + 1] - row_ptr[l]);
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// warm_start_from (solver.hpp:218-259) in link space, given L = R x0:
// slack = max(c - L, 0); ps = slack - c; pbar = (L + ps)/(d+1);
// A = x0 (done by the caller), B = pbar, zs = ps - pbar, Q = L.
__global__ void k_warm_links(const double* __restrict__ L, const int* __restrict__ deg,
                             const int* __restrict__ row_ptr, const double* __restrict__ cap,
                             long long m, double* __restrict__ B, double* __restrict__ zs,
                             double* __restrict__ Q, double* __restrict__ ps0,
                             double* __restrict__ pbar0) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    const double c = cap[l];
    const double load = L[l];
    const double slack = dmax_ref(c - load, 0.0);
    const double ps = slack - c;
    const int d = deg ? deg[l] : row_ptr[l + 1] - row_ptr[l];
    const double pbar = (load + ps) / static_cast<double>(d + 1);
    B[l] = pbar;
    zs[l] = ps - pbar;
    Q[l] = load;
    ps0[l] = ps;
    pbar0[l] = pbar;
  }
}

// Link part of state materialisation after >= 1 iteration: the slack flow
// and link average of the last iteration, recomputed with the identical
// arithmetic from the previous-iterate buffers.
__global__ void k_materialize_links(const double* __restrict__ L, const int* __restrict__ deg,
                                    const int* __restrict__ row_ptr,
                                    const double* __restrict__ cap,
                                    const double* __restrict__ zs_prev,
                                    const double* __restrict__ pr_prev, double rho_iter,
                                    long long m, double* __restrict__ ps,
                                    double* __restrict__ pbar) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    const double u = pr_prev[l] / rho_iter;
    const double p = dmax_ref(zs_prev[l] - u, -cap[l]);
    const int d = deg ? deg[l] : row_ptr[l + 1] - row_ptr[l];
    ps[l] = p;
    pbar[l] = (L[l] + p) / static_cast<double>(d + 1);
  }
}

// Terminal-space expansion: p_t = x_j, z_t = A_j - B_l (and the previous
// iterate's copies) for traffic terminals.
__global__ void k_expand_terminals(const int* __restrict__ col_ptr, const int* __restrict__ row_idx,
                                   long long n, const double* __restrict__ x,
                                   const double* __restrict__ A, const double* __restrict__ B,
                                   const double* __restrict__ A_prev,
                                   const double* __restrict__ B_prev, double* __restrict__ p,
                                   double* __restrict__ z, double* __restrict__ z_prev) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const int b = col_ptr[j], e = col_ptr[j + 1];
    for (int t = b; t < e; ++t) {
      const int l = row_idx[t];
      if (p) p[t] = x[j];
      if (z) z[t] = A[j] - B[l];
      if (z_prev) z_prev[t] = A_prev[j] - B_prev[l];
    }
  }
}

// Post-processing (solver.hpp:483-504): x clamp of tiny negatives, lambda,
// lambda_raw; objective partials (clamped for Solution.objective,
// unclamped for the final trace row).
__global__ void __launch_bounds__(kThreads) k_post_streams(const double* __restrict__ x,
                                                           const double* __restrict__ w,
                                                           const unsigned char* __restrict__ kind,
                                                           long long n, double eps_abs,
                                                           double* __restrict__ x_sol,
                                                           double* __restrict__ part) {
  double v[2] = {0.0, 0.0};
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const double xj = x[j];
    const double xc = (xj < 0.0 && -xj < eps_abs) ? 0.0 : xj;
    x_sol[j] = xc;
    const bool lg = kind[j] == NUMPMP_KIND_LOG;
    v[0] += lg ? w[j] * log(xc) : w[j] * xc;
    v[1] += lg ? w[j] * log(xj) : w[j] * xj;
  }
  block_sum_store<2>(v, part + 2 * blockIdx.x);
}
__global__ void k_post_links(const double* __restrict__ L, const double* __restrict__ cap,
                             const double* __restrict__ price, long long m,
                             double* __restrict__ s, double* __restrict__ lambda) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    s[l] = dmax_ref(cap[l] - L[l], 0.0);
    lambda[l] = dmax_ref(price[l], 0.0);
  }
}
__global__ void k_sum_parts(const double* __restrict__ part, int count, double* __restrict__ out) {
  const double a = block_sum_array(part, count, 2, 0);
  const double b = block_sum_array(part, count, 2, 1);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

__global__ void k_start_clock(Ctrl* c) { c->t0_ns = globaltimer_ns(); }

// residuals() (solver.hpp:139-154) on terminal-space device arrays: per-CTA
// partials of r^2 = sum_l |l| pbar_l^2 (|l| = deg + 1) and
// s^2 = sum_t (rho (z_t - z'_t))^2 over a fixed grid-stride mapping, summed
// in CTA order by k_sum_parts.  Launched with the same shape on every call,
// so the result is a function of the arrays alone: numpmp_gpu_step returns
// exactly what numpmp_gpu_residuals computes from the states it issued.
constexpr int kResidualGrid = 4 * 148;
__global__ void __launch_bounds__(kThreads) k_residual_parts(const double* __restrict__ pbar,
                                                             const int* __restrict__ deg, long long m,
                                                             const double* __restrict__ z,
                                                             const double* __restrict__ zp, long long J,
                                                             double rho, double* __restrict__ part) {
  double v[2] = {0.0, 0.0};
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m; l += stride) {
    const double pb = pbar[l];
    v[0] += static_cast<double>(deg[l] + 1) * pb * pb;
  }
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < J; t += stride) {
    const double d = rho * (z[t] - zp[t]);
    v[1] += d * d;
  }
  block_sum_store<2>(v, part + 2 * blockIdx.x);
}

// ---------------------------------------------- warm-start recipes (warm.hpp)
// ratio_l = c_after / c_before; price_l = lambda_raw_l / ratio_l (warm.hpp:29-51).
__global__ void k_degrade_links(const double* __restrict__ cap_after, long long m,
                                double* __restrict__ ratio, double* __restrict__ price) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    const double r = cap_after[l] / ratio[l];
    ratio[l] = r;
    price[l] = price[l] / r;
  }
}
// x0_j *= min over the route of ratio (std::min, route order); log streams
// floored at 1e-8 (warm.hpp:42-49).
__global__ void k_route_min_scale(const int* __restrict__ col_ptr, const int* __restrict__ row_idx,
                                  long long n, const double* __restrict__ ratio,
                                  const unsigned char* __restrict__ kind, double* __restrict__ x) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    double cut = 1.0;
    for (int t = col_ptr[j]; t < col_ptr[j + 1]; ++t) {
      const double r = ratio[row_idx[t]];
      cut = (r < cut) ? r : cut;
    }
    double v = x[j] * cut;
    if (kind[j] == NUMPMP_KIND_LOG && !(v > 0.0)) v = 1e-8;
    x[j] = v;
  }
}
// transit.hpp:290-302 path_prices: pi_j = sum of lambda along the route, in
// route order.
__global__ void k_path_prices(const int* __restrict__ col_ptr, const int* __restrict__ row_idx,
                              long long n, const double* __restrict__ lambda, double* __restrict__ pi) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    double total = 0.0;
    for (int t = col_ptr[j]; t < col_ptr[j + 1]; ++t) total += lambda[row_idx[t]];
    pi[j] = total;
  }
}
// warm.hpp:73-82: price_l *= min(1, load_l / c_l); clamped = max(price, 0).
__global__ void k_prune_prices(const double* __restrict__ load, const double* __restrict__ cap,
                               long long m, double* __restrict__ price, double* __restrict__ clamped) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    const double f = load[l] / cap[l];
    const double p = price[l] * ((f < 1.0) ? f : 1.0);
    price[l] = p;
    clamped[l] = (p < 0.0) ? 0.0 : p;
  }
}
// warm.hpp:84-91: log streams re-centred on the path price.
__global__ void k_recenter_log(const double* __restrict__ pi, const double* __restrict__ w,
                               const unsigned char* __restrict__ kind, long long n,
                               double* __restrict__ x) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    if (kind[j] != NUMPMP_KIND_LOG) continue;
    double v = x[j];
    if (pi[j] > 1e-10) v = w[j] / pi[j];
    if (!(v > 0.0)) v = 1e-8;
    x[j] = v;
  }
}
// Per-link sums in ascending stream order over the column blocks' CSRs (one
// accumulator per link, the reference's loop order).
struct BlockCsrs {
  const int* row_ptr[kMaxBlocks];
  const int* col_idx[kMaxBlocks];
  int nblocks;
};
__global__ void k_row_sums_seq(BlockCsrs bc, long long m, const double* __restrict__ src,
                               double* __restrict__ out) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < bc.nblocks; ++b)
      for (int k = bc.row_ptr[b][l]; k < bc.row_ptr[b][l + 1]; ++k) acc += src[bc.col_idx[b][k]];
    out[l] = acc;
  }
}

__global__ void k_int_to_double(const int* __restrict__ in, long long count, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}
__global__ void k_double_to_int(const double* __restrict__ in, long long count, int* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = static_cast<int>(in[i]);
}

}  // namespace numpmp_dev
