// pmp_p2p.cuh -- the sharded engine's peer-memory exchange (one process per
// GPU on one NVLink/NVSwitch node), fused into the iteration's kernels.
//
// streams (columns of R) are sharded, so each rank holds a
// partial load R_g x_g for every link.  Instead of an all-reduce of the m
// partial loads followed by a replicated link epilogue on every rank, the
// links are owned in contiguous ranges of mo = ceil(m / world):
//
//   k_link_pass<LP_P2P>  every row's local load goes straight from the tail
//                        lane into the owner's slot for this rank (an
//                        NVLink store, overlapped with the remaining
//                        gathers); the last CTA signals "loads stored".
//   k_p2p_wait<0>        1 CTA: waits for all ranks' signals (system-scope
//                        acquire on a local counter).
//   k_p2p_epilogue       the owner sums its links' slots in rank order (a
//                        fixed order: deterministic, identical whatever the
//                        arrival order), runs the link epilogue for its links
//                        only, stores v_l into every rank's v (NVLink), and
//                        the last CTA publishes the rank's residual partials
//                        to every rank and signals "epilogue done".
//   k_p2p_finalize       1 CTA: waits, sums the ranks' partials in rank
//                        order -- the same numbers on every rank, so every
//                        rank takes the same termination / rho decision --
//                        and runs finalize_iteration.
//
// Fused mode (the default when no two ranks share a GPU): the wait and the
// finalize fold into k_p2p_epilogue<true> -- every CTA's thread 0 acquires
// "loads stored" itself and the last CTA waits for "epilogue done" and
// finalizes -- so an iteration is 2 NB + 1 launches, as on one device.
// Ranks sharing a GPU (the one-GPU test boxes) keep the three launches:
// there, a spinning CTA could hold the SMs another rank's link pass needs.
//
// On rho-update iterations the owner also stores v for both candidate rhos
// (rho*gamma, rho/gamma) into every rank; finalize_iteration selects one
// (Ctrl::v_sel), so nothing rebuilds v inside the loop.  Traffic per rank and iteration: 8 (world-1)/world
// bytes per link in each direction, the same as a ring all-reduce, but the
// epilogue work is divided by world and no NCCL kernel sits in the loop.
//
// Ordering (why no buffer is overwritten while it is read): a rank stores
// into a peer's slots only in k_link_pass(k+1), after its finalize(k) saw
// every rank's "epilogue done"(k), which each rank signals after reading its
// slots; v is written in epilogue(k) only after every rank's "loads
// stored"(k), i.e. after every rank's stream passes of iteration k.
//
// Barrier counters are cumulative (flags[i] on the receiving rank, bumped by
// every rank with one fence.acq_rel.sys + red.relaxed.sys); done_cnt[i] counts the barriers of kind
// i this rank has completed, identical on all ranks because every rank runs
// the same sequence: target = world * (done_cnt[i] + 1).
//   flags[0] loads stored / aux push, flags[1] epilogue done / aux result,
//   flags[3] aux buffers free (flags[2] unused).
#pragma once

#include "pmp_kernels.cuh"

namespace numpmp_dev {

constexpr long long kP2PTimeoutNs = 60ll * 1000 * 1000 * 1000;  // a dead peer traps, never hangs

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin until barrier `which` of the current round has every rank's signal.
// Does not count the round as completed (several CTAs may wait on it).
__device__ __forceinline__ void p2p_spin_counter(const P2PArgs& p, int which) {
  const unsigned long long target =
      static_cast<unsigned long long>(p.world) * (p.done_cnt[which] + 1);
  const long long t0 = globaltimer_ns();
  while (ld_acquire_sys(p.flags + which) < target) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > kP2PTimeoutNs) __trap();
  }
}

__device__ __forceinline__ void p2p_wait_counter(const P2PArgs& p, int which) {
  p2p_spin_counter(p, which);
  p.done_cnt[which] += 1;
  __threadfence();
}

__device__ __forceinline__ void p2p_signal_all(const P2PArgs& p, int which) {
  signal_all_sys(p.flags_peer, p.world, which);
}

// ---------------------------------------------------------------- iteration
// After "epilogue done": the ranks' residual partials in rank order (the
// same numbers on every rank), then the device finalize.
__device__ __forceinline__ void p2p_sum_finalize(const IterArgs& a, double rho) {
  const P2PArgs& p = a.p2p;
  double s[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const double* xs = ld_ptr(p.xs_peer + p.rank);
  for (int q = 0; q < p.world; ++q)
    for (int i = 0; i < 7; ++i) s[i] += __ldcg(xs + 8 * q + i);
  finalize_iteration(a, rho, s[0], s[1], s[2], s[3], s[4], s[5], s[6]);
}

template <int kWhich>
__global__ void k_p2p_wait(IterArgs a) {
  if (threadIdx.x != 0) return;
  if (kernel_should_exit(a.ctrl)) return;
  p2p_wait_counter(a.p2p, kWhich);
}

// kFused (one GPU per rank): every CTA's thread 0 waits for "loads stored"
// itself (no k_p2p_wait launch), and the last CTA, after publishing its
// partials, waits for "epilogue done" and runs the finalize (no
// k_p2p_finalize launch).  Only valid when no other rank's kernels need this
// GPU's SMs: a spinning CTA holds its slot.
template <bool kFused>
__global__ void __launch_bounds__(kThreads, NUMPMP_EPI_MINB) k_p2p_epilogue(IterArgs a) {
  __shared__ bool s_last;
  if (kernel_should_exit(a.ctrl)) return;
  const P2PArgs& p = a.p2p;
  if (kFused) {
    if (threadIdx.x == 0) p2p_spin_counter(p, 0);  // the round is counted by the last CTA
    __syncthreads();
  }
  const double rho = a.ctrl->rho;
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  double part[4] = {0.0, 0.0, 0.0, 0.0};
  const double* slots = ld_ptr(p.slots_peer + p.rank);
  // rho-update iteration: v for both candidate rhos too (finalize picks one)
  const bool cand = a.mode == MODE_RUN && (a.ctrl->run_k + 1) % a.rho_interval == 0;
  auto finish = [&](long long l, double L, int d, const LinkIn& in) {
    double Bn, prn;
    const double v = link_update(a, l, L, d, in, rho, part, pol_last, &Bn, &prn);
    const double vu = cand ? Bn + prn / (rho * a.gamma) : 0.0;
    const double vd = cand ? Bn + prn / (rho / a.gamma) : 0.0;
    for (int q = 0; q < p.world; ++q) {
      if (q == p.rank) continue;  // local copies written by link_update
      double* vq = ld_ptr(p.v_peer + q);
      vq[l] = v;
      if (cand) {
        vq[a.m + l] = vu;
        vq[2 * a.m + l] = vd;
      }
    }
  };
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long l = p.l0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; l < p.l1; l += 2 * stride) {
    // two links' loads in flight per thread (same link order as one at a time)
    const long long l1 = l + stride;
    const bool has1 = l1 < p.l1;
    const LinkIn in0 = load_link(a, l, pol_first);
    const int d0 = __ldg(a.deg + l);
    LinkIn in1{};
    int d1 = 0;
    if (has1) {
      in1 = load_link(a, l1, pol_first);
      d1 = __ldg(a.deg + l1);
    }
    double L0 = 0.0, L1 = 0.0;  // the ranks' partial loads, rank order
    for (int q = 0; q < p.world; ++q) {
      L0 += __ldcg(slots + q * p.mo + (l - p.l0));
      if (has1) L1 += __ldcg(slots + q * p.mo + (l1 - p.l0));
    }
    finish(l, L0, d0, in0);
    if (has1) finish(l1, L1, d1, in1);
  }
  block_sum_store<4>(part, p.ep_part + 4 * blockIdx.x);  // ends with bar.sync
  if (threadIdx.x == 0) {  // one cumulative fence per CTA (grid.sync pattern; scope: see k_link_pass LP_P2P)
    if (p.cta_sysfence)
      __threadfence_system();
    else
      __threadfence();
    s_last = (atomicAdd(&a.ctrl->ticket3, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // this rank's six sums, one warp each: the stream passes' (tau dA^2,
  // objective) and the owner epilogue's four -- the fixed orders of
  // last_block_finalize
  static_assert(kWarps >= 6, "one warp per sum");
  __shared__ double sums[6];
  {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double v = 0.0;
    if (wib < 2)
      v = warp_sum_array(a.k1_part, a.grid1 * a.nblocks, 2, wib, lane);
    else if (wib < 6)
      v = warp_sum_array(p.ep_part, gridDim.x, 4, wib - 2, lane);
    if (wib < 6 && lane == 0) sums[wib] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the residual partials and this rank's time-limit flag (finalize sums
    // the flags, so every rank takes the same TimeLimit decision)
    const double row[7] = {sums[0], sums[1], sums[2], sums[3], sums[4], sums[5], time_over_flag(a)};
    for (int q = 0; q < p.world; ++q) {
      double* xs = ld_ptr(p.xs_peer + q) + 8 * p.rank;
      for (int i = 0; i < 7; ++i) xs[i] = row[i];
    }
    a.ctrl->ticket3 = 0;
    if (kFused) {
      p.done_cnt[0] += 1;  // every CTA has passed its wait on barrier 0
      __threadfence();
    }
    p2p_signal_all(p, 1);
    if (kFused) {
      p2p_wait_counter(p, 1);
      p2p_sum_finalize(a, rho);
    }
  }
}

__global__ void k_p2p_finalize(IterArgs a) {
  if (threadIdx.x != 0) return;
  if (kernel_should_exit(a.ctrl)) return;
  p2p_wait_counter(a.p2p, 1);
  p2p_sum_finalize(a, a.ctrl->rho);
}

// ------------------------------------------------- collectives (setup/post)
// Used outside the iteration loop (degrees at connect, R x for warm starts
// and post-processing, the owners' link state after a run).  Each is
// push -> barrier -> combine -> barrier "buffers free".
__global__ void k_p2p_aux_wait(P2PArgs p, int which) {
  if (blockIdx.x == 0 && threadIdx.x == 0) p2p_wait_counter(p, which);
}
__global__ void k_p2p_aux_signal(P2PArgs p, int which) {
  if (blockIdx.x == 0 && threadIdx.x == 0) p2p_signal_all(p, which);
}
// src[m] -> owners' slots [rank][local] (reduce layout)
__global__ void k_p2p_push_partials(P2PArgs p, const double* __restrict__ src, long long m) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
       l += (long long)gridDim.x * blockDim.x) {
    const long long q = l / p.mo;
    ld_ptr(p.slots_peer + q)[p.rank * p.mo + (l - q * p.mo)] = src[l];
  }
  __threadfence_system();
}
// owner: sum of the ranks' partials (rank order) -> every rank's v
__global__ void k_p2p_reduce_bcast(P2PArgs p) {
  const double* slots = ld_ptr(p.slots_peer + p.rank);
  for (long long l = p.l0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; l < p.l1;
       l += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < p.world; ++q) s += __ldcg(slots + q * p.mo + (l - p.l0));
    for (int q = 0; q < p.world; ++q) ld_ptr(p.v_peer + q)[l] = s;
  }
  __threadfence_system();
}
// owner's links of src -> every rank's slots, global link layout (gather)
__global__ void k_p2p_push_owned(P2PArgs p, const double* __restrict__ src) {
  for (long long l = p.l0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; l < p.l1;
       l += (long long)gridDim.x * blockDim.x) {
    const double x = src[l];
    for (int q = 0; q < p.world; ++q) ld_ptr(p.slots_peer + q)[l] = x;
  }
  __threadfence_system();
}
// k scalars of this rank -> every rank's xs row `rank`
__global__ void k_p2p_push_scalars(P2PArgs p, const double* __restrict__ src, int k) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int q = 0; q < p.world; ++q) {
    double* xs = ld_ptr(p.xs_peer + q) + 8 * p.rank;
    for (int i = 0; i < k; ++i) xs[i] = src[i];
  }
  __threadfence_system();
}
__global__ void k_p2p_sum_scalars(P2PArgs p, double* __restrict__ dst, int k) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const double* xs = ld_ptr(p.xs_peer + p.rank);
  for (int i = 0; i < k; ++i) {
    double s = 0.0;
    for (int q = 0; q < p.world; ++q) s += __ldcg(xs + 8 * q + i);
    dst[i] = s;
  }
}

}  // namespace numpmp_dev
