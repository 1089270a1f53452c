// dsmem_bench.cu -- the bounded experiment on the L1->L2 request ceiling
// ("next round" item 5): can a thread-block cluster turn the
// stream pass's random v gathers into (a) gathers of link-SORTED indices
// (several values per L2 request) plus (b) random 8-byte scatters into
// distributed shared memory, faster than one L2 request per nonzero?
//
// Part 1: random 8-byte accesses to shared memory, per SM:
//   mode 0: st.shared::cluster to a random CTA of the cluster (DSMEM scatter)
//   mode 1: st.shared to a random local address
//   mode 2: ld.shared from a random local address
//   mode 3: ld.shared::cluster from a random CTA of the cluster
// Part 2: gathers v[idx[k]] (v = 1M doubles, 8 MB, L2-resident) with the
//   index stream coalesced, idx sorted within tiles of T entries (density
//   T/m per link) vs unsorted.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dsmem_bench scripts/dsmem_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

namespace cg = cooperative_groups;

constexpr int kSmemD = 16384;  // doubles per CTA (128 KB)

template <int MODE>
__global__ void k_dsmem(int iters, double* sink) {
  extern __shared__ double buf[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned cs = cl.num_blocks();
  for (int i = threadIdx.x; i < kSmemD; i += blockDim.x) buf[i] = 0.0;
  cl.sync();
  unsigned h = (blockIdx.x * 1024u + threadIdx.x) * 2654435761u + 12345u;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      const unsigned off = (h >> 8) & (kSmemD - 1);
      const unsigned tgt = (h >> 24) % cs;
      if (MODE == 0) {
        double* p = cl.map_shared_rank(buf, tgt);
        p[off] = (double)it;
      } else if (MODE == 1) {
        buf[off] = (double)it;
      } else if (MODE == 2) {
        acc += buf[off];
      } else {
        const double* p = cl.map_shared_rank(buf, tgt);
        acc += p[off];
      }
    }
  }
  cl.sync();
  if (acc == 1.2345 || buf[threadIdx.x] == 1.2345) sink[0] = acc;
}

template <int U>
__global__ void k_gather(const int* __restrict__ idx, long long n, const double* __restrict__ src,
                         double* sink) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (long long r = warp; r * 32 * U < n; r += nwarps) {
    const long long b = r * 32 * U + lane;
    int id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) id[u] = (b + 32 * u < n) ? __ldg(idx + b + 32 * u) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(src + id[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"remote st (DSMEM scatter)", "local st", "local ld", "remote ld (DSMEM gather)"};
  for (int mode = 0; mode < 4; ++mode) {
    void (*fn)(int, double*) = mode == 0 ? k_dsmem<0> : mode == 1 ? k_dsmem<1> : mode == 2 ? k_dsmem<2> : k_dsmem<3>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemD * 8);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
      if ((mode == 1 || mode == 2) && cs > 1) continue;
      for (int threads : {256, 512, 1024}) {
        const int iters = 256;
        const int grid = (sms / cs) * cs * 2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = kSmemD * 8;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
        float best = 1e9, ms;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(e0);
          cudaLaunchKernelEx(&cfg, fn, iters, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
          best = std::min(best, ms);
        }
        const double ops = (double)grid * threads * iters * 8;
        // grid = 2 waves of the resident CTAs (1 CTA per SM at 128 KB)
        const double active_sms = std::min<double>(grid / 2.0, (double)ncl * cs);
        printf("%-28s cluster=%2d threads=%4d active_clusters=%3d: %.3f ms  %.1f G ops/s  %.2f ops/clk/SM (at %d MHz, %d SMs)\n",
               names[mode], cs, threads, ncl, best, ops / (best * 1e-3) / 1e9,
               ops / (best * 1e-3) / (active_sms * clk * 1e3), clk / 1000, (int)active_sms);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));

  // Part 2: sorted-tile gathers
  const long long n = 100000000, m = 1000000;
  int* idx;
  double* src;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&src, m * 8);
  cudaMemset(src, 0, m * 8);
  std::vector<int> h(n);
  std::mt19937_64 rng(7);
  for (long long T : {0LL, 100000LL, 200000LL, 400000LL, 800000LL}) {
    for (long long i = 0; i < n; ++i) h[i] = (int)(rng() % m);
    if (T > 0)
      for (long long b = 0; b < n; b += T) std::sort(h.begin() + b, h.begin() + std::min(n, b + T));
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int occ : {4, 8}) {
      float best = 1e9, ms;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k_gather<8><<<sms * occ, 256>>>(idx, n, src, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      printf("gather v (1M doubles), idx sorted in tiles of %7lld (density %.2f/link), blocks/SM=%d: %.3f ms -> %.1f G gathers/s\n",
             T, T / (double)m, occ, best, n / (best * 1e-3) / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
