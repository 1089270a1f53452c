// gather_lanes_bench.cu -- does the B200 random-gather rate depend on how
// many lanes of a warp are active per gather instruction?
// 1e8 random 8-byte gathers from an L2-resident vector (1M doubles), issued
// by warps with only `act` of 32 lanes active (the others predicated off),
// `unroll` gathers in flight per lane.  Same total gathers for every case.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_lanes_bench scripts/gather_lanes_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

template <int U>
__global__ void k_gather(const int* __restrict__ idx, long long n, const double* __restrict__ src, int act,
                         double* sink) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long per_round = (long long)act * U;
  double acc = 0.0;
  if (lane < act) {
    for (long long r = warp; r * per_round < n; r += nwarps) {
      const long long b = r * per_round + lane;
      int id[U];
#pragma unroll
      for (int u = 0; u < U; ++u) id[u] = (b + u * act < n) ? __ldg(idx + b + u * act) : 0;
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(src + id[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u];
    }
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  const long long n = 100000000, range = 1000000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* idx;
  double *src, *sink;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&src, range * 8);
  cudaMalloc(&sink, 64);
  cudaMemset(src, 0, range * 8);
  std::vector<int> h(n);
  unsigned long long s = 88172645463325252ULL;
  for (long long i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = (int)(s % range);
  }
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int occ : {4, 8}) {
    for (int act : {32, 24, 19, 16, 8}) {
      for (int U : {4, 8}) {
        float best = 1e9, ms;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(e0);
          if (U == 4) k_gather<4><<<sms * occ, 256>>>(idx, n, src, act, sink);
          else k_gather<8><<<sms * occ, 256>>>(idx, n, src, act, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        printf("blocks/SM=%d active lanes=%2d unroll=%d: %.3f ms -> %.1f G gathers/s\n", occ, act, U, best,
               n / (best * 1e-3) / 1e9);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
