// gather_bench.cu -- microbenchmark of the two memory rates that bound the
// PMP passes on B200: HBM streaming (int4 loads) and random 8-byte gathers
// from an L2-resident vector (v: 8 MB; x: 80 MB).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_stream(const int4* __restrict__ a, long long n4, int4* __restrict__ sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    int4 v = __ldg(a + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

template <int U>
__global__ void k_gather(const int* __restrict__ idx, long long n, const double* __restrict__ src, double* sink) {
  double acc = 0.0;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    int id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) id[u] = (i + u * stride < n) ? __ldg(idx + i + u * stride) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __ldg(src + id[u]);
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  const long long nidx = 100000000;
  int* idx; double* src; double* sink; int4* big;
  cudaMalloc(&idx, nidx * 4);
  cudaMalloc(&src, 10000000LL * 8);
  cudaMalloc(&sink, 64);
  const long long bigb = 2LL << 30;
  cudaMalloc(&big, bigb);
  cudaMemset(big, 1, bigb);
  cudaMemset(src, 0, 10000000LL * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // HBM stream
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_stream<<<sms * 8, 256>>>(big, bigb / 16, (int4*)sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("hbm_stream_read_GBs %.1f\n", bigb / (ms * 1e-3) / 1e9);
  for (long long range : {1000000LL, 10000000LL}) {
    std::vector<int> h(nidx);
    unsigned long long s = 88172645463325252ULL;
    for (long long i = 0; i < nidx; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % range); }
    cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
    for (int occ : {4, 8, 16}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_gather<8><<<sms * occ, 256>>>(idx, nidx, src, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("gather range=%lld MB=%lld blocks/SM=%d: %.3f ms for 1e8 -> %.1f Ggathers/s (idx stream %.0f GB/s)\n",
             range, range * 8 / 1000000, occ, ms, nidx / (ms * 1e-3) / 1e9, nidx * 4 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
