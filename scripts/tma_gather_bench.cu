// tma_gather_bench.cu -- can TMA tile::gather4 (sm_100a) beat LSU gathers?
// Random 8-byte gathers from a vector of N doubles, three ways:
//   (1) LDG per lane (the production path),
//   (2) TMA gather4: the vector viewed as rows of 2 doubles (16 B, the TMA
//       minimum); one elected lane per warp issues 32 gather4 per 128
//       indices into shared memory, completion on an mbarrier,
//   (3) cp.async (LDGSTS) 8 B per lane into shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather_bench tma_gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_ldg(const int* __restrict__ idx, long long n, const double* __restrict__ src, double* sink) {
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride * 4) {
    int id[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) id[u] = (i + u * stride < n) ? __ldg(idx + i + u * stride) : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += __ldg(src + id[u]);
  }
  if (acc == 1.2345) sink[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int WARPS = 4;
constexpr int BATCH = 128;   // indices per warp per round
constexpr int STAGES = 2;

// (2) TMA gather4.  Each warp: rounds of 128 indices; lane 0 arms the
// mbarrier with expect_tx(128*16 B) and issues 32 gather4; all lanes wait,
// then each lane reads its 4 values from shared memory.
__global__ void __launch_bounds__(WARPS * 32) k_tma(const __grid_constant__ CUtensorMap tmap,
                                                   const int* __restrict__ idx, long long n,
                                                   double* sink) {
  __shared__ __align__(128) double buf[WARPS][STAGES][BATCH * 4];  // 128-B aligned gather4 slots
  __shared__ __align__(8) uint64_t bar[WARPS][STAGES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  double acc = 0.0;
  const long long nrounds = n / BATCH;
  const long long gw = (long long)blockIdx.x * WARPS + w, nw = (long long)gridDim.x * WARPS;
  uint32_t phase[STAGES] = {0, 0};
  auto issue = [&](long long r, int s) {
    // lane l owns indices 4l..4l+3 of the round
    const int4 ids = *reinterpret_cast<const int4*>(idx + r * BATCH + 4 * lane);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][s])),
                   "r"(BATCH * 16) : "memory");
    __syncwarp();
    // rows = id >> 1 ; every lane issues its own gather4 (4 rows)
    const uint32_t dst = smem_u32(&buf[w][s][16 * lane]);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(&tmap), "r"(0), "r"(ids.x >> 1),
        "r"(ids.y >> 1), "r"(ids.z >> 1), "r"(ids.w >> 1), "r"(smem_u32(&bar[w][s]))
        : "memory");
    return ids;
  };
  long long r = gw;
  int4 cur_ids = make_int4(0, 0, 0, 0);
  if (r < nrounds) cur_ids = issue(r, 0);
  int s = 0;
  while (r < nrounds) {
    const long long rn = r + nw;
    int4 nxt_ids = make_int4(0, 0, 0, 0);
    if (rn < nrounds) nxt_ids = issue(rn, s ^ 1);
    // wait for stage s
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[w][s])), "r"(phase[s]) : "memory");
    }
    phase[s] ^= 1;
    const double* row = &buf[w][s][16 * lane];
    acc += row[0 + (cur_ids.x & 1)] + row[2 + (cur_ids.y & 1)] + row[4 + (cur_ids.z & 1)] +
           row[6 + (cur_ids.w & 1)];
    __syncwarp();
    cur_ids = nxt_ids;
    r = rn;
    s ^= 1;
  }
  if (acc == 1.2345) sink[0] = acc;
}

// (3) cp.async 8 B per lane into shared memory (LDGSTS)
__global__ void __launch_bounds__(WARPS * 32) k_cpasync(const int* __restrict__ idx, long long n,
                                                       const double* __restrict__ src, double* sink) {
  __shared__ __align__(16) double buf[WARPS][BATCH];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  const long long nrounds = n / BATCH;
  for (long long r = (long long)blockIdx.x * WARPS + w; r < nrounds; r += (long long)gridDim.x * WARPS) {
    const int4 ids = *reinterpret_cast<const int4*>(idx + r * BATCH + 4 * lane);
    const int e[4] = {ids.x, ids.y, ids.z, ids.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&buf[w][4 * lane + q])),
                   "l"(src + e[q]) : "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    acc += buf[w][4 * lane] + buf[w][4 * lane + 1] + buf[w][4 * lane + 2] + buf[w][4 * lane + 3];
    __syncwarp();
  }
  if (acc == 1.2345) sink[0] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long n = 100000000;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* idx;
  double* src;
  double* sink;
  CK(cudaMalloc(&idx, n * 4));
  CK(cudaMalloc(&src, 10000000LL * 8));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(src, 0, 10000000LL * 8));
  EncodeTiled encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (long long range : {1000000LL, 10000000LL}) {
    std::vector<int> h(n);
    unsigned long long s = 88172645463325252ULL;
    for (long long i = 0; i < n; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % range);
    }
    CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    CUtensorMap tmap;
    cuuint64_t dims[2] = {2, (cuuint64_t)(range / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
    for (int occ : {4, 8}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_ldg<<<sms * occ, 256>>>(idx, n, src, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("range %lld LDG   blocks/SM=%d: %.3f ms -> %.1f G/s\n", range, occ, ms, n / (ms * 1e-3) / 1e9);
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_tma<<<sms * occ, WARPS * 32>>>(tmap, idx, n, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      }
      CK(cudaGetLastError());
      printf("range %lld TMA4  blocks/SM=%d: %.3f ms -> %.1f G/s\n", range, occ, ms, n / (ms * 1e-3) / 1e9);
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_cpasync<<<sms * occ, WARPS * 32>>>(idx, n, src, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      }
      CK(cudaGetLastError());
      printf("range %lld CPASY blocks/SM=%d: %.3f ms -> %.1f G/s\n", range, occ, ms, n / (ms * 1e-3) / 1e9);
    }
  }
  // correctness of the TMA path on a small case
  return 0;
}
