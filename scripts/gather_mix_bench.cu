// gather_mix_bench.cu -- do the B200's gather engines add up?
// Random 8-byte gathers from a vector of R doubles, split between three
// engines inside ONE kernel (warp roles), to see whether the TMA gather4
// path and the texture path run beside the LSU (LDG) path or share its
// L1TEX data-stage wavefronts:
//   LDG : ld.global.nc per lane (the production path),
//   TMA : cp.async.bulk.tensor.2d tile::gather4 (16-B rows) into smem,
//   TEX : tex1Dfetch<int2> on a linear texture object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_mix_bench scripts/gather_mix_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int WARPS = 8;
constexpr int BATCH = 128;  // indices per warp per round
constexpr int STAGES = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct Roles {
  int ldg, tma, tex;          // warps per block of each role (sum = WARPS)
  long long n_ldg, n_tma, n_tex;  // rounds of BATCH indices per role
};

__global__ void __launch_bounds__(WARPS * 32) k_mix(const __grid_constant__ CUtensorMap tmap,
                                                   cudaTextureObject_t tex, const int* __restrict__ idx,
                                                   const double* __restrict__ src, Roles ro, double* sink) {
  extern __shared__ __align__(128) double dyn[];
  double (*buf)[STAGES][BATCH * 4] = reinterpret_cast<double (*)[STAGES][BATCH * 4]>(dyn);
  __shared__ __align__(8) uint64_t bar[WARPS][STAGES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  if (w < ro.ldg) {
    const long long gw = (long long)blockIdx.x * ro.ldg + w, nw = (long long)gridDim.x * ro.ldg;
    const int* base = idx;
    for (long long r = gw; r < ro.n_ldg; r += 2 * nw) {
      const int4 a = *reinterpret_cast<const int4*>(base + r * BATCH + 4 * lane);
      int4 b = make_int4(0, 0, 0, 0);
      const bool hb = r + nw < ro.n_ldg;
      if (hb) b = *reinterpret_cast<const int4*>(base + (r + nw) * BATCH + 4 * lane);
      double v0 = __ldg(src + a.x), v1 = __ldg(src + a.y), v2 = __ldg(src + a.z), v3 = __ldg(src + a.w);
      double v4 = 0, v5 = 0, v6 = 0, v7 = 0;
      if (hb) { v4 = __ldg(src + b.x); v5 = __ldg(src + b.y); v6 = __ldg(src + b.z); v7 = __ldg(src + b.w); }
      acc += v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7;
    }
  } else if (w < ro.ldg + ro.tma) {
    const int tw = w - ro.ldg;
    const int* base = idx + ro.n_ldg * BATCH;
    if (lane == 0)
      for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long long gw = (long long)blockIdx.x * ro.tma + tw, nw = (long long)gridDim.x * ro.tma;
    uint32_t phase[STAGES] = {0, 0};
    auto issue = [&](long long r, int s) {
      const int4 ids = *reinterpret_cast<const int4*>(base + r * BATCH + 4 * lane);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][s])),
                     "r"(BATCH * 16) : "memory");
      __syncwarp();
      const uint32_t dst = smem_u32(&buf[w][s][16 * lane]);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(&tmap), "r"(0), "r"(ids.x >> 1),
          "r"(ids.y >> 1), "r"(ids.z >> 1), "r"(ids.w >> 1), "r"(smem_u32(&bar[w][s]))
          : "memory");
      return ids;
    };
    long long r = gw;
    int4 cur = make_int4(0, 0, 0, 0);
    if (r < ro.n_tma) cur = issue(r, 0);
    int s = 0;
    while (r < ro.n_tma) {
      const long long rn = r + nw;
      int4 nxt = make_int4(0, 0, 0, 0);
      if (rn < ro.n_tma) nxt = issue(rn, s ^ 1);
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(&bar[w][s])), "r"(phase[s]) : "memory");
      phase[s] ^= 1;
      const double* row = &buf[w][s][16 * lane];
      acc += row[0 + (cur.x & 1)] + row[2 + (cur.y & 1)] + row[4 + (cur.z & 1)] + row[6 + (cur.w & 1)];
      __syncwarp();
      cur = nxt;
      r = rn;
      s ^= 1;
    }
  } else {
    const int xw = w - ro.ldg - ro.tma;
    const int* base = idx + (ro.n_ldg + ro.n_tma) * BATCH;
    const long long gw = (long long)blockIdx.x * ro.tex + xw, nw = (long long)gridDim.x * ro.tex;
    for (long long r = gw; r < ro.n_tex; r += 2 * nw) {
      const int4 a = *reinterpret_cast<const int4*>(base + r * BATCH + 4 * lane);
      int4 b = make_int4(0, 0, 0, 0);
      const bool hb = r + nw < ro.n_tex;
      if (hb) b = *reinterpret_cast<const int4*>(base + (r + nw) * BATCH + 4 * lane);
      int2 t0 = tex1Dfetch<int2>(tex, a.x), t1 = tex1Dfetch<int2>(tex, a.y), t2 = tex1Dfetch<int2>(tex, a.z),
           t3 = tex1Dfetch<int2>(tex, a.w);
      int2 t4 = make_int2(0, 0), t5 = t4, t6 = t4, t7 = t4;
      if (hb) { t4 = tex1Dfetch<int2>(tex, b.x); t5 = tex1Dfetch<int2>(tex, b.y); t6 = tex1Dfetch<int2>(tex, b.z); t7 = tex1Dfetch<int2>(tex, b.w); }
      acc += __hiloint2double(t0.y, t0.x) + __hiloint2double(t1.y, t1.x) + __hiloint2double(t2.y, t2.x) +
             __hiloint2double(t3.y, t3.x) + __hiloint2double(t4.y, t4.x) + __hiloint2double(t5.y, t5.x) +
             __hiloint2double(t6.y, t6.x) + __hiloint2double(t7.y, t7.x);
    }
  }
  if (acc == 1.2345) sink[0] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long n = 100000000;  // gathers per launch (multiple of BATCH)
  const long long rounds = n / BATCH;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* idx;
  double* src;
  double* sink;
  const long long maxr = 10000000;
  CK(cudaMalloc(&idx, n * 4));
  CK(cudaMalloc(&src, maxr * 8));
  CK(cudaMalloc(&sink, 64));
  {
    std::vector<double> hs(maxr);
    for (long long i = 0; i < maxr; ++i) hs[i] = 1e-9 * (double)(i % 1000);
    CK(cudaMemcpy(src, hs.data(), maxr * 8, cudaMemcpyHostToDevice));
  }
  EncodeTiled encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int dyn_bytes = WARPS * STAGES * BATCH * 4 * 8;
  CK(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_bytes));
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = src;
  rd.res.linear.desc = cudaCreateChannelDesc<int2>();
  rd.res.linear.sizeInBytes = maxr * 8;
  cudaTextureDesc td{};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  for (long long range : {1000000LL, 2500000LL, 10000000LL}) {
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
    if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    // warp roles {ldg, tma, tex}; the rounds are split in proportion to an
    // assumed per-warp rate so that all roles finish together if additive.
    const int cfgs[][3] = {{8, 0, 0}, {0, 8, 0}, {0, 0, 8}, {6, 2, 0}, {5, 3, 0}, {4, 4, 0},
                           {6, 0, 2}, {4, 0, 4}, {5, 2, 1}, {4, 2, 2}};
    // trial rate weights per warp (relative): LDG 1.0, TMA 0.55, TEX x (try 1.0)
    for (auto& c : cfgs) {
      for (double tex_w : {1.0, 0.5}) {
        if (c[2] == 0 && tex_w != 1.0) continue;
        const double wl = c[0] * 1.0, wt = c[1] * 0.55, wx = c[2] * tex_w, tot = wl + wt + wx;
        Roles ro{c[0], c[1], c[2], 0, 0, 0};
        ro.n_tma = c[1] ? (long long)(rounds * wt / tot) : 0;
        ro.n_tex = c[2] ? (long long)(rounds * wx / tot) : 0;
        ro.n_ldg = rounds - ro.n_tma - ro.n_tex;
        if (!c[0]) { ro.n_ldg = 0; if (c[1]) ro.n_tma = rounds - ro.n_tex; else ro.n_tex = rounds; }
        for (int occ : {2, 4}) {
          float best = 1e9, ms;
          for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            k_mix<<<sms * occ, WARPS * 32, dyn_bytes>>>(tmap, tex, idx, src, ro, sink);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
          }
          CK(cudaGetLastError());
          printf("range %8lld roles ldg=%d tma=%d tex=%d (tex_w %.1f) blocks/SM=%d: %.3f ms -> %.1f G/s\n", range, c[0],
                 c[1], c[2], tex_w, occ, best, n / (best * 1e-3) / 1e9);
        }
      }
    }
  }
  return 0;
}
