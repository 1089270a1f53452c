// pmp_solver.cu -- the C-ABI of libnumpmp_cuda.so (include/numpmp_gpu.h):
// device problem, CSR build, state upload/materialisation and the
// graph-batched, device-controlled PMP iteration loop.
//
// Reference boundary replaced: numpmp::PmpSolver (solver.hpp:265-519).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a profiler attached

#include "numpmp_gpu.h"
#include "numpmp_host.h"
#include "pmp_aux.cuh"
#include "pmp_kernels.cuh"
#include "pmp_p2p.cuh"

using namespace numpmp_dev;

namespace {

constexpr int kBatchIters = 32;  // iterations per CUDA-graph launch (even)
constexpr int kIdxPad = 64;      // int32 padding after index arrays (int4 over-read)

struct GpuError {
  int code;
  std::string msg;
};

#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw GpuError{NUMPMP_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
// NCCL is resolved lazily with dlopen, only for sharded (multi-GPU)
// handles: the single-GPU path never loads it, and a process that already
// loaded an NCCL (e.g. PyTorch's bundled one, for torch.distributed) shares
// that copy instead of pulling in a second, older libnccl.so.2.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(lib, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(lib, "ncclAllReduce"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(lib, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(lib, "ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.CommDestroy || !a.GetErrorString)
      a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  if (!api.error.empty()) throw GpuError{NUMPMP_NCCL_ERROR, api.error};
  return api;
}

#define NK(call)                                                                           \
  do {                                                                                     \
    const NcclApi& api_ = nccl();                                                          \
    ncclResult_t r_ = (api_.call);                                                         \
    if (r_ != ncclSuccess)                                                                 \
      throw GpuError{NUMPMP_NCCL_ERROR, std::string(#call) + ": " + api_.GetErrorString(r_)}; \
  } while (0)

thread_local std::string g_create_err;

// Pinned host slots for the control-block reads (2 Ctrl per handle), from a
// process-wide free list: cudaMallocHost / cudaFreeHost per handle cost
// milliseconds and synchronize the device.
struct PinnedCtrlPool {
  std::mutex mu;
  std::vector<void*> free_slots;
  void* get(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    if (!free_slots.empty()) {
      void* p = free_slots.back();
      free_slots.pop_back();
      return p;
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
  }
  void put(void* p) {
    std::lock_guard<std::mutex> lk(mu);
    free_slots.push_back(p);
  }
};
PinnedCtrlPool& ctrl_pool() {
  static PinnedCtrlPool* pool = new PinnedCtrlPool();  // never destroyed: slots outlive handles
  return *pool;
}

// Device memory comes from a stream-ordered pool private to this library
// (one per device, created on first use) that keeps freed memory reserved:
// creating and destroying solver handles (e2e steps, warm re-solves) then
// costs no cudaMalloc/cudaFree round trips, and the device's default pool --
// which other CUDA code in the host process may use -- is left untouched.
cudaMemPool_t lib_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  static const char* mode = std::getenv("NUMPMP_POOL");  // A/B: "default" = the device's default pool
  if (mode && std::strcmp(mode, "default") == 0) return nullptr;
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    if (!(mode && std::strcmp(mode, "reuse") == 0)) {
      // No cross-stream reuse with inserted dependencies: handles of
      // in-process peer-memory ranks share this pool, and a dependency of one
      // rank's stream on another's (which may hold a barrier wait) deadlocks.
      int off = 0;
      cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowInternalDependencies, &off);
      cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowOpportunistic, &off);
    }
    pools[device] = p;
  }
  return pools[device];
}

// cudaMallocAsync from the library pool of the stream's current device.
cudaError_t lib_malloc_async(void** p, size_t bytes, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = lib_pool(dev);
  if (!pool) return cudaMallocAsync(p, bytes, stream);
  return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

// The device-wide persisting-L2 limit is raised for the handles' lifetime
// and restored to the caller's value when the last handle on the device is
// destroyed.
struct L2LimitGuard {
  std::mutex mu;
  int users[64] = {};
  size_t saved[64] = {};
  void acquire(int device, size_t want) {
    if (device < 0 || device >= 64 || want == 0) return;
    std::lock_guard<std::mutex> lk(mu);
    size_t cur = 0;
    if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) != cudaSuccess) return;
    if (users[device]++ == 0) saved[device] = cur;
    int dev_max = 0;
    cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxPersistingL2CacheSize, device);
    const size_t set = std::min<size_t>(want, static_cast<size_t>(dev_max));
    if (cur != set) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set);
  }
  void release(int device) {
    if (device < 0 || device >= 64) return;
    std::lock_guard<std::mutex> lk(mu);
    if (users[device] == 0 || --users[device] > 0) return;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, saved[device]);
  }
};
L2LimitGuard& l2_guard() {
  static L2LimitGuard* g = new L2LimitGuard();
  return *g;
}

template <class T>
T* dalloc(size_t count, int64_t* bytes, cudaStream_t stream) {
  T* p = nullptr;
  const size_t b = sizeof(T) * (count > 0 ? count : 1);
  CK(lib_malloc_async(reinterpret_cast<void**>(&p), b, stream));
  *bytes += static_cast<int64_t>(b);
  return p;
}

int grid_for(long long work, int threads = 256) {
  long long b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<int>(b);
}

// One NVTX range per C-ABI call (profiler ranges for
// ncu / nsys timelines), named after the entry point.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// NUMPMP_TIMING=1: host wall time of the setup / run / teardown phases on
// stderr (end-to-end accounting of the C-ABI calls).
struct PhaseTimer {
  bool on = std::getenv("NUMPMP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[numpmp] %-28s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// One column block of the device problem (see pmp_kernels.cuh).
struct ColBlock {
  int64_t s0 = 0, s1 = 0, nnz = 0, nv = 0;
  int* row_ptr = nullptr;     // m+1
  int* col_idx = nullptr;     // nnz + pad, global stream ids
  int* vptr = nullptr;        // nv+1: first CSR entry of each segment
  int* vrow = nullptr;        // nv: link of each segment
  int2* units = nullptr;      // nu: segment range of each warp unit (whole rows)
  int4* pieces = nullptr;     // npieces: split-row pieces (BlockArgs::pieces)
  unsigned* uctr = nullptr;   // per split-row slot: pieces done (at the row's first slot)
  double* upart = nullptr;    // per slot: a piece's partial load
  int64_t nu = 0, npieces = 0;
  int seg = 0;                // max entries per segment
  int row_mode = 0;           // k_link_pass in row mode (longest row short, see BlockArgs)
  int pair_tiles = 0;         // k_stream_pass on pair tiles (short routes, see BlockArgs)
};

}  // namespace

struct numpmp_gpu {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // side stream of the pipelined graph (stream passes)
  cudaEvent_t pipe_ev[2 * kMaxBlocks + 2] = {};
  bool split_epilogue = true;      // NUMPMP_SPLIT_EPILOGUE=0: epilogue fused into the last link pass
  bool pipeline = true;            // NUMPMP_PIPELINE=0: serial graph (K1(b+1) no longer overlaps K2(b))
  std::string err;
  numpmp_config cfg{};
  int64_t m = 0, n = 0, nnz = 0;
  int64_t n_total = 0, nnz_total = 0, stream_begin = 0;  // global sizes (sharded)
  bool sharded = false;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  // peer-memory exchange (pmp_p2p.cuh); xregion = [v | slots | xs | flags],
  // cudaMalloc'd so that it can be exported with CUDA IPC
  bool p2p = false;
  bool p2p_fused = false;  // one GPU per rank: wait + finalize inside the owner epilogue
  bool p2p_cta_sysfence = std::getenv("NUMPMP_P2P_SYSFENCE") != nullptr;  // A/B: per-CTA system fences
  void* xregion = nullptr;
  size_t xregion_bytes = 0;
  int64_t mo = 0, l0 = 0, l1 = 0;
  std::vector<void*> peer_bases;     // opened IPC mappings (closed at destroy)
  void** peer_tables = nullptr;      // device: 4 tables of world pointers
  unsigned long long* done_cnt = nullptr;
  double* ep_part = nullptr;
  int64_t dev_bytes = 0;
  bool l2_guard_held = false;  // holds a reference on the device's persisting-L2 limit
  // get_state fingerprint: set_state of exactly the state the handle last
  // issued (nothing ran since) keeps the device state instead of
  // re-decomposing z on the host
  uint64_t issued_fp = 0;
  bool issued_valid = false;

  // problem
  int* col_ptr = nullptr;
  int* row_idx = nullptr;
  double* w = nullptr;
  unsigned char* kind = nullptr;
  int* deg = nullptr;  // link degrees (global)
  double* cap = nullptr;
  std::vector<ColBlock> blocks;

  // state (ping-pong between iterations)
  double* A[2] = {nullptr, nullptr};
  double* B[2] = {nullptr, nullptr};
  double* zs[2] = {nullptr, nullptr};
  double* pr[2] = {nullptr, nullptr};
  double* Q[2] = {nullptr, nullptr};
  double* x = nullptr;
  double* v = nullptr;
  double* v_alt[2] = {nullptr, nullptr};  // v for rho*gamma, rho/gamma (rho-update iterations)
  double* ps0 = nullptr;    // slack flows of an uploaded state
  double* pbar0 = nullptr;  // link averages of an uploaded state
  double* Lbuf = nullptr;   // m + 3 (sharded: loads, stream-pass scalars, time-limit flag)
  double* Lacc = nullptr;   // m: link loads accumulated over the column blocks
  double* k1_part = nullptr;
  double* k2_part = nullptr;
  double* scratch_m = nullptr;
  double* scratch_m2 = nullptr;
  double* scratch_n = nullptr;
  double* scalars = nullptr;  // 2
  Ctrl* ctrl = nullptr;
  Ctrl* ctrl_host = nullptr;  // pinned, 2 slots
  numpmp_trace_row* trace_dev = nullptr;
  int64_t trace_cap = 0;

  int cur = 0;  // index of the current iterate buffers
  int grid1 = 0, grid2 = 0, grid3 = 0;
  int grid2r = 0;  // link pass in row mode (its own occupancy)
  int64_t iters_since_upload = 0;
  bool host_p_valid = false;  // set_state keeps p / p_bar verbatim for get_state
  std::vector<double> host_p, host_pbar;
  int64_t run_iters = 0;
  int last_status = NUMPMP_MAXITERS;

  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  cudaGraphExec_t prof_graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [parity][set]
  cudaEvent_t ev_batch[2] = {nullptr, nullptr};
  bool profiling = false;
  std::vector<cudaEvent_t> prof_ev;  // 2 sets of 1 + kBatchIters * launches_per_iteration
  int64_t prof_launches = 0, prof_iters = 0;
  double prof_ms_k1 = 0.0, prof_ms_k2 = 0.0;

  int64_t h2d = 0, d2h = 0;
  cudaEvent_t ev_run[2] = {nullptr, nullptr};
  double last_run_ms = 0.0;

  int nb() const { return static_cast<int>(blocks.size()); }
  // kernel launches of one iteration (the NCCL all-reduce is not ours)
  int launches_per_iteration() const {
    return p2p ? 2 * nb() + (p2p_fused ? 1 : 3) : 2 * nb() + ((sharded || split_epilogue) ? 1 : 0);
  }
  std::vector<int> launch_side;  // per launch of an iteration: 1 stream side, 2 link side
};

namespace {

int set_err(numpmp_gpu* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  g_create_err = msg;
  return code;
}

const char* validate_config(const numpmp_config* c) {
  // solver.hpp:32-44, same order and messages
  if (!(c->eps_abs > 0.0)) return "eps_abs must be > 0";
  if (!(c->rho0 > 0.0)) return "rho0 must be > 0";
  if (!(c->alpha >= 1.0 && c->alpha <= 2.0)) return "alpha must be in [1, 2]";
  if (!(c->mu > 1.0)) return "mu must be > 1";
  if (!(c->gamma > 1.0)) return "gamma must be > 1";
  if (c->rho_update_interval < 1) return "rho_update_interval must be >= 1";
  if (c->max_iters < 1) return "max_iters must be >= 1";
  if (c->trace_every < 1) return "trace_every must be >= 1";
  if (c->threads < 0) return "threads must be >= 0";
  if (c->time_limit < 0.0) return "time_limit must be >= 0";
  return nullptr;
}

// Exchange region layout: [v: m][v_alt: 2m][slots: world*mo][xs: world*8]
// doubles, then [flags: 4] u64.
size_t xr_slots_off(const numpmp_gpu* h) { return 24 * static_cast<size_t>(h->m); }
size_t xr_xs_off(const numpmp_gpu* h) {
  return xr_slots_off(h) + 8 * static_cast<size_t>(h->world) * static_cast<size_t>(h->mo);
}
size_t xr_flags_off(const numpmp_gpu* h) { return xr_xs_off(h) + 64 * static_cast<size_t>(h->world); }

P2PArgs p2p_args(const numpmp_gpu* h) {
  P2PArgs p{};
  p.rank = h->rank;
  p.world = h->world;
  p.mo = h->mo;
  p.l0 = h->l0;
  p.l1 = h->l1;
  const size_t W = static_cast<size_t>(h->world);
  p.slots_peer = reinterpret_cast<double* const*>(h->peer_tables);
  p.v_peer = reinterpret_cast<double* const*>(h->peer_tables + W);
  p.xs_peer = reinterpret_cast<double* const*>(h->peer_tables + 2 * W);
  p.flags_peer = reinterpret_cast<unsigned long long* const*>(h->peer_tables + 3 * W);
  p.flags = reinterpret_cast<unsigned long long*>(static_cast<char*>(h->xregion) + xr_flags_off(h));
  p.done_cnt = h->done_cnt;
  p.ep_part = h->ep_part;
  p.cta_sysfence = h->p2p_cta_sysfence ? 1 : 0;
  return p;
}

IterArgs make_args(numpmp_gpu* h, int parity, int mode) {
  IterArgs a{};
  a.col_ptr = h->col_ptr;
  a.row_idx = h->row_idx;
  a.w = h->w;
  a.kind = h->kind;
  a.deg = h->deg;
  a.cap = h->cap;
  a.n = h->n;
  a.m = h->m;
  a.alpha = h->cfg.alpha;
  // check_termination (solver.hpp:157-163): eps_abs * sqrt(J), J global.
  a.eps_tol = h->cfg.eps_abs * std::sqrt(static_cast<double>(h->nnz_total + h->m));
  a.mu = h->cfg.mu;
  a.gamma = h->cfg.gamma;
  a.rho_interval = h->cfg.rho_update_interval;
  a.trace_every = h->cfg.trace_every;
  a.max_iters = h->cfg.max_iters;
  a.time_limit_ns = static_cast<long long>(h->cfg.time_limit * 1e9);
  a.mode = mode;
  const int i = parity, o = parity ^ 1;
  a.A_in = h->A[i];
  a.A_out = h->A[o];
  a.x = h->x;
  a.B_in = h->B[i];
  a.B_out = h->B[o];
  a.zs_in = h->zs[i];
  a.zs_out = h->zs[o];
  a.pr_in = h->pr[i];
  a.pr_out = h->pr[o];
  a.Q_in = h->Q[i];
  a.Q_out = h->Q[o];
  a.v = h->v;
  a.v_alt[0] = h->v_alt[0];
  a.v_alt[1] = h->v_alt[1];
  a.k1_part = h->k1_part;
  a.k2_part = h->k2_part;
  a.grid1 = h->grid1;
  a.grid2 = h->grid2;
  a.grid3 = h->grid3;
  a.nblocks = h->nb();
  a.Lacc = h->Lacc;
  a.Lbuf = h->Lbuf;
  a.ctrl = h->ctrl;
  a.trace = h->trace_dev;
  a.trace_cap = h->trace_cap;
  if (h->p2p) a.p2p = p2p_args(h);
  return a;
}

BlockArgs block_args(const numpmp_gpu* h, int b) {
  const ColBlock& cb = h->blocks[static_cast<size_t>(b)];
  BlockArgs k{};
  k.s0 = cb.s0;
  k.s1 = cb.s1;
  k.col_idx = cb.col_idx;
  k.vptr = cb.vptr;
  k.vrow = cb.vrow;
  k.units = cb.units;
  k.nv = cb.nv;
  k.nu = cb.nu;
  k.index = b;
  k.first = b == 0;
  k.row_mode = cb.row_mode;
  k.pair_tiles = cb.pair_tiles;
  k.row_ptr = cb.row_ptr;
  k.m = h->m;
  k.pieces = cb.pieces;
  k.npieces = cb.npieces;
  k.uctr = cb.uctr;
  k.upart = cb.upart;
  return k;
}

// The link pass of one column block in its form: row mode, warp units, or
// warp units + split-row pieces (k_link_pass kForm 0 / 1 / 2).
template <int kPhase>
void launch_link_pass(const numpmp_gpu* h, const IterArgs& a, const BlockArgs& bk, const double* src, double* out) {
  if (bk.row_mode)
    k_link_pass<kPhase, 0><<<h->grid2r, kThreads, 0, h->stream>>>(a, bk, src, out);
  else if (bk.npieces == 0)
    k_link_pass<kPhase, 1><<<h->grid2, kThreads, 0, h->stream>>>(a, bk, src, out);
  else
    k_link_pass<kPhase, 2><<<h->grid2, kThreads, 0, h->stream>>>(a, bk, src, out);
}


// One PMP iteration on the stream: for each column block b the stream pass
// K1(b) and the link-pass gather K2(b); the last block's link pass is fused
// with the link epilogue and the device-side finalize (single GPU), or
// followed by the NCCL all-reduce of the partial loads and the replicated
// epilogue (sharded).  ev (nullable): events[0..launches] recorded around
// every launch; ev[0] is skipped when record_first is false.
// One PMP iteration: for each column block b the stream pass K1(b) and the
// link pass K2(b), then the tail: the streaming link epilogue + finalize
// (one device), the NCCL all-reduce + replicated epilogue, or the
// peer-memory wait / owner epilogue / finalize (pmp_p2p.cuh).
// pipelined: the stream passes run on a side stream, so K1(b+1) fills
// K2(b)'s tail; K1(b+2) waits for K2(b) (at most two x blocks live in L2).
// Launch order, work split and summation order are those of the serial
// form, so results are bit-identical.  ev (serial form only, nullable):
// events[0..launches] around every launch; ev[0] skipped unless record_first.
void enqueue_iteration(numpmp_gpu* h, int parity, int mode, cudaEvent_t* ev, bool record_first,
                       bool pipelined = false) {
  IterArgs a = make_args(h, parity, mode);
  int e = 0;
  std::vector<int> side;
  auto mark = [&](int s) {  // after every launch: event + stream/link side for profiling
    CK(cudaGetLastError());
    if (ev) CK(cudaEventRecordWithFlags(ev[e], h->stream, cudaEventRecordExternal));
    ++e;
    side.push_back(s);
  };
  if (record_first && ev) CK(cudaEventRecordWithFlags(ev[0], h->stream, cudaEventRecordExternal));
  ++e;
  const int nb = h->nb();
  cudaEvent_t* ev_k1 = h->pipe_ev;               // [nb]: K1(b) done
  cudaEvent_t* ev_k2 = h->pipe_ev + kMaxBlocks;  // [nb]: K2(b) done
  if (pipelined) {
    CK(cudaEventRecord(h->pipe_ev[2 * kMaxBlocks], h->stream));
    CK(cudaStreamWaitEvent(h->stream2, h->pipe_ev[2 * kMaxBlocks], 0));
  }
  const bool acc_last = h->split_epilogue && !h->sharded;
  for (int b = 0; b < nb; ++b) {
    const BlockArgs bk = block_args(h, b);
    cudaStream_t s1 = pipelined ? h->stream2 : h->stream;
    if (pipelined && b >= 2) CK(cudaStreamWaitEvent(h->stream2, ev_k2[b - 2], 0));
    if (bk.pair_tiles == 4)
      k_stream_pass<4><<<h->grid1, kThreads, 0, s1>>>(a, bk);
    else if (bk.pair_tiles == 2)
      k_stream_pass<2><<<h->grid1, kThreads, 0, s1>>>(a, bk);
    else
      k_stream_pass<1><<<h->grid1, kThreads, 0, s1>>>(a, bk);
    mark(1);
    if (pipelined) {
      CK(cudaEventRecord(ev_k1[b], h->stream2));
      CK(cudaStreamWaitEvent(h->stream, ev_k1[b], 0));
    }
    if (b + 1 < nb || acc_last)
      launch_link_pass<LP_ACC>(h, a, bk, h->x, nullptr);
    else if (h->p2p)
      launch_link_pass<LP_P2P>(h, a, bk, h->x, nullptr);
    else if (!h->sharded)
      launch_link_pass<LP_FUSED>(h, a, bk, h->x, nullptr);
    else
      launch_link_pass<LP_GATHER>(h, a, bk, h->x, nullptr);
    mark(2);
    if (pipelined) CK(cudaEventRecord(ev_k2[b], h->stream));
  }
  if (h->p2p && h->p2p_fused) {
    k_p2p_epilogue<true><<<h->grid3, kThreads, 0, h->stream>>>(a);
    mark(2);
  } else if (h->p2p) {
    k_p2p_wait<0><<<1, 32, 0, h->stream>>>(a);
    mark(2);
    k_p2p_epilogue<false><<<h->grid3, kThreads, 0, h->stream>>>(a);
    mark(2);
    k_p2p_finalize<<<1, 32, 0, h->stream>>>(a);
    mark(2);
  } else if (h->sharded) {
    NK(AllReduce(h->Lbuf, h->Lbuf, static_cast<size_t>(h->m + 3), ncclDouble, ncclSum, h->comm,
                 h->stream));
    k_link_epilogue<0><<<h->grid3, kThreads, 0, h->stream>>>(a);
    mark(2);
  } else if (acc_last) {
    k_link_epilogue<1><<<h->grid3, kThreads, 0, h->stream>>>(a);
    mark(2);
  }
  h->launch_side = side;
}

cudaGraphExec_t build_graph(numpmp_gpu* h, int parity, int ev_set) {
  cudaGraph_t g = nullptr;
  const int lpi = h->launches_per_iteration();
  const size_t set_base = ev_set < 0 ? 0 : static_cast<size_t>(ev_set) * (kBatchIters * lpi + 1);
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  try {
    for (int i = 0; i < kBatchIters; ++i) {
      enqueue_iteration(h, parity ^ (i & 1), MODE_RUN,
                        ev_set >= 0 ? &h->prof_ev[set_base + static_cast<size_t>(i * lpi)] : nullptr,
                        i == 0, h->pipeline && ev_set < 0);
    }
  } catch (...) {
    cudaStreamEndCapture(h->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CK(cudaStreamEndCapture(h->stream, &g));
  cudaGraphExec_t exec = nullptr;
  CK(cudaGraphInstantiate(&exec, g, 0));
  CK(cudaGraphDestroy(g));
  return exec;
}

void upload(numpmp_gpu* h, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
  h->h2d += static_cast<int64_t>(bytes);
}
void download(numpmp_gpu* h, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
  h->d2h += static_cast<int64_t>(bytes);
}

Ctrl read_ctrl(numpmp_gpu* h) {
  CK(cudaMemcpyAsync(h->ctrl_host, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return h->ctrl_host[0];
}

// ------------------------------------------ peer-memory collectives (aux)
// Outside the iteration loop (pmp_p2p.cuh): every call is collective over
// the ranks, which run the same sequence.  They use v as the result buffer,
// so v is rebuilt afterwards (p2p_mark_v_stale).
void p2p_barrier(numpmp_gpu* h, int which) {
  const P2PArgs p = p2p_args(h);
  k_p2p_aux_signal<<<1, 32, 0, h->stream>>>(p, which);
  CK(cudaGetLastError());
  k_p2p_aux_wait<<<1, 32, 0, h->stream>>>(p, which);
  CK(cudaGetLastError());
}
// v was used as a result buffer: rebuild it from B and price (current on
// every rank outside the loop: after set_cold / set_warm, or after
// p2p_sync_link_state) with the next iteration's rho.
void p2p_mark_v_stale(numpmp_gpu* h) {
  k_set_v<<<grid_for(h->m), 256, 0, h->stream>>>(make_args(h, h->cur, MODE_AUX));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
}
// dst[0:m) = sum over ranks of src[0:m) (rank order); src may alias dst.
void p2p_allreduce(numpmp_gpu* h, const double* src, double* dst) {
  const P2PArgs p = p2p_args(h);
  k_p2p_push_partials<<<grid_for(h->m), 256, 0, h->stream>>>(p, src, h->m);
  CK(cudaGetLastError());
  p2p_barrier(h, 0);
  k_p2p_reduce_bcast<<<grid_for(std::max<int64_t>(1, h->l1 - h->l0)), 256, 0, h->stream>>>(p);
  CK(cudaGetLastError());
  p2p_barrier(h, 1);
  CK(cudaMemcpyAsync(dst, h->v, 8 * static_cast<size_t>(h->m), cudaMemcpyDeviceToDevice, h->stream));
  p2p_barrier(h, 3);
  p2p_mark_v_stale(h);
}
// vec[0:m): every rank receives the owners' values of their links.
void p2p_allgather_owned(numpmp_gpu* h, double* vec) {
  const P2PArgs p = p2p_args(h);
  k_p2p_push_owned<<<grid_for(std::max<int64_t>(1, h->l1 - h->l0)), 256, 0, h->stream>>>(p, vec);
  CK(cudaGetLastError());
  p2p_barrier(h, 0);
  CK(cudaMemcpyAsync(vec, static_cast<char*>(h->xregion) + xr_slots_off(h), 8 * static_cast<size_t>(h->m),
                     cudaMemcpyDeviceToDevice, h->stream));
  p2p_barrier(h, 3);
}
// d[0:k) (device, k <= 8) = sum over ranks, rank order.
void p2p_allreduce_scalars(numpmp_gpu* h, double* d, int k) {
  const P2PArgs p = p2p_args(h);
  k_p2p_push_scalars<<<1, 32, 0, h->stream>>>(p, d, k);
  CK(cudaGetLastError());
  p2p_barrier(h, 1);
  k_p2p_sum_scalars<<<1, 32, 0, h->stream>>>(p, d, k);
  CK(cudaGetLastError());
  p2p_barrier(h, 3);
}
// After a run / step the link state (B, zs, price, Q, both iterates) is
// current only on the owners: gather it on every rank.
void p2p_sync_link_state(numpmp_gpu* h) {
  for (int i = 0; i < 2; ++i)
    for (double* vec : {h->B[i], h->zs[i], h->pr[i], h->Q[i]}) p2p_allgather_owned(h, vec);
  p2p_mark_v_stale(h);
}

// Per-link sums of src over this device's columns, block by block in the
// same order as the link pass (+ the sum over ranks when sharded).
void global_row_sums(numpmp_gpu* h, const double* src, double* out) {
  IterArgs a = make_args(h, h->cur, MODE_AUX);
  for (int b = 0; b < h->nb(); ++b) {
    if (b + 1 < h->nb())
      launch_link_pass<LP_ACC>(h, a, block_args(h, b), src, nullptr);
    else
      launch_link_pass<LP_ROWSUM>(h, a, block_args(h, b), src, out);
    CK(cudaGetLastError());
  }
  if (h->p2p)
    p2p_allreduce(h, out, out);
  else if (h->sharded)
    NK(AllReduce(out, out, static_cast<size_t>(h->m), ncclDouble, ncclSum, h->comm, h->stream));
}

// Link-major CSR of the columns [s0, s1) on the device: a stable radix sort
// of their terminals by link (stable => ascending terminal, hence
// ascending stream, within a link, exactly the counting sort of
// model.hpp:193-199), then column index = the terminal's (global) stream.
// sorted_terms_out (nullable, host) receives the terminal ids in CSR order,
// i.e. the reference's link_terminals without the slack terminals.
void build_csr(numpmp_gpu* h, int64_t s0, int64_t s1, int* row_ptr_out, int* col_idx_out,
               int* sorted_terms_out) {
  std::vector<int> bounds(2);
  CK(cudaMemcpy(&bounds[0], h->col_ptr + s0, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&bounds[1], h->col_ptr + s1, 4, cudaMemcpyDeviceToHost));
  const long long t0 = bounds[0], nnz = bounds[1] - bounds[0], ns = s1 - s0;
  int64_t tmpb = 0;
  int* keys_out = dalloc<int>(static_cast<size_t>(nnz) + kIdxPad, &tmpb, h->stream);
  int* vals_in = dalloc<int>(static_cast<size_t>(nnz) + kIdxPad, &tmpb, h->stream);
  int* vals_out = dalloc<int>(static_cast<size_t>(nnz) + kIdxPad, &tmpb, h->stream);
  int* t2s = dalloc<int>(static_cast<size_t>(h->nnz) + kIdxPad, &tmpb, h->stream);
  void* temp = nullptr;
  auto release = [&]() {
    cudaFreeAsync(temp, h->stream);
    cudaFreeAsync(keys_out, h->stream);
    cudaFreeAsync(vals_in, h->stream);
    cudaFreeAsync(vals_out, h->stream);
    cudaFreeAsync(t2s, h->stream);
  };
  try {
    k_iota<<<grid_for(nnz), 256, 0, h->stream>>>(vals_in, nnz, t0);
    k_terminal_stream<<<grid_for(ns), 256, 0, h->stream>>>(h->col_ptr + s0, ns, s0, t2s);
    CK(cudaGetLastError());
    int end_bit = 1;
    while ((1ll << end_bit) < h->m) ++end_bit;
    size_t temp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, h->row_idx + t0, keys_out, vals_in,
                                       vals_out, static_cast<int>(nnz), 0, end_bit, h->stream));
    CK(lib_malloc_async(&temp, temp_bytes > 0 ? temp_bytes : 1, h->stream));
    CK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, h->row_idx + t0, keys_out, vals_in,
                                       vals_out, static_cast<int>(nnz), 0, end_bit, h->stream));
    k_row_ptr_from_sorted<<<grid_for(nnz + 1), 256, 0, h->stream>>>(keys_out, nnz, h->m,
                                                                      row_ptr_out);
    k_gather_i32<<<grid_for(nnz), 256, 0, h->stream>>>(t2s, vals_out, col_idx_out, nnz);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(col_idx_out + nnz, 0, sizeof(int) * kIdxPad, h->stream));
    if (sorted_terms_out)
      download(h, sorted_terms_out, vals_out, sizeof(int) * static_cast<size_t>(nnz));
    CK(cudaStreamSynchronize(h->stream));
  } catch (...) {
    release();
    throw;
  }
  release();
}

void check_view(const numpmp_problem_view* pv) {
  if (!pv || !pv->capacities || !pv->weights || !pv->kinds || !pv->stream_offsets ||
      (pv->nnz > 0 && !pv->route_links))
    throw GpuError{NUMPMP_INVALID_ARGUMENT, "problem view has null arrays"};
  if (pv->m < 1 || pv->n < 1) throw GpuError{NUMPMP_VALIDATION_ERROR, "invalid problem: empty"};
  if (pv->stream_offsets[0] != 0 || pv->stream_offsets[pv->n] != pv->nnz)
    throw GpuError{NUMPMP_VALIDATION_ERROR,
                   "invalid problem: [incidence-nnz: incidence nonzero count does not equal "
                   "sum of route lengths]"};
  if (pv->nnz >= (1LL << 31) - 2 * kIdxPad || pv->n >= (1LL << 31) - 1 ||
      pv->m >= (1LL << 31) - 1)
    throw GpuError{NUMPMP_INVALID_ARGUMENT, "problem exceeds the int32 index range of one device"};
}

// Column blocking: x of one block should stay L2-resident between its
// stream pass and its link-pass gather (126 MB L2, shared with the
// streamed index and state arrays).  NUMPMP_COL_BLOCKS overrides.
int choose_blocks(int64_t n, int64_t m, int64_t nnz) {
  if (const char* env = std::getenv("NUMPMP_COL_BLOCKS")) {
    const int v = std::atoi(env);
    if (v >= 1) return static_cast<int>(std::min<int64_t>(v, std::max<int64_t>(1, n / 32)));
  }
  const int64_t xbytes = 8 * n;
  // Every block after the first re-reads its CSR's row pointers and the
  // accumulated loads (4 + 2 x 8 bytes per link).  When that is as large as x
  // itself, keeping x L2-resident costs more than it saves: the paper shape P
  // (10M links, 5M streams) runs 0.745 ms/iteration in one block against
  // 0.798 in two (profiles/r2_col_blocks_sweep.txt).
  if (20 * m >= xbytes) return 1;
  const int64_t target = 24ll << 20;
  int64_t nb = (xbytes + target - 1) / target;
  // ... and no block below ~12.5M nonzeros: each block's two launches (their
  // tails, the per-block row pass) are a fixed cost, and short routes make
  // the blocks of the transit instance E light (51.7M nonzeros: 6 blocks by
  // x alone 0.373 ms/iteration, 4 blocks 0.361; C keeps 4)
  nb = std::min<int64_t>(nb, std::max<int64_t>(1, nnz / 12500000));
  nb = std::max<int64_t>(1, std::min<int64_t>(nb, 16));
  return static_cast<int>(std::min<int64_t>(nb, std::max<int64_t>(1, n / 32)));
}

// Warp-unit segmentation of one column block's CSR (k_link_pass): the
// segment bound is kSeg, raised so that the longest row fits one warp unit
// (32 segments); consecutive whole rows are then packed greedily into units
// of <= 32 segments (host pass over the per-row segment counts).
void segment_block(numpmp_gpu* h, ColBlock& cb) {
  const int64_t m = h->m;
  int64_t tmpb = 0;
  int* dmax = dalloc<int>(1, &tmpb, h->stream);
  CK(cudaMemsetAsync(dmax, 0, sizeof(int), h->stream));
  k_max_degree<<<grid_for(m), 256, 0, h->stream>>>(cb.row_ptr, m, dmax);
  CK(cudaGetLastError());
  int maxd = 0;
  CK(cudaMemcpyAsync(&maxd, dmax, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFreeAsync(dmax, h->stream);
  // Segments of <= kSeg entries; a row of more than 32 segments (a hot link)
  // is split over several warp units and combined in unit order.
  cb.seg = kSeg;
  // Row mode when the longest row is short: a lane per row costs no
  // segment metadata or scan.  NUMPMP_ROW_MODE_MAX, default 64 entries
  // (C: -1.8%, P: -8%; B with 100-entry rows stays in units,
  // profiles/r1_row_mode_sweep.txt).
  int row_mode_max = 64;
  if (const char* env = std::getenv("NUMPMP_ROW_MODE_MAX")) row_mode_max = std::atoi(env);
  cb.row_mode = maxd <= row_mode_max ? 1 : 0;
  int* nseg = dalloc<int>(static_cast<size_t>(m) + 1, &tmpb, h->stream);
  int* row_vstart = dalloc<int>(static_cast<size_t>(m) + 1, &tmpb, h->stream);
  CK(cudaMemsetAsync(nseg + m, 0, sizeof(int), h->stream));
  k_seg_count<<<grid_for(m), 256, 0, h->stream>>>(cb.row_ptr, m, cb.seg, nseg);
  CK(cudaGetLastError());
  size_t temp_bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, nseg, row_vstart, static_cast<int>(m + 1),
                                   h->stream));
  void* temp = nullptr;
  CK(lib_malloc_async(&temp, temp_bytes > 0 ? temp_bytes : 1, h->stream));
  CK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, nseg, row_vstart, static_cast<int>(m + 1),
                                   h->stream));
  std::vector<int> vstart(static_cast<size_t>(m) + 1);
  CK(cudaMemcpyAsync(vstart.data(), row_vstart, sizeof(int) * (static_cast<size_t>(m) + 1),
                     cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFreeAsync(temp, h->stream);
  cudaFreeAsync(nseg, h->stream);
  const int nv = vstart[static_cast<size_t>(m)];
  cb.nv = nv;
  // Greedy packing of whole rows into units of <= 32 segments.  Rows of
  // more than kSplitMin entries (> 32 segments) are left out of the units:
  // they become pieces of <= kPiece entries (BlockArgs::pieces), ordered by
  // their relative position in the row, then by row.  Row mode has no
  // units (a lane per row, any length).
  std::vector<int> rp;
  if (!cb.row_mode) {
    rp.resize(static_cast<size_t>(m) + 1);
    CK(cudaMemcpyAsync(rp.data(), cb.row_ptr, sizeof(int) * rp.size(), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  std::vector<int2> units;
  units.reserve(static_cast<size_t>(nv / 16 + 2));
  struct PieceKey {
    double pos;
    int4 pc;
  };
  std::vector<PieceKey> pieces;
  int nslots = 0;
  int ubeg = 0;
  auto close = [&](int end) {
    if (end > ubeg) units.push_back(make_int2(ubeg, end));
  };
  for (int64_t l = 0; l < m && !cb.row_mode; ++l) {
    const int rs = vstart[static_cast<size_t>(l)], re = vstart[static_cast<size_t>(l) + 1];
    const int b = rp[static_cast<size_t>(l)], d = rp[static_cast<size_t>(l) + 1] - b;
    if (d > kSplitMin) {
      close(rs);
      ubeg = re;  // the row's segments stay in vptr (contiguity) but in no unit
      const int np = (d + kPiece - 1) / kPiece;
      for (int k = 0; k < np; ++k)
        pieces.push_back(PieceKey{(k + 0.5) / np,
                                  make_int4(b + k * kPiece, b + std::min(d, (k + 1) * kPiece),
                                            static_cast<int>(l), nslots)});
      nslots += np;
      continue;
    }
    if (re - ubeg > 32) {
      close(rs);
      ubeg = rs;
    }
  }
  close(nv);
  cb.nu = static_cast<int64_t>(units.size());
  cb.npieces = static_cast<int64_t>(pieces.size());
  if (!pieces.empty()) {
    std::stable_sort(pieces.begin(), pieces.end(),
                     [](const PieceKey& x, const PieceKey& y) { return x.pos < y.pos; });
    std::vector<int4> pc(pieces.size());
    for (size_t i = 0; i < pieces.size(); ++i) pc[i] = pieces[i].pc;
    cb.pieces = dalloc<int4>(pc.size(), &h->dev_bytes, h->stream);
    cb.uctr = dalloc<unsigned>(static_cast<size_t>(nslots), &h->dev_bytes, h->stream);
    cb.upart = dalloc<double>(static_cast<size_t>(nslots), &h->dev_bytes, h->stream);
    CK(cudaMemcpyAsync(cb.pieces, pc.data(), sizeof(int4) * pc.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(cb.uctr, 0, sizeof(unsigned) * static_cast<size_t>(nslots), h->stream));
    CK(cudaStreamSynchronize(h->stream));  // pc is host memory
  }
  if (!units.empty()) {
    cb.units = dalloc<int2>(units.size(), &h->dev_bytes, h->stream);
    CK(cudaMemcpyAsync(cb.units, units.data(), sizeof(int2) * units.size(), cudaMemcpyHostToDevice,
                       h->stream));
  }
  cb.vptr = dalloc<int>(static_cast<size_t>(nv) + 1, &h->dev_bytes, h->stream);
  cb.vrow = dalloc<int>(static_cast<size_t>(nv), &h->dev_bytes, h->stream);
  k_seg_fill<<<grid_for(m), 256, 0, h->stream>>>(cb.row_ptr, row_vstart, m, cb.vptr, cb.vrow);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));  // `units` is host memory
  cudaFreeAsync(row_vstart, h->stream);
}

// CUDA loads kernels lazily (CUDA_MODULE_LOADING=LAZY, the CUDA 12
// default), and loading one may wait for the kernels already running on the
// device.  Peer-memory ranks in one process spin in barrier kernels while
// their peers launch kernels, so a first-use load deadlocks them (every
// wait traps after 60 s).  Every kernel of the library is therefore loaded
// up front, once per device, before any handle runs.
template <int kPhase>
void preload_link_pass(std::vector<const void*>& f) {
  f.push_back(reinterpret_cast<const void*>(&k_link_pass<kPhase, 0>));
  f.push_back(reinterpret_cast<const void*>(&k_link_pass<kPhase, 1>));
  f.push_back(reinterpret_cast<const void*>(&k_link_pass<kPhase, 2>));
}
void preload_kernels(int device) {
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  std::vector<const void*> f;
#define NUMPMP_K(k) f.push_back(reinterpret_cast<const void*>(&k))
  NUMPMP_K(k_stream_pass<1>); NUMPMP_K(k_stream_pass<2>); NUMPMP_K(k_stream_pass<4>);
  NUMPMP_K(k_link_epilogue<0>); NUMPMP_K(k_link_epilogue<1>);
  NUMPMP_K(k_refresh_v); NUMPMP_K(k_set_v); NUMPMP_K(k_residual_parts);
  NUMPMP_K(k_p2p_wait<0>); NUMPMP_K(k_p2p_epilogue<false>); NUMPMP_K(k_p2p_epilogue<true>); NUMPMP_K(k_p2p_finalize);
  NUMPMP_K(k_p2p_aux_wait); NUMPMP_K(k_p2p_aux_signal); NUMPMP_K(k_p2p_push_partials);
  NUMPMP_K(k_p2p_reduce_bcast); NUMPMP_K(k_p2p_push_owned); NUMPMP_K(k_p2p_push_scalars);
  NUMPMP_K(k_p2p_sum_scalars);
  NUMPMP_K(k_validate); NUMPMP_K(k_iota); NUMPMP_K(k_degree); NUMPMP_K(k_add_degree); NUMPMP_K(k_max_degree);
  NUMPMP_K(k_offsets_to_i32); NUMPMP_K(k_gather_i32); NUMPMP_K(k_terminal_stream); NUMPMP_K(k_row_ptr_from_sorted);
  NUMPMP_K(k_seg_count); NUMPMP_K(k_seg_fill); NUMPMP_K(k_row_sums_seq);
  NUMPMP_K(k_int_to_double); NUMPMP_K(k_double_to_int);
  NUMPMP_K(k_materialize_links); NUMPMP_K(k_expand_terminals); NUMPMP_K(k_post_streams); NUMPMP_K(k_post_links);
  NUMPMP_K(k_sum_parts); NUMPMP_K(k_start_clock); NUMPMP_K(k_warm_links); NUMPMP_K(k_path_prices);
  NUMPMP_K(k_degrade_links); NUMPMP_K(k_route_min_scale); NUMPMP_K(k_prune_prices); NUMPMP_K(k_recenter_log);
#undef NUMPMP_K
  preload_link_pass<LP_ACC>(f);
  preload_link_pass<LP_FUSED>(f);
  preload_link_pass<LP_GATHER>(f);
  preload_link_pass<LP_ROWSUM>(f);
  preload_link_pass<LP_P2P>(f);
  // NUMPMP_CARVEOUT=<percent>: shared-memory carveout preference for every
  // kernel (A/B of the L1 share the gathered vectors get; unset: driver default)
  const char* carve = std::getenv("NUMPMP_CARVEOUT");
  for (const void* fn : f) {
    cudaFuncAttributes attr;
    CK(cudaFuncGetAttributes(&attr, fn));
    if (carve) CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(carve)));
  }
  done[device] = true;
}

void create_common(numpmp_gpu* h, const numpmp_problem_view* pv) {
  PhaseTimer pt;
  CK(cudaSetDevice(h->device));
  preload_kernels(h->device);
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
  for (cudaEvent_t& e : h->pipe_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (const char* env = std::getenv("NUMPMP_SPLIT_EPILOGUE")) h->split_epilogue = std::atoi(env) != 0;
  if (const char* env = std::getenv("NUMPMP_PIPELINE")) h->pipeline = std::atoi(env) != 0;
  // L2 set-aside for the evict_last lines (x of the live column blocks, v):
  // 32 MB measured best at config C (profiles/r1_l2_sweep.txt);
  // NUMPMP_L2_PERSIST_MB overrides (0 = leave the device limit alone).
  // Restored when the last handle on the device is destroyed.
  {
    size_t want = size_t(32) << 20;
    if (const char* env = std::getenv("NUMPMP_L2_PERSIST_MB")) want = static_cast<size_t>(std::atoll(env)) << 20;
    if (want > 0) {
      l2_guard().acquire(h->device, want);
      h->l2_guard_held = true;
    }
  }
  pt.mark("create: stream");
  const int64_t m = h->m, n = h->n, nnz = h->nnz;
  int64_t* b = &h->dev_bytes;
  h->col_ptr = dalloc<int>(static_cast<size_t>(n) + 1, b, h->stream);
  h->row_idx = dalloc<int>(static_cast<size_t>(nnz) + kIdxPad, b, h->stream);
  h->w = dalloc<double>(static_cast<size_t>(n), b, h->stream);
  h->kind = dalloc<unsigned char>(static_cast<size_t>(n), b, h->stream);
  h->cap = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  h->deg = dalloc<int>(static_cast<size_t>(m), b, h->stream);
  for (int i = 0; i < 2; ++i) {
    h->A[i] = dalloc<double>(static_cast<size_t>(n), b, h->stream);
    h->B[i] = dalloc<double>(static_cast<size_t>(m), b, h->stream);
    h->zs[i] = dalloc<double>(static_cast<size_t>(m), b, h->stream);
    h->pr[i] = dalloc<double>(static_cast<size_t>(m), b, h->stream);
    h->Q[i] = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  }
  h->x = dalloc<double>(static_cast<size_t>(n), b, h->stream);
  h->v = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  for (int i = 0; i < 2; ++i) h->v_alt[i] = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  h->ps0 = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  h->pbar0 = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  h->Lbuf = dalloc<double>(static_cast<size_t>(m) + 3, b, h->stream);
  h->Lacc = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  h->scratch_m = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  h->scratch_m2 = dalloc<double>(static_cast<size_t>(m), b, h->stream);
  h->scratch_n = dalloc<double>(static_cast<size_t>(n), b, h->stream);
  h->scalars = dalloc<double>(2, b, h->stream);
  h->ctrl = dalloc<Ctrl>(1, b, h->stream);
  h->ctrl_host = static_cast<Ctrl*>(ctrl_pool().get(2 * sizeof(Ctrl)));
  if (!h->ctrl_host) throw GpuError{NUMPMP_CUDA_ERROR, "pinned host allocation failed"};
  CK(cudaMemsetAsync(h->row_idx + nnz, 0, sizeof(int) * kIdxPad, h->stream));
  CK(cudaMemsetAsync(h->ctrl, 0, sizeof(Ctrl), h->stream));

  // Upload.  Offsets travel as int64 and are narrowed on the device.
  long long* off64 = nullptr;
  CK(lib_malloc_async(reinterpret_cast<void**>(&off64), 8 * static_cast<size_t>(n + 1), h->stream));
  upload(h, off64, pv->stream_offsets, 8 * static_cast<size_t>(n + 1));
  k_offsets_to_i32<<<grid_for(n + 1), 256, 0, h->stream>>>(off64, h->col_ptr, n + 1);
  CK(cudaGetLastError());
  upload(h, h->row_idx, pv->route_links, 4 * static_cast<size_t>(nnz));
  upload(h, h->w, pv->weights, 8 * static_cast<size_t>(n));
  upload(h, h->kind, pv->kinds, static_cast<size_t>(n));
  upload(h, h->cap, pv->capacities, 8 * static_cast<size_t>(m));
  pt.mark("create: alloc + upload");

  // Model validation (model.hpp:76-155) on the device; only an invalid
  // problem pays for the host validator, which words the reference's exact
  // ValidationError message.  Extension streams: SolverError
  // (solver.hpp:275-284; no device prox).
  {
    unsigned long long* bad = nullptr;
    CK(lib_malloc_async(reinterpret_cast<void**>(&bad), 6 * sizeof(unsigned long long), h->stream));
    CK(cudaMemsetAsync(bad, 0, 6 * sizeof(unsigned long long), h->stream));
    k_validate<<<grid_for(std::max(n, m)), 256, 0, h->stream>>>(off64, h->row_idx, h->w, h->kind,
                                                               h->cap, n, m, bad);
    CK(cudaGetLastError());
    unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(cnt, bad, sizeof(cnt), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFreeAsync(bad, h->stream);
    cudaFreeAsync(off64, h->stream);
    if (cnt[0] + cnt[1] + cnt[2] + cnt[3] + cnt[4] > 0) {
      std::vector<char> msg(4096);
      numpmp_validate(pv->m, pv->n, pv->capacities, pv->weights, pv->kinds, pv->stream_offsets,
                      pv->route_links, msg.data(), static_cast<int64_t>(msg.size()));
      throw GpuError{NUMPMP_VALIDATION_ERROR, msg.data()};
    }
    if (cnt[5] > 0)
      throw GpuError{NUMPMP_SOLVER_ERROR,
                     "no extension registered for utility (extension utilities are host "
                     "callbacks and are not supported by the device engine)"};
  }
  pt.mark("create: device validation");

  // Column blocks (stream ranges rounded to 32-stream tiles) and their CSRs.
  const int nbk = choose_blocks(n, m, nnz);
  CK(cudaMemsetAsync(h->deg, 0, sizeof(int) * static_cast<size_t>(m), h->stream));
  for (int k = 0; k < nbk; ++k) {
    ColBlock cb;
    cb.s0 = (n * k / nbk) & ~31LL;
    cb.s1 = (k + 1 == nbk) ? n : ((n * (k + 1) / nbk) & ~31LL);
    const int64_t tb = pv->stream_offsets[cb.s0], te = pv->stream_offsets[cb.s1];
    cb.nnz = te - tb;
    cb.row_ptr = dalloc<int>(static_cast<size_t>(m) + 1, b, h->stream);
    cb.col_idx = dalloc<int>(static_cast<size_t>(cb.nnz) + kIdxPad, b, h->stream);
    h->blocks.push_back(cb);
    build_csr(h, cb.s0, cb.s1, cb.row_ptr, cb.col_idx, nullptr);
    // multi-route tiles for short routes: mean route length <= NUMPMP_PAIR_TILE_TAU
    // (default 6) -> NUMPMP_TILE_Q (default 2) streams per lane
    double pair_tau = 6.0;
    if (const char* env = std::getenv("NUMPMP_PAIR_TILE_TAU")) pair_tau = std::atof(env);
    int tile_q = 2;
    if (const char* env = std::getenv("NUMPMP_TILE_Q")) tile_q = std::atoi(env) >= 4 ? 4 : 2;
    h->blocks.back().pair_tiles =
        (cb.s1 > cb.s0 && static_cast<double>(cb.nnz) <= pair_tau * static_cast<double>(cb.s1 - cb.s0))
            ? tile_q : 1;
    k_add_degree<<<grid_for(m), 256, 0, h->stream>>>(cb.row_ptr, m, h->deg);
    CK(cudaGetLastError());
    segment_block(h, h->blocks.back());
  }
  CK(cudaStreamSynchronize(h->stream));
  pt.mark("create: device CSR build");

  // Persistent grids: resident blocks x SMs.
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  int occ1 = 0, occ2 = 0;
  {  // the stream pass of the blocks' tile form (multi-route tiles have their own launch bound)
    const int q0 = h->blocks.empty() ? 1 : h->blocks.front().pair_tiles;
    void (*k1)(IterArgs, BlockArgs) = q0 == 4 ? k_stream_pass<4> : q0 == 2 ? k_stream_pass<2> : k_stream_pass<1>;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k1, kThreads, 0));
  }
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_link_pass<LP_FUSED, 2>, kThreads, 0));
  int occ3 = 0, occ2r = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_link_epilogue<0>, kThreads, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2r, k_link_pass<LP_ACC, 0>, kThreads, 0));
  int64_t max_bs = 0, max_nu = 0;
  for (const ColBlock& cb : h->blocks) {
    max_bs = std::max(max_bs, cb.s1 - cb.s0);
    max_nu = std::max(max_nu, cb.row_mode ? (m + 31) / 32 : cb.nu + cb.npieces);
  }
  const long long tiles1 = (max_bs + 31) / 32, tiles2 = max_nu;
  // grids: NUMPMP_GRID_MULT x the resident CTAs (1 = persistent)
  long long gmult = 1;
  if (const char* env = std::getenv("NUMPMP_GRID_MULT")) gmult = std::max(1, std::atoi(env));
  h->grid1 = static_cast<int>(std::max(
      1LL, std::min<long long>((tiles1 + kWarps - 1) / kWarps, gmult * sms * std::max(occ1, 1))));
  h->grid2 = static_cast<int>(std::max(
      1LL, std::min<long long>((tiles2 + kWarps - 1) / kWarps, gmult * sms * std::max(occ2, 1))));
  long long emult = 1;  // NUMPMP_EPI_GRID_MULT: link-epilogue grid, x the resident CTAs (A/B)
  if (const char* env = std::getenv("NUMPMP_EPI_GRID_MULT")) emult = std::max(1, std::atoi(env));
  h->grid3 = static_cast<int>(std::max(
      1LL, std::min<long long>((m + kThreads - 1) / kThreads, emult * sms * std::max(occ3, 1))));
  h->grid2r = static_cast<int>(std::max(
      1LL, std::min<long long>(((m + 31) / 32 + kWarps - 1) / kWarps, gmult * sms * std::max(occ2r, 1))));
  h->k1_part = dalloc<double>(2 * static_cast<size_t>(nbk) * static_cast<size_t>(h->grid1) +
                                  2 * static_cast<size_t>(std::max(h->grid3, h->grid1)),
                              b, h->stream);
  h->k2_part = dalloc<double>(4 * static_cast<size_t>(std::max({h->grid2, h->grid2r, h->grid3})), b, h->stream);
  h->trace_cap = h->cfg.max_iters / h->cfg.trace_every + 2;
  h->trace_dev = dalloc<numpmp_trace_row>(static_cast<size_t>(h->trace_cap), b, h->stream);
  for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&h->ev_batch[i], cudaEventDisableTiming));
  CK(cudaStreamSynchronize(h->stream));
  pt.mark("create: grids + buffers");
}

void reset_ctrl(numpmp_gpu* h, double rho, int64_t iter) {
  h->issued_valid = false;
  Ctrl c{};
  c.rho = rho;
  c.rho_iter = rho;
  c.iter = iter;
  c.run_k = 0;
  c.status = ST_RUNNING;
  c.rho_changed = 1;  // k_refresh_v builds v from B and price
  std::memcpy(&h->ctrl_host[1], &c, sizeof(Ctrl));
  CK(cudaMemcpyAsync(h->ctrl, &h->ctrl_host[1], sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream));
  // v = B + price / rho of the new state, over all links (after set_cold /
  // set_warm / set_state, B and price are complete on every rank of a
  // sharded engine too)
  k_refresh_v<<<h->grid3, kThreads, 0, h->stream>>>(make_args(h, h->cur, MODE_AUX));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
}

// Cold state (solver.hpp:293-303): p = z = 0, price = 0, rho = rho0.
void do_set_cold(numpmp_gpu* h) {
  h->cur = 0;
  const size_t mb = 8 * static_cast<size_t>(h->m), nb = 8 * static_cast<size_t>(h->n);
  CK(cudaMemsetAsync(h->A[0], 0, nb, h->stream));
  CK(cudaMemsetAsync(h->x, 0, nb, h->stream));
  CK(cudaMemsetAsync(h->B[0], 0, mb, h->stream));
  CK(cudaMemsetAsync(h->zs[0], 0, mb, h->stream));
  CK(cudaMemsetAsync(h->Q[0], 0, mb, h->stream));
  CK(cudaMemsetAsync(h->pr[0], 0, mb, h->stream));
  CK(cudaMemsetAsync(h->ps0, 0, mb, h->stream));
  CK(cudaMemsetAsync(h->pbar0, 0, mb, h->stream));
  h->host_p_valid = false;
  h->iters_since_upload = 0;
  reset_ctrl(h, h->cfg.rho0, 0);
}

void set_warm_from_device(numpmp_gpu* h, double rho);

// warm_state (solver.hpp:305-314) + warm_start_from (218-259).
void do_set_warm(numpmp_gpu* h, const double* x0, const double* price, double rho) {
  if (!x0) throw GpuError{NUMPMP_INVALID_ARGUMENT, "warm start: x0 length does not match n"};
  std::vector<uint8_t> kinds(static_cast<size_t>(h->n));
  CK(cudaMemcpy(kinds.data(), h->kind, static_cast<size_t>(h->n), cudaMemcpyDeviceToHost));
  for (int64_t j = 0; j < h->n; ++j)
    if (kinds[static_cast<size_t>(j)] == NUMPMP_KIND_LOG && !(x0[j] > 0.0))
      throw GpuError{NUMPMP_DOMAIN_ERROR, "warm start: log stream " +
                                              std::to_string(j + h->stream_begin) +
                                              " needs a positive rate"};
  const size_t nb = 8 * static_cast<size_t>(h->n), mb = 8 * static_cast<size_t>(h->m);
  upload(h, h->x, x0, nb);
  if (price)
    upload(h, h->pr[0], price, mb);
  else
    CK(cudaMemsetAsync(h->pr[0], 0, mb, h->stream));
  set_warm_from_device(h, rho);
}

// warm_start_from (solver.hpp:218-259) with x0 already in h->x and the
// prices in h->pr[0] (device): A = x0, load = R x0, B / zs / Q / slack.
void set_warm_from_device(numpmp_gpu* h, double rho) {
  h->cur = 0;
  const size_t nb = 8 * static_cast<size_t>(h->n);
  CK(cudaMemcpyAsync(h->A[0], h->x, nb, cudaMemcpyDeviceToDevice, h->stream));
  global_row_sums(h, h->x, h->scratch_m);  // load = R x0
  k_warm_links<<<grid_for(h->m), 256, 0, h->stream>>>(h->scratch_m, h->deg, nullptr, h->cap,
                                                       h->m, h->B[0], h->zs[0], h->Q[0], h->ps0,
                                                       h->pbar0);
  CK(cudaGetLastError());
  h->host_p_valid = false;
  h->iters_since_upload = 0;
  reset_ctrl(h, rho > 0.0 ? rho : h->cfg.rho0, 0);
}

// Per-link sums of src over this device's columns in the reference's order
// (ascending stream id, one accumulator per link, model.hpp / warm.hpp
// loops): bit-exact with the host loops on one device.
void row_sums_sequential(numpmp_gpu* h, const double* src, double* out) {
  BlockCsrs bc{};
  bc.nblocks = h->nb();
  for (int b = 0; b < h->nb(); ++b) {
    bc.row_ptr[b] = h->blocks[static_cast<size_t>(b)].row_ptr;
    bc.col_idx[b] = h->blocks[static_cast<size_t>(b)].col_idx;
  }
  k_row_sums_seq<<<grid_for(h->m), 256, 0, h->stream>>>(bc, h->m, src, out);
  CK(cudaGetLastError());
  if (h->p2p)
    p2p_allreduce(h, out, out);
  else if (h->sharded)
    NK(AllReduce(out, out, static_cast<size_t>(h->m), ncclDouble, ncclSum, h->comm, h->stream));
}

// warm.hpp:25-57 warm_start_after_degrade on the device: the handle holds
// the degraded problem; cap_before, prior_x (this handle's streams) and
// prior_lambda_raw are the prior problem's capacities and solution.
void do_warm_after_degrade(numpmp_gpu* h, const double* cap_before, const double* prior_x,
                           const double* prior_lambda_raw, double prior_rho, double* x0_out,
                           double* price_out, double* rho_out) {
  if (!cap_before || !prior_x || !prior_lambda_raw)
    throw GpuError{NUMPMP_INVALID_ARGUMENT, "degrade warm start: null input"};
  const size_t nb = 8 * static_cast<size_t>(h->n), mb = 8 * static_cast<size_t>(h->m);
  double* ratio = h->scratch_m2;
  upload(h, ratio, cap_before, mb);                 // c_before -> ratio = c_after / c_before
  upload(h, h->pr[0], prior_lambda_raw, mb);
  upload(h, h->x, prior_x, nb);
  k_degrade_links<<<grid_for(h->m), 256, 0, h->stream>>>(h->cap, h->m, ratio, h->pr[0]);
  CK(cudaGetLastError());
  k_route_min_scale<<<grid_for(h->n), 256, 0, h->stream>>>(h->col_ptr, h->row_idx, h->n, ratio,
                                                           h->kind, h->x);
  CK(cudaGetLastError());
  // worst cut = min over links (exact in any order)
  size_t temp_bytes = 0;
  CK(cub::DeviceReduce::Min(nullptr, temp_bytes, ratio, h->scalars, static_cast<int>(h->m), h->stream));
  void* temp = nullptr;
  CK(lib_malloc_async(&temp, temp_bytes > 0 ? temp_bytes : 1, h->stream));
  CK(cub::DeviceReduce::Min(temp, temp_bytes, ratio, h->scalars, static_cast<int>(h->m), h->stream));
  double worst = 1.0;
  CK(cudaMemcpyAsync(&worst, h->scalars, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFreeAsync(temp, h->stream);
  worst = std::min(1.0, worst);  // warm.hpp:33-41 starts from worst_cut = 1.0
  const double rho = prior_rho / worst;
  if (x0_out) download(h, x0_out, h->x, nb);
  if (price_out) download(h, price_out, h->pr[0], mb);
  if (rho_out) *rho_out = rho;
  set_warm_from_device(h, rho);
}

// warm.hpp:62-94 warm_start_after_prune on the device.  x0 / price are the
// prior solution already projected onto the survivors (PruneMap::project_*,
// a host gather by the caller).
void do_warm_after_prune(numpmp_gpu* h, const double* x0_proj, const double* price_proj,
                         double prior_rho, double* x0_out, double* price_out, double* rho_out) {
  if (!x0_proj || !price_proj) throw GpuError{NUMPMP_INVALID_ARGUMENT, "prune warm start: null input"};
  const size_t nb = 8 * static_cast<size_t>(h->n), mb = 8 * static_cast<size_t>(h->m);
  upload(h, h->x, x0_proj, nb);
  upload(h, h->pr[0], price_proj, mb);
  row_sums_sequential(h, h->x, h->scratch_m);  // load, in the reference's order
  k_prune_prices<<<grid_for(h->m), 256, 0, h->stream>>>(h->scratch_m, h->cap, h->m, h->pr[0],
                                                        h->scratch_m2);
  CK(cudaGetLastError());
  k_path_prices<<<grid_for(h->n), 256, 0, h->stream>>>(h->col_ptr, h->row_idx, h->n, h->scratch_m2,
                                                       h->scratch_n);
  CK(cudaGetLastError());
  k_recenter_log<<<grid_for(h->n), 256, 0, h->stream>>>(h->scratch_n, h->w, h->kind, h->n, h->x);
  CK(cudaGetLastError());
  if (x0_out) download(h, x0_out, h->x, nb);
  if (price_out) download(h, price_out, h->pr[0], mb);
  if (rho_out) *rho_out = prior_rho;
  CK(cudaStreamSynchronize(h->stream));
  set_warm_from_device(h, prior_rho);
}

void p2p_wire(numpmp_gpu* h, const std::vector<void*>& bases) {
  const size_t W = static_cast<size_t>(h->world);
  std::vector<void*> t(4 * W);
  for (size_t q = 0; q < W; ++q) {
    char* b = static_cast<char*>(bases[q]);
    t[q] = b + xr_slots_off(h);
    t[W + q] = b;
    t[2 * W + q] = b + xr_xs_off(h);
    t[3 * W + q] = b + xr_flags_off(h);
  }
  CK(cudaMemcpyAsync(h->peer_tables, t.data(), sizeof(void*) * t.size(), cudaMemcpyHostToDevice,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->p2p = true;
  // One GPU per rank (no peer region on this device): the wait and the
  // finalize fold into the owner epilogue (pmp_p2p.cuh, fused mode).  Ranks
  // that share a GPU keep the separate one-CTA kernels, so a spinning CTA
  // never holds SMs another rank's link pass needs.
  bool distinct = true;
  for (size_t q = 0; q < W; ++q) {
    if (static_cast<int>(q) == h->rank) continue;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, bases[q]) != cudaSuccess) {
      cudaGetLastError();  // unknown placement: keep the form that is safe on a shared GPU
      distinct = false;
    } else if (at.device == h->device) {
      distinct = false;
    }
  }
  h->p2p_fused = distinct;
  // A/B: 0 off, 1 on where no rank shares this GPU; 2 on regardless (tests
  // with grids small enough that spinning CTAs cannot starve a peer's kernels)
  if (const char* env = std::getenv("NUMPMP_P2P_FUSED")) {
    const int f = std::atoi(env);
    h->p2p_fused = f == 2 || (f == 1 && distinct);
  }
  for (int i = 0; i < 2; ++i) {  // captured graphs hold the old launch list
    if (h->graph[i]) cudaGraphExecDestroy(h->graph[i]);
    h->graph[i] = nullptr;
    for (int set = 0; set < 2; ++set) {
      if (h->prof_graph[i][set]) cudaGraphExecDestroy(h->prof_graph[i][set]);
      h->prof_graph[i][set] = nullptr;
    }
  }
}
}  // namespace

// ------------------------------------------------------------------ C-ABI
extern "C" {

const char* numpmp_gpu_last_error(const numpmp_gpu* h) {
  return h ? h->err.c_str() : g_create_err.c_str();
}

int numpmp_gpu_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  try {
    NK(GetUniqueId(&id));
  } catch (const GpuError& e) {
    return set_err(nullptr, e.code, e.msg);
  }
  std::memcpy(out128, &id, sizeof(id));
  return NUMPMP_OK;
}

// exchange: 0 single device, 1 NCCL all-reduce, 2 peer memory (pmp_p2p.cuh)
static int create_impl(const numpmp_problem_view* pv, const numpmp_config* cfg, int device,
                       int rank, int world, const void* nccl_id, int64_t stream_begin,
                       int64_t n_total, numpmp_gpu** out, int exchange = -1) {
  if (!out) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "out is null");
  NvtxRange nvtx_range_("numpmp_gpu_create");
  *out = nullptr;
  if (!cfg) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "config is null");
  if (const char* msg = validate_config(cfg)) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, msg);
  numpmp_gpu* h = nullptr;
  PhaseTimer pt;
  try {
    check_view(pv);
    h = new numpmp_gpu();
    h->cfg = *cfg;
    h->device = device;
    h->m = pv->m;
    h->n = pv->n;
    h->nnz = pv->nnz;
    h->n_total = pv->n;
    h->nnz_total = pv->nnz;
    if (exchange < 0) exchange = (world >= 1 && nccl_id != nullptr) ? 1 : 0;
    if (exchange == 2) {
      if (world < 1 || world > kMaxRanks)
        throw GpuError{NUMPMP_INVALID_ARGUMENT, "peer-memory exchange supports 1..8 ranks"};
      h->sharded = true;
      h->rank = rank;
      h->world = world;
      h->stream_begin = stream_begin;
      h->n_total = n_total;
      CK(cudaSetDevice(device));
    } else if (exchange == 1) {
      // Sharded handle (also with world == 1: the same kernels and the
      // same all-reduce, over a one-rank communicator).
      h->sharded = true;
      h->rank = rank;
      h->world = world;
      h->stream_begin = stream_begin;
      h->n_total = n_total;
      CK(cudaSetDevice(device));
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      NK(CommInitRank(&h->comm, world, id, rank));
    }
    create_common(h, pv);
    if (exchange == 2) {
      // Exchange region (IPC-exportable, so plain cudaMalloc), v inside it.
      h->mo = (h->m + world - 1) / world;
      h->l0 = std::min<int64_t>(h->m, static_cast<int64_t>(rank) * h->mo);
      h->l1 = std::min<int64_t>(h->m, h->l0 + h->mo);
      h->xregion_bytes = xr_flags_off(h) + 4 * sizeof(unsigned long long);
      CK(cudaMalloc(&h->xregion, h->xregion_bytes));
      CK(cudaMemsetAsync(h->xregion, 0, h->xregion_bytes, h->stream));
      cudaFreeAsync(h->v, h->stream);
      cudaFreeAsync(h->v_alt[0], h->stream);
      cudaFreeAsync(h->v_alt[1], h->stream);
      h->v = static_cast<double*>(h->xregion);
      h->v_alt[0] = h->v + h->m;
      h->v_alt[1] = h->v + 2 * h->m;
      int64_t* b = &h->dev_bytes;
      h->done_cnt = dalloc<unsigned long long>(4, b, h->stream);
      CK(cudaMemsetAsync(h->done_cnt, 0, 4 * sizeof(unsigned long long), h->stream));
      h->ep_part = dalloc<double>(4 * static_cast<size_t>(h->grid3), b, h->stream);
      h->peer_tables = dalloc<void*>(4 * static_cast<size_t>(world), b, h->stream);
      CK(cudaStreamSynchronize(h->stream));
    } else if (h->sharded) {
      // Global link degrees and nnz: sums of the shards' local counts.
      NK(AllReduce(h->deg, h->deg, static_cast<size_t>(h->m), ncclInt32, ncclSum, h->comm,
                   h->stream));
      double nnz_local = static_cast<double>(h->nnz);
      CK(cudaMemcpyAsync(h->scalars, &nnz_local, 8, cudaMemcpyHostToDevice, h->stream));
      NK(AllReduce(h->scalars, h->scalars, 1, ncclDouble, ncclSum, h->comm, h->stream));
      double nnz_global = 0.0;
      CK(cudaMemcpyAsync(&nnz_global, h->scalars, 8, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      h->nnz_total = static_cast<int64_t>(nnz_global);
    }
    do_set_cold(h);
    pt.mark("create: total after validation");
    h->h2d = 0;
    h->d2h = 0;
    *out = h;
    return NUMPMP_OK;
  } catch (const GpuError& e) {
    int code = e.code;
    std::string msg = e.msg;
    if (h) numpmp_gpu_destroy(h);
    return set_err(nullptr, code, msg);
  } catch (const std::bad_alloc&) {
    if (h) numpmp_gpu_destroy(h);
    return set_err(nullptr, NUMPMP_CUDA_ERROR, "host allocation failed");
  }
}

int numpmp_gpu_create(const numpmp_problem_view* problem, const numpmp_config* config, int device,
                      numpmp_gpu** out) {
  return create_impl(problem, config, device, 0, 1, nullptr, 0, problem ? problem->n : 0, out);
}

int numpmp_gpu_create_sharded(const numpmp_problem_view* shard, const numpmp_config* config,
                              int device, int rank, int world, const void* nccl_id,
                              int64_t stream_begin, int64_t n_total, numpmp_gpu** out) {
  if (world < 1 || rank < 0 || rank >= world)
    return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "bad rank/world");
  if (!nccl_id) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "nccl_id is null");
  return create_impl(shard, config, device, rank, world, nccl_id, stream_begin, n_total, out);
}

#define GUARD(h, ...)                                                   \
  do {                                                                  \
    if (!(h)) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "null handle"); \
    NvtxRange nvtx_range_(__func__);                                    \
    try {                                                               \
      CK(cudaSetDevice((h)->device));                                   \
      __VA_ARGS__;                                                      \
      return NUMPMP_OK;                                                 \
    } catch (const GpuError& e) {                                       \
      return set_err((h), e.code, e.msg);                               \
    } catch (const std::bad_alloc&) {                                   \
      return set_err((h), NUMPMP_CUDA_ERROR, "host allocation failed"); \
    }                                                                   \
  } while (0)

int numpmp_gpu_create_p2p(const numpmp_problem_view* shard, const numpmp_config* config,
                          int device, int rank, int world, int64_t stream_begin, int64_t n_total,
                          numpmp_gpu** out) {
  if (world < 1 || rank < 0 || rank >= world)
    return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "bad rank/world");
  return create_impl(shard, config, device, rank, world, nullptr, stream_begin, n_total, out, 2);
}

int numpmp_gpu_p2p_export(numpmp_gpu* h, void* out64) {
  GUARD(h, {
    if (!h->xregion) throw GpuError{NUMPMP_INVALID_ARGUMENT, "not a peer-memory handle"};
    if (!out64) throw GpuError{NUMPMP_INVALID_ARGUMENT, "out is null"};
    cudaIpcMemHandle_t hd;
    CK(cudaIpcGetMemHandle(&hd, h->xregion));
    static_assert(sizeof(hd) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(out64, &hd, sizeof(hd));
  });
}


int numpmp_gpu_p2p_connect(numpmp_gpu* h, const void* handles) {
  GUARD(h, {
    if (!h->xregion || h->p2p)
      throw GpuError{NUMPMP_INVALID_ARGUMENT, "not an unconnected peer-memory handle"};
    if (!handles) throw GpuError{NUMPMP_INVALID_ARGUMENT, "handles is null"};
    CK(cudaSetDevice(h->device));
    std::vector<void*> bases(static_cast<size_t>(h->world));
    for (int q = 0; q < h->world; ++q) {
      if (q == h->rank) {
        bases[static_cast<size_t>(q)] = h->xregion;
        continue;
      }
      cudaIpcMemHandle_t hd;
      std::memcpy(&hd, static_cast<const char*>(handles) + 64 * q, sizeof(hd));
      void* base = nullptr;
      CK(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
      h->peer_bases.push_back(base);
      bases[static_cast<size_t>(q)] = base;
    }
    p2p_wire(h, bases);
  });
}

int numpmp_gpu_p2p_connect_local(numpmp_gpu** hs, int world) {
  if (!hs || world < 1) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "bad handle list");
  std::vector<void*> bases(static_cast<size_t>(world));
  for (int q = 0; q < world; ++q) {
    if (!hs[q] || !hs[q]->xregion || hs[q]->p2p || hs[q]->world != world || hs[q]->rank != q)
      return set_err(hs[q], NUMPMP_INVALID_ARGUMENT, "not an unconnected peer-memory handle of this world");
    bases[static_cast<size_t>(q)] = hs[q]->xregion;
  }
  for (int q = 0; q < world; ++q) {
    numpmp_gpu* h = hs[q];
    try {
      CK(cudaSetDevice(h->device));
      for (int r = 0; r < world; ++r)
        if (hs[r]->device != h->device) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(hs[r]->device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
          cudaGetLastError();
        }
      p2p_wire(h, bases);
    } catch (const GpuError& e) {
      return set_err(h, e.code, e.msg);
    }
  }
  return NUMPMP_OK;
}

int numpmp_gpu_p2p_start(numpmp_gpu* h) {
  GUARD(h, {
    if (!h->p2p) throw GpuError{NUMPMP_INVALID_ARGUMENT, "peer-memory handle is not connected"};
    CK(cudaSetDevice(h->device));
    // Global link degrees and nnz: sums of the shards' local counts
    // (exact in fp64).
    k_int_to_double<<<grid_for(h->m), 256, 0, h->stream>>>(h->deg, h->m, h->scratch_m);
    CK(cudaGetLastError());
    p2p_allreduce(h, h->scratch_m, h->scratch_m);
    k_double_to_int<<<grid_for(h->m), 256, 0, h->stream>>>(h->scratch_m, h->m, h->deg);
    CK(cudaGetLastError());
    const double nnz_local = static_cast<double>(h->nnz);
    CK(cudaMemcpyAsync(h->scalars, &nnz_local, 8, cudaMemcpyHostToDevice, h->stream));
    p2p_allreduce_scalars(h, h->scalars, 1);
    double nnz_global = 0.0;
    CK(cudaMemcpyAsync(&nnz_global, h->scalars, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->nnz_total = static_cast<int64_t>(nnz_global);
    do_set_cold(h);
  });
}

int numpmp_gpu_set_cold(numpmp_gpu* h) { GUARD(h, do_set_cold(h)); }

int numpmp_gpu_warm_after_degrade(numpmp_gpu* h, const double* cap_before, const double* prior_x,
                                  const double* prior_lambda_raw, double prior_rho, double* x0_out,
                                  double* price_out, double* rho_out) {
  GUARD(h, do_warm_after_degrade(h, cap_before, prior_x, prior_lambda_raw, prior_rho, x0_out,
                                 price_out, rho_out));
}

int numpmp_gpu_warm_after_prune(numpmp_gpu* h, const double* x0_proj, const double* price_proj,
                                double prior_rho, double* x0_out, double* price_out, double* rho_out) {
  GUARD(h, do_warm_after_prune(h, x0_proj, price_proj, prior_rho, x0_out, price_out, rho_out));
}

int numpmp_gpu_path_prices(numpmp_gpu* h, const double* lambda, double* pi) {
  GUARD(h, {
    if (!lambda || !pi) throw GpuError{NUMPMP_INVALID_ARGUMENT, "path_prices: null array"};
    upload(h, h->scratch_m2, lambda, 8 * static_cast<size_t>(h->m));
    k_path_prices<<<grid_for(h->n), 256, 0, h->stream>>>(h->col_ptr, h->row_idx, h->n,
                                                         h->scratch_m2, h->scratch_n);
    CK(cudaGetLastError());
    download(h, pi, h->scratch_n, 8 * static_cast<size_t>(h->n));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int numpmp_gpu_set_warm(numpmp_gpu* h, const double* x0, const double* price, double rho) {
  GUARD(h, do_set_warm(h, x0, price, rho));
}

namespace {
uint64_t state_fingerprint(const double* p, const double* z, const double* p_bar, const double* price,
                           size_t J, size_t m, double rho, int64_t iter);
}  // namespace

// Loads an arbitrary terminal-space state.  z is decomposed as
// z_t = A_j - B_l by a breadth-first walk over each connected component of
// the stream/link incidence (root link potential B = 0), then verified.
int numpmp_gpu_set_state(numpmp_gpu* h, const double* p, const double* z, const double* p_bar,
                         const double* price, double rho, int64_t iter) {
  GUARD(h, {
    if (h->sharded)
      throw GpuError{NUMPMP_INVALID_ARGUMENT, "set_state is not supported on sharded handles"};
    if (!p || !z || !p_bar || !price)
      throw GpuError{NUMPMP_INVALID_ARGUMENT, "state arrays must not be null"};
    if (!(rho > 0.0)) throw GpuError{NUMPMP_INVALID_ARGUMENT, "state rho must be > 0"};
    const int64_t n = h->n, m = h->m, nnz = h->nnz;
    if (h->issued_valid &&
        state_fingerprint(p, z, p_bar, price, static_cast<size_t>(nnz + m), static_cast<size_t>(m), rho, iter) ==
            h->issued_fp) {
      return NUMPMP_OK;  // the state this handle issued last and still holds: nothing to upload
    }
    std::vector<int> col_ptr(static_cast<size_t>(n) + 1), row_idx(static_cast<size_t>(nnz));
    CK(cudaMemcpy(col_ptr.data(), h->col_ptr, 4 * (n + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(row_idx.data(), h->row_idx, 4 * nnz, cudaMemcpyDeviceToHost));
    // link -> (stream, terminal) adjacency on the host
    std::vector<int64_t> loff(static_cast<size_t>(m) + 1, 0);
    for (int64_t t = 0; t < nnz; ++t) ++loff[static_cast<size_t>(row_idx[static_cast<size_t>(t)]) + 1];
    for (int64_t l = 0; l < m; ++l) loff[static_cast<size_t>(l) + 1] += loff[static_cast<size_t>(l)];
    std::vector<int64_t> cursor(loff.begin(), loff.end() - 1), lterm(static_cast<size_t>(nnz));
    for (int64_t t = 0; t < nnz; ++t) lterm[static_cast<size_t>(cursor[static_cast<size_t>(row_idx[static_cast<size_t>(t)])]++)] = t;
    std::vector<int64_t> t2s(static_cast<size_t>(nnz));
    for (int64_t j = 0; j < n; ++j)
      for (int t = col_ptr[static_cast<size_t>(j)]; t < col_ptr[static_cast<size_t>(j) + 1]; ++t)
        t2s[static_cast<size_t>(t)] = j;
    std::vector<double> A(static_cast<size_t>(n), 0.0), Bv(static_cast<size_t>(m), 0.0);
    std::vector<char> seen_s(static_cast<size_t>(n), 0), seen_l(static_cast<size_t>(m), 0);
    std::vector<int64_t> queue;  // >= 0 link, < 0 stream (-(j+1))
    for (int64_t root = 0; root < m; ++root) {
      if (seen_l[static_cast<size_t>(root)]) continue;
      seen_l[static_cast<size_t>(root)] = 1;
      queue.assign(1, root);
      for (size_t qi = 0; qi < queue.size(); ++qi) {
        const int64_t node = queue[qi];
        if (node >= 0) {
          for (int64_t k = loff[static_cast<size_t>(node)]; k < loff[static_cast<size_t>(node) + 1]; ++k) {
            const int64_t t = lterm[static_cast<size_t>(k)];
            const int64_t j = t2s[static_cast<size_t>(t)];
            if (seen_s[static_cast<size_t>(j)]) continue;
            seen_s[static_cast<size_t>(j)] = 1;
            A[static_cast<size_t>(j)] = z[t] + Bv[static_cast<size_t>(node)];
            queue.push_back(-(j + 1));
          }
        } else {
          const int64_t j = -node - 1;
          for (int t = col_ptr[static_cast<size_t>(j)]; t < col_ptr[static_cast<size_t>(j) + 1]; ++t) {
            const int l = row_idx[static_cast<size_t>(t)];
            if (seen_l[static_cast<size_t>(l)]) continue;
            seen_l[static_cast<size_t>(l)] = 1;
            Bv[static_cast<size_t>(l)] = A[static_cast<size_t>(j)] - z[t];
            queue.push_back(l);
          }
        }
      }
    }
    for (int64_t j = 0; j < n; ++j)
      for (int t = col_ptr[static_cast<size_t>(j)]; t < col_ptr[static_cast<size_t>(j) + 1]; ++t) {
        const double rec =
            A[static_cast<size_t>(j)] - Bv[static_cast<size_t>(row_idx[static_cast<size_t>(t)])];
        const double scale = std::max({1.0, std::fabs(z[t]), std::fabs(A[static_cast<size_t>(j)])});
        if (!(std::fabs(rec - z[t]) <= 1e-12 * scale))
          throw GpuError{NUMPMP_INVALID_ARGUMENT,
                         "state: z is not decomposable as A_j - B_l over the incidence"};
      }
    h->cur = 0;
    const size_t nb = 8 * static_cast<size_t>(n), mb = 8 * static_cast<size_t>(m);
    upload(h, h->A[0], A.data(), nb);
    upload(h, h->B[0], Bv.data(), mb);
    upload(h, h->zs[0], z + nnz, mb);
    upload(h, h->pr[0], price, mb);
    // stream rates of the given p (first terminal of each stream), for get_state
    std::vector<double> x0(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) x0[static_cast<size_t>(j)] = p[col_ptr[static_cast<size_t>(j)]];
    upload(h, h->x, x0.data(), nb);
    global_row_sums(h, h->A[0], h->Q[0]);  // Q = R A
    h->host_p.assign(p, p + nnz + m);
    h->host_pbar.assign(p_bar, p_bar + m);
    h->host_p_valid = true;
    h->iters_since_upload = 0;
    reset_ctrl(h, rho, iter);
  });
}

namespace {

// Fingerprint of a terminal-space state (4 independent multiply-xor lanes
// over the raw 64-bit words): set_state recognises the state get_state
// issued last.
uint64_t state_fingerprint(const double* p, const double* z, const double* p_bar, const double* price,
                           size_t J, size_t m, double rho, int64_t iter) {
  uint64_t h[4] = {0x243f6a8885a308d3ull, 0x13198a2e03707344ull, 0xa4093822299f31d0ull, 0x082efa98ec4e6c89ull};
  auto mix = [&](const double* a, size_t n) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(a);
    size_t i = 0;
    for (; i + 4 <= n; i += 4)
      for (int k = 0; k < 4; ++k) h[k] = (h[k] ^ w[i + k]) * 0x100000001b3ull;
    for (; i < n; ++i) h[0] = (h[0] ^ w[i]) * 0x100000001b3ull;
    for (int k = 0; k < 4; ++k) h[k] ^= h[k] >> 29;
  };
  mix(p, J);
  mix(z, J);
  mix(p_bar, m);
  mix(price, m);
  mix(&rho, 1);
  uint64_t it = static_cast<uint64_t>(iter);
  mix(reinterpret_cast<const double*>(&it), 1);
  return h[0] ^ (h[1] * 3) ^ (h[2] * 5) ^ (h[3] * 7);
}

// The current state in terminal space on the device (get_state, step):
// p / z / prev_z (length J, any may be null) and the device pointers of the
// slack flows and link averages.
void materialize_state(numpmp_gpu* h, const Ctrl& c, double* dp, double* dz, double* dzp, double** ps_out,
                       double** pbar_out) {
  const int64_t n = h->n, m = h->m, nnz = h->nnz;
  const int cu = h->cur, pv = h->cur ^ 1;
  double* ps_d = h->ps0;
  double* pbar_d = h->pbar0;
  if (h->iters_since_upload > 0) {
    // slack flows and averages of the last iteration, same arithmetic
    global_row_sums(h, h->x, h->scratch_m);
    k_materialize_links<<<grid_for(m), 256, 0, h->stream>>>(
        h->scratch_m, h->deg, nullptr, h->cap, h->zs[pv], h->pr[pv], c.rho_iter, m,
        h->scratch_m2, h->Lbuf);
    CK(cudaGetLastError());
    ps_d = h->scratch_m2;
    pbar_d = h->Lbuf;
  }
  if (dp || dz || dzp) {
    k_expand_terminals<<<grid_for(n), 256, 0, h->stream>>>(
        h->col_ptr, h->row_idx, n, h->x, h->A[cu], h->B[cu], h->A[pv], h->B[pv], dp, dz, dzp);
    CK(cudaGetLastError());
    if (dp) CK(cudaMemcpyAsync(dp + nnz, ps_d, 8 * m, cudaMemcpyDeviceToDevice, h->stream));
    if (dz) CK(cudaMemcpyAsync(dz + nnz, h->zs[cu], 8 * m, cudaMemcpyDeviceToDevice, h->stream));
    if (dzp) CK(cudaMemcpyAsync(dzp + nnz, h->zs[pv], 8 * m, cudaMemcpyDeviceToDevice, h->stream));
  }
  if (ps_out) *ps_out = ps_d;
  if (pbar_out) *pbar_out = pbar_d;
}

// r, s of residuals() (solver.hpp:139-154) from device arrays (k_residual_parts).
void device_residuals(numpmp_gpu* h, const double* pbar_d, const double* z_d, const double* zp_d, double rho,
                      double* r_norm, double* s_norm) {
  double* part = nullptr;
  CK(lib_malloc_async(reinterpret_cast<void**>(&part), 16 * kResidualGrid, h->stream));
  k_residual_parts<<<kResidualGrid, kThreads, 0, h->stream>>>(pbar_d, h->deg, h->m, z_d, zp_d, h->nnz + h->m,
                                                              rho, part);
  CK(cudaGetLastError());
  k_sum_parts<<<1, kThreads, 0, h->stream>>>(part, kResidualGrid, h->scalars);
  CK(cudaGetLastError());
  double rs[2] = {0.0, 0.0};
  CK(cudaMemcpyAsync(rs, h->scalars, 16, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFreeAsync(part, h->stream);
  *r_norm = std::sqrt(rs[0]);
  *s_norm = std::sqrt(rs[1]);
}

}  // namespace

int numpmp_gpu_get_state(numpmp_gpu* h, double* p, double* z, double* p_bar, double* price,
                         double* rho, int64_t* iter, double* prev_z) {
  GUARD(h, {
    const Ctrl c = read_ctrl(h);
    const int64_t m = h->m, nnz = h->nnz;
    const bool stepped = h->iters_since_upload > 0;
    if (rho) *rho = c.rho;
    if (iter) *iter = c.iter;
    if (price) download(h, price, h->pr[h->cur], 8 * static_cast<size_t>(m));
    const size_t J = static_cast<size_t>(nnz + m);
    double *dp = nullptr, *dz = nullptr, *dzp = nullptr;
    if (p) CK(lib_malloc_async(reinterpret_cast<void**>(&dp), 8 * J, h->stream));
    if (z) CK(lib_malloc_async(reinterpret_cast<void**>(&dz), 8 * J, h->stream));
    if (prev_z) CK(lib_malloc_async(reinterpret_cast<void**>(&dzp), 8 * J, h->stream));
    double* pbar_d = nullptr;
    materialize_state(h, c, dp, dz, dzp, nullptr, &pbar_d);
    if (p) download(h, p, dp, 8 * J);
    if (z) download(h, z, dz, 8 * J);
    if (prev_z) download(h, prev_z, dzp, 8 * J);
    if (p_bar) download(h, p_bar, pbar_d, 8 * static_cast<size_t>(m));
    CK(cudaStreamSynchronize(h->stream));
    cudaFreeAsync(dp, h->stream);
    cudaFreeAsync(dz, h->stream);
    cudaFreeAsync(dzp, h->stream);
    if (!stepped && h->host_p_valid) {
      if (p) std::memcpy(p, h->host_p.data(), 8 * J);
      if (p_bar) std::memcpy(p_bar, h->host_pbar.data(), 8 * static_cast<size_t>(m));
    }
    h->issued_valid = false;
    if (p && z && p_bar && price && !h->sharded) {
      h->issued_fp = state_fingerprint(p, z, p_bar, price, J, static_cast<size_t>(m), c.rho, c.iter);
      h->issued_valid = true;
    }
  });
}

// Replaces residuals(state, prev, layout) (solver.hpp:139-154) with the
// device reduction numpmp_gpu_step uses.
int numpmp_gpu_residuals(numpmp_gpu* h, const double* p_bar, const double* z, const double* prev_z,
                         double rho, double* r_norm, double* s_norm) {
  GUARD(h, {
    if (h->sharded) throw GpuError{NUMPMP_INVALID_ARGUMENT, "residuals is not supported on sharded handles"};
    if (!p_bar || !z || !prev_z || !r_norm || !s_norm)
      throw GpuError{NUMPMP_INVALID_ARGUMENT, "residuals: arrays must not be null"};
    const size_t J = static_cast<size_t>(h->nnz + h->m), mb = 8 * static_cast<size_t>(h->m);
    double *dpb = nullptr, *dz = nullptr, *dzp = nullptr;
    CK(lib_malloc_async(reinterpret_cast<void**>(&dpb), mb, h->stream));
    CK(lib_malloc_async(reinterpret_cast<void**>(&dz), 8 * J, h->stream));
    CK(lib_malloc_async(reinterpret_cast<void**>(&dzp), 8 * J, h->stream));
    upload(h, dpb, p_bar, mb);
    upload(h, dz, z, 8 * J);
    upload(h, dzp, prev_z, 8 * J);
    device_residuals(h, dpb, dz, dzp, rho, r_norm, s_norm);
    cudaFreeAsync(dpb, h->stream);
    cudaFreeAsync(dz, h->stream);
    cudaFreeAsync(dzp, h->stream);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int numpmp_gpu_step(numpmp_gpu* h, double* r_norm, double* s_norm) {
  GUARD(h, {
    h->issued_valid = false;
    {  // a previous run left `done` set: clear the run control (as run_loop does)
      Ctrl c = read_ctrl(h);
      c.run_k = 0;
      c.done = 0;
      c.status = ST_RUNNING;
      c.ticket = 0;
      c.ticket2 = 0;
      c.ticket3 = 0;
      std::memcpy(&h->ctrl_host[1], &c, sizeof(Ctrl));
      CK(cudaMemcpyAsync(h->ctrl, &h->ctrl_host[1], sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream));
    }
    enqueue_iteration(h, h->cur, MODE_STEP, nullptr, false);
    if (h->p2p) p2p_sync_link_state(h);
    const Ctrl c = read_ctrl(h);
    h->cur ^= 1;
    h->iters_since_upload += 1;
    double r = c.r_norm, s = c.s_norm;
    if (!h->sharded) {
      // step() returns residuals(after, before) (solver.hpp:316-318): the
      // direct terminal-space form on the materialised states, the same
      // reduction numpmp_gpu_residuals runs on host copies of them
      const size_t J = static_cast<size_t>(h->nnz + h->m);
      double *dz = nullptr, *dzp = nullptr, *pbar_d = nullptr;
      CK(lib_malloc_async(reinterpret_cast<void**>(&dz), 8 * J, h->stream));
      CK(lib_malloc_async(reinterpret_cast<void**>(&dzp), 8 * J, h->stream));
      materialize_state(h, c, nullptr, dz, dzp, nullptr, &pbar_d);
      device_residuals(h, pbar_d, dz, dzp, c.rho_iter, &r, &s);
      cudaFreeAsync(dz, h->stream);
      cudaFreeAsync(dzp, h->stream);
      CK(cudaStreamSynchronize(h->stream));
    }
    if (r_norm) *r_norm = r;
    if (s_norm) *s_norm = s;
  });
}

namespace {

// The device-controlled loop of PmpSolver::run (solver.hpp:450-476).
// Batches of kBatchIters iterations are launched as one CUDA graph; the
// host looks at the control block of batch b only after batch b+1 is
// queued, so the device never idles on the host.  Kernels queued after
// the device set `done` exit at entry.
void run_loop(numpmp_gpu* h) {
  PhaseTimer pt;
  h->issued_valid = false;
  const int start = h->cur;
  const int lpi = h->launches_per_iteration();
  const size_t set_size = static_cast<size_t>(kBatchIters * lpi + 1);
  if (h->profiling) {
    if (h->prof_ev.empty()) {
      h->prof_ev.resize(2 * set_size);
      for (auto& e : h->prof_ev) CK(cudaEventCreate(&e));
    }
    for (int set = 0; set < 2; ++set)
      if (!h->prof_graph[start][set]) h->prof_graph[start][set] = build_graph(h, start, set);
  } else if (!h->graph[start]) {
    h->graph[start] = build_graph(h, start, -1);
  }
  // fresh run: control counters, trace, device clock
  {
    Ctrl c = read_ctrl(h);
    c.run_k = 0;
    c.trace_len = 0;
    c.done = 0;
    c.status = ST_RUNNING;
    c.ticket = 0;
    c.ticket2 = 0;
    c.ticket3 = 0;
    std::memcpy(&h->ctrl_host[1], &c, sizeof(Ctrl));
    CK(cudaMemcpyAsync(h->ctrl, &h->ctrl_host[1], sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  if (!h->ev_run[0]) {
    CK(cudaEventCreate(&h->ev_run[0]));
    CK(cudaEventCreate(&h->ev_run[1]));
  }
  CK(cudaEventRecord(h->ev_run[0], h->stream));
  pt.mark("run: graph + control reset");
  k_start_clock<<<1, 1, 0, h->stream>>>(h->ctrl);
  CK(cudaGetLastError());
  // Per-kernel event times of a finished batch (profiling mode): only the
  // iterations that batch actually ran count.
  int64_t k_seen = 0;
  auto account = [&](int set, const Ctrl& c) {
    const int64_t ran = c.run_k - k_seen;
    for (int64_t i = 0; i < ran && i < kBatchIters; ++i) {
      for (int l = 0; l < lpi; ++l) {
        float t = 0.f;
        const size_t e0 = static_cast<size_t>(set) * set_size + static_cast<size_t>(i * lpi + l);
        CK(cudaEventElapsedTime(&t, h->prof_ev[e0], h->prof_ev[e0 + 1]));
        if (h->launch_side[static_cast<size_t>(l)] == 1)
          h->prof_ms_k1 += t;
        else
          h->prof_ms_k2 += t;
      }
      h->prof_iters += 1;
    }
    k_seen = c.run_k;
  };
  int inflight = 0, slot = 0;
  bool done = false;
  while (!done) {
    CK(cudaGraphLaunch(h->profiling ? h->prof_graph[start][slot] : h->graph[start], h->stream));
    CK(cudaMemcpyAsync(h->ctrl_host + slot, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaEventRecord(h->ev_batch[slot], h->stream));
    ++inflight;
    h->prof_launches += static_cast<int64_t>(kBatchIters) * lpi;
    if (inflight == 2) {
      const int prev = slot ^ 1;
      CK(cudaEventSynchronize(h->ev_batch[prev]));
      if (h->profiling) account(prev, h->ctrl_host[prev]);
      done = h->ctrl_host[prev].done != 0;
      --inflight;
    }
    slot ^= 1;
  }
  if (h->profiling) {  // the last batch queued (ran nothing if `done` was already set)
    CK(cudaEventSynchronize(h->ev_batch[slot ^ 1]));
    account(slot ^ 1, h->ctrl_host[slot ^ 1]);
  }
  CK(cudaEventRecord(h->ev_run[1], h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const Ctrl c = read_ctrl(h);
  {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev_run[0], h->ev_run[1]));
    h->last_run_ms = ms;
  }
  pt.mark("run: iteration loop");
  if (h->p2p) p2p_sync_link_state(h);
  h->run_iters = c.run_k;
  h->iters_since_upload += c.run_k;
  h->cur = static_cast<int>((start + c.run_k) & 1);
  if (c.status == ST_NONFINITE)
    throw GpuError{NUMPMP_SOLVER_ERROR,
                   "non-finite state at iteration " + std::to_string(c.run_k)};
  h->last_status = c.status == ST_CONVERGED ? NUMPMP_CONVERGED
                   : c.status == ST_TIMELIMIT ? NUMPMP_TIMELIMIT
                                              : NUMPMP_MAXITERS;
}

// Solution post-processing (solver.hpp:478-504) on the device.
void post_process(numpmp_gpu* h, double* x, double* s, double* lambda, double* lambda_raw,
                  numpmp_solution_info* info, numpmp_trace_row* trace, int64_t trace_cap) {
  PhaseTimer pt;
  const Ctrl c = read_ctrl(h);
  const int cu = h->cur;
  const int gpost = std::min(grid_for(h->n), h->grid1);
  k_post_streams<<<gpost, kThreads, 0, h->stream>>>(h->x, h->w, h->kind, h->n, h->cfg.eps_abs,
                                                   h->scratch_n, h->k1_part);
  CK(cudaGetLastError());
  k_sum_parts<<<1, kThreads, 0, h->stream>>>(h->k1_part, gpost, h->scalars);
  CK(cudaGetLastError());
  if (h->p2p)
    p2p_allreduce_scalars(h, h->scalars, 2);
  else if (h->sharded)
    NK(AllReduce(h->scalars, h->scalars, 2, ncclDouble, ncclSum, h->comm, h->stream));
  global_row_sums(h, h->scratch_n, h->scratch_m);  // load = R x (clamped x)
  k_post_links<<<grid_for(h->m), 256, 0, h->stream>>>(h->scratch_m, h->cap, h->pr[cu], h->m,
                                                      h->scratch_m2, h->Lbuf);
  CK(cudaGetLastError());
  double obj[2] = {0.0, 0.0};
  CK(cudaMemcpyAsync(obj, h->scalars, 16, cudaMemcpyDeviceToHost, h->stream));
  if (x) download(h, x, h->scratch_n, 8 * static_cast<size_t>(h->n));
  if (s) download(h, s, h->scratch_m2, 8 * static_cast<size_t>(h->m));
  if (lambda) download(h, lambda, h->Lbuf, 8 * static_cast<size_t>(h->m));
  if (lambda_raw) download(h, lambda_raw, h->pr[cu], 8 * static_cast<size_t>(h->m));
  int64_t tl = std::min<int64_t>(c.trace_len, h->trace_cap);
  std::vector<numpmp_trace_row> rows(static_cast<size_t>(tl) + 1);
  if (tl > 0) download(h, rows.data(), h->trace_dev, sizeof(numpmp_trace_row) * tl);
  CK(cudaStreamSynchronize(h->stream));
  // Final trace sample (solver.hpp:478-481).
  if (tl == 0 || rows[static_cast<size_t>(tl) - 1].iter != c.iter) {
    numpmp_trace_row& r = rows[static_cast<size_t>(tl)];
    r.iter = c.iter;
    r.r_norm = c.r_norm;
    r.s_norm = c.s_norm;
    r.rho = c.rho;
    r.objective = obj[1];
    ++tl;
  }
  pt.mark("post-process + download");
  if (trace)
    std::memcpy(trace, rows.data(),
                sizeof(numpmp_trace_row) * static_cast<size_t>(std::min(tl, trace_cap)));
  if (info) {
    info->objective = obj[0];
    info->r_norm = c.r_norm;
    info->s_norm = c.s_norm;
    info->rho_final = c.rho;
    info->iterations = c.iter;
    info->status = h->last_status;
    info->trace_len = tl;
  }
}

}  // namespace

int numpmp_gpu_run(numpmp_gpu* h, double* x, double* s, double* lambda, double* lambda_raw,
                   numpmp_solution_info* info, numpmp_trace_row* trace, int64_t trace_cap) {
  GUARD(h, {
    run_loop(h);
    post_process(h, x, s, lambda, lambda_raw, info, trace, trace_cap);
  });
}

int numpmp_gpu_run_device(numpmp_gpu* h, numpmp_solution_info* info) {
  GUARD(h, {
    run_loop(h);
    const Ctrl c = read_ctrl(h);
    if (info) {
      std::memset(info, 0, sizeof(*info));
      info->r_norm = c.r_norm;
      info->s_norm = c.s_norm;
      info->rho_final = c.rho;
      info->iterations = c.iter;
      info->status = h->last_status;
      info->trace_len = c.trace_len;
    }
  });
}

int numpmp_gpu_export_layout(numpmp_gpu* h, int64_t* link_offsets, int64_t* link_terminals,
                             int32_t* link_counts) {
  GUARD(h, {
    if (h->sharded)
      throw GpuError{NUMPMP_INVALID_ARGUMENT, "export_layout is not supported on sharded handles"};
    const int64_t m = h->m, nnz = h->nnz;
    // The global link-major CSR built on the device exactly as the column
    // blocks are, plus the terminal ids the sort carried along.
    int64_t tmpb = 0;
    int* rp = dalloc<int>(static_cast<size_t>(m) + 1, &tmpb, h->stream);
    int* ci = dalloc<int>(static_cast<size_t>(nnz) + kIdxPad, &tmpb, h->stream);
    std::vector<int> row_ptr(static_cast<size_t>(m) + 1), terms(static_cast<size_t>(nnz));
    try {
      build_csr(h, 0, h->n, rp, ci, terms.data());
      CK(cudaMemcpy(row_ptr.data(), rp, 4 * (m + 1), cudaMemcpyDeviceToHost));
    } catch (...) {
      cudaFreeAsync(rp, h->stream);
      cudaFreeAsync(ci, h->stream);
      throw;
    }
    cudaFreeAsync(rp, h->stream);
    cudaFreeAsync(ci, h->stream);
    // model.hpp:182-199: |l| = degree + 1, slack terminal nnz + l last.
    link_offsets[0] = 0;
    for (int64_t l = 0; l < m; ++l) {
      const int64_t d = row_ptr[static_cast<size_t>(l) + 1] - row_ptr[static_cast<size_t>(l)];
      if (link_counts) link_counts[l] = static_cast<int32_t>(d + 1);
      link_offsets[l + 1] = link_offsets[l] + d + 1;
      int64_t o = link_offsets[l];
      for (int k = row_ptr[static_cast<size_t>(l)]; k < row_ptr[static_cast<size_t>(l) + 1]; ++k)
        link_terminals[o++] = terms[static_cast<size_t>(k)];
      link_terminals[o] = nnz + l;
    }
  });
}

int numpmp_gpu_sizes(const numpmp_gpu* h, int64_t* m, int64_t* n, int64_t* nnz) {
  if (!h) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "null handle");
  if (m) *m = h->m;
  if (n) *n = h->n;
  if (nnz) *nnz = h->nnz;
  return NUMPMP_OK;
}

int numpmp_gpu_set_profiling(numpmp_gpu* h, int enable) {
  if (!h) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "null handle");
  h->profiling = enable != 0;
  h->prof_launches = 0;
  h->prof_iters = 0;
  h->prof_ms_k1 = 0.0;
  h->prof_ms_k2 = 0.0;
  return NUMPMP_OK;
}

int numpmp_gpu_profile(const numpmp_gpu* h, int64_t* launches, double* ms_stream_pass,
                       double* ms_link_pass, int64_t* iterations_timed) {
  if (!h) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "null handle");
  if (launches) *launches = h->prof_launches;
  if (ms_stream_pass) *ms_stream_pass = h->prof_ms_k1;
  if (ms_link_pass) *ms_link_pass = h->prof_ms_k2;
  if (iterations_timed) *iterations_timed = h->prof_iters;
  return NUMPMP_OK;
}

int numpmp_gpu_last_run_ms(const numpmp_gpu* h, double* ms) {
  if (!h) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "null handle");
  if (ms) *ms = h->last_run_ms;
  return NUMPMP_OK;
}

int numpmp_gpu_pin_host(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return NUMPMP_OK;
  cudaError_t e = cudaHostRegister(ptr, static_cast<size_t>(bytes), cudaHostRegisterDefault);
  if (e != cudaSuccess) return set_err(nullptr, NUMPMP_CUDA_ERROR, cudaGetErrorString(e));
  return NUMPMP_OK;
}

int numpmp_gpu_unpin_host(void* ptr) {
  if (!ptr) return NUMPMP_OK;
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) return set_err(nullptr, NUMPMP_CUDA_ERROR, cudaGetErrorString(e));
  return NUMPMP_OK;
}

int numpmp_gpu_transfer_bytes(const numpmp_gpu* h, int64_t* h2d, int64_t* d2h) {
  if (!h) return set_err(nullptr, NUMPMP_INVALID_ARGUMENT, "null handle");
  if (h2d) *h2d = h->h2d;
  if (d2h) *d2h = h->d2h;
  return NUMPMP_OK;
}

void numpmp_gpu_destroy(numpmp_gpu* h) {
  if (!h) return;
  NvtxRange nvtx_range_("numpmp_gpu_destroy");
  PhaseTimer pt;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->l2_guard_held) l2_guard().release(h->device);
  for (void* base : h->peer_bases) cudaIpcCloseMemHandle(base);
  if (h->xregion) {
    cudaFree(h->xregion);
    h->v = h->v_alt[0] = h->v_alt[1] = nullptr;  // lived in the exchange region
  }
  std::vector<void*> bufs = {h->col_ptr, h->row_idx, h->w,         h->kind,       h->deg,
                             h->cap,     h->x,       h->v,         h->ps0,        h->pbar0,
                             h->done_cnt, h->ep_part, h->peer_tables,
                             h->v_alt[0], h->v_alt[1],
                             h->Lbuf,    h->Lacc,    h->k1_part,   h->k2_part,    h->scratch_m,
                             h->scratch_m2, h->scratch_n, h->scalars, h->ctrl, h->trace_dev};
  pt.mark("destroy: sync + ipc");
  for (int i = 0; i < 2; ++i) {
    if (h->graph[i]) cudaGraphExecDestroy(h->graph[i]);
    for (int set = 0; set < 2; ++set)
      if (h->prof_graph[i][set]) cudaGraphExecDestroy(h->prof_graph[i][set]);
    if (h->ev_batch[i]) cudaEventDestroy(h->ev_batch[i]);
    if (h->ev_run[i]) cudaEventDestroy(h->ev_run[i]);
    for (void* p : {static_cast<void*>(h->A[i]), static_cast<void*>(h->B[i]),
                    static_cast<void*>(h->zs[i]), static_cast<void*>(h->pr[i]),
                    static_cast<void*>(h->Q[i])})
      bufs.push_back(p);
  }
  for (auto& e : h->prof_ev) cudaEventDestroy(e);
  pt.mark("destroy: graphs + events");
  for (ColBlock& cb : h->blocks)
    for (void* p : {static_cast<void*>(cb.row_ptr), static_cast<void*>(cb.col_idx),
                    static_cast<void*>(cb.units), static_cast<void*>(cb.vptr),
                    static_cast<void*>(cb.vrow), static_cast<void*>(cb.pieces),
                    static_cast<void*>(cb.uctr), static_cast<void*>(cb.upart)})
      bufs.push_back(p);
  for (void* p : bufs)  // back to the (retained) stream-ordered pool
    if (p) {
      if (h->stream)
        cudaFreeAsync(p, h->stream);
      else
        cudaFree(p);
    }
  pt.mark("destroy: frees queued");
  if (h->ctrl_host) ctrl_pool().put(h->ctrl_host);
  if (h->comm) nccl().CommDestroy(h->comm);
  for (cudaEvent_t e : h->pipe_ev)
    if (e) cudaEventDestroy(e);
  if (h->stream2) cudaStreamDestroy(h->stream2);
  if (h->stream) {
    cudaStreamSynchronize(h->stream);
    cudaStreamDestroy(h->stream);
  }
  delete h;
  pt.mark("destroy");
}

}  // extern "C"
