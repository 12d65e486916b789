// Host side of the C ABI (include/robench_b200.h): engine lifecycle, pack
// upload, validation in the reference's order, kernel selection and launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include <map>
#include <condition_variable>
#include <functional>
#include <thread>

#include "rb_fnspec.cuh"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (no link dependency)

namespace rb {
extern const void* const kernels_f64[N_VARIANTS];
extern const void* const kernels_f32[N_VARIANTS];
extern const void* const kernels_spec_f64[FN_COUNT_SPEC];
extern const void* const kernels_spec_f32[FN_COUNT_SPEC];
extern const void* const fixup_f64;
extern const void* const plan_image_f64[2];     // [MT2]
extern const void* const plan_image_f32;
extern const void* const big_f64;
extern const void* const big_f32;
cudaError_t set_weier_f64x(const double* a_then_c);
cudaError_t set_weier_f32x(const float* a_then_c);
void phase_read_f64x(unsigned long long out[8], bool reset);
void phase_read_f32x(unsigned long long out[8], bool reset);
cudaError_t set_weier_f64(const double* a_then_c);
cudaError_t set_weier_f32(const float* a_then_c);
void phase_read_f64(unsigned long long out[8], bool reset);
void phase_read_f32(unsigned long long out[8], bool reset);

// ------------------------------------------------- on-device population
// numpy.random.Philox (Philox4x64-10) as numpy runs it: counter starting at
// 0 and incremented before each 4-word block, key from the SeedSequence;
// Generator.uniform(low, high) = low + (high - low) * ((u64 >> 11) * 2^-53).
// Element e of the stream comes from block e / 4 (counter e / 4 + 1), word
// e % 4, so any row range is generated independently (row-sharded ranks
// produce exactly their slice of the single-GPU population).
__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

__global__ void uniform_population_kernel(uint64_t k0, uint64_t k1, uint64_t first, int64_t n,
                                          double low, double high, double* out64, float* out32) {
  const double range = high - low;
  const uint64_t b0 = first / 4;                       // first block touched
  const uint64_t b1 = (first + (uint64_t)n + 3) / 4;   // one past the last
  for (uint64_t b = b0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < b1;
       b += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c[4] = {b + 1, 0, 0, 0};                  // 256-bit counter b + 1 (b < 2^64 - 1)
    philox4x64_10(c, k0, k1);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint64_t e = b * 4 + w;
      if (e < first || e >= first + (uint64_t)n) continue;
      const double u = (double)(c[w] >> 11) * (1.0 / 9007199254740992.0);
      const double x = low + range * u;
      if (out64) out64[e - first] = x;
      if (out32) out32[e - first] = (float)x;
    }
  }
}

// The fitness all-gather of the single-process multi-device path
// (rb_func_evaluate_sharded): one device's slice of f stored into every
// peer's full-length f over NVLink (P2P stores; peers' slices are disjoint).
constexpr int kMaxDevices = 16;
struct PeerDst {
  void* p[kMaxDevices];
  int n;
};

template <class T>
__global__ void peer_scatter_kernel(const T* __restrict__ src, int64_t n, PeerDst dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = src[i];
    for (int k = 0; k < dst.n; ++k) static_cast<T*>(dst.p[k])[i] = v;
  }
}

// float32 rows from float64 rows (engine.py:201's astype: round to nearest)
__global__ void cast_rows_kernel(const double* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __double2float_rn(x[i]);
}

__global__ void np_powf_kernel(const float* x, const float* y, float* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rb_svml::powf_np(x[i], y[i]);
}
}  // namespace rb

namespace {

// NVTX range over a C-ABI call (tracing); ~free when no
// tool is attached.  Shows the API boundary beside the kernels in nsys /
// ncu --nvtx timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
constexpr uint32_t kFlagSlots = 4096;      // a power of two: slot = counter & (kFlagSlots - 1)
constexpr int kSlotInts = 4;               // [0] non-finite, [1] rows left for fixup, [2] call number
static_assert((kFlagSlots & (kFlagSlots - 1)) == 0, "flag ring must be a power of two");

// cudaFuncAttributeMaxDynamicSharedMemorySize is process-wide per (device,
// kernel), while engines of different dims and function sets coexist: it is
// only ever raised, to the largest need any engine has declared.
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, size_t> g_attr;

rb_status fail(rb_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

#define RB_CUDA(call)                                                               \
  do {                                                                              \
    cudaError_t err_ = (call);                                                      \
    if (err_ != cudaSuccess)                                                        \
      return fail(RB_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(err_)); \
  } while (0)

template <class X>
rb_status upload(X** dst, const X* src, int64_t count) {
  *dst = nullptr;
  if (count <= 0) return RB_OK;
  RB_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), sizeof(X) * count));
  RB_CUDA(cudaMemcpy(*dst, src, sizeof(X) * count, cudaMemcpyHostToDevice));
  return RB_OK;
}

int pad_to(int v, int mod, int rem) {   // smallest u >= v with u % mod == rem
  int u = v;
  while (u % mod != rem) ++u;
  return u;
}

// Launch configuration of one (function, precision).
struct Launch {
  const void* func = nullptr;
  size_t smem = 0;
  int grid_cap = 0;
  int ldv = 0, max_q = 0;
  int nbuf = 1;
  int opt_rows = 0;
  bool mt2 = false;                 // float64 DMMA units cover both m-tiles (rb_device.cuh MT2)
  bool big = false;                 // evaluate_big_kernel: tiles in global scratch (per_cta bytes per CTA)
  size_t per_cta = 0;
  size_t smem_nbuf[3] = {0, 0, 0};
};

// RB_BIG=1 serves every function with evaluate_big_kernel (tests: the
// large-dimension path at dimensions whose tiles fit).
int big_mode() {
  const char* v = std::getenv("RB_BIG");
  return v ? std::atoi(v) : 0;
}

// RB_PREFETCH=0/1 forces single / double X buffering (default: auto).
int prefetch_mode() {
  const char* v = std::getenv("RB_PREFETCH");
  return v ? std::atoi(v) : -1;
}

// RB_SPEC=0 keeps hybrids / compositions on the generic kernel.
int spec_mode() {
  const char* v = std::getenv("RB_SPEC");
  return v ? std::atoi(v) : 1;
}

// RB_L2PF=0 disables the L2 prefetch of upcoming X tiles (default on).
int l2_prefetch() {
  static const int v = [] {
    const char* e = std::getenv("RB_L2PF");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

}  // namespace

struct rb_engine {
  int device = 0;
  int dim = 0;
  int64_t max_concurrency = 0;
  int ldz[2] = {0, 0};                       // [0] fp64, [1] fp32
  std::vector<rb_function> fns;              // host copy for validation
  std::vector<std::string> why[2];           // per precision: non-empty = function unsupported
  std::vector<int> fixup;                    // float64: bitmask of exact64 members (fixup_kernel)
  int fixup_grid = 0;
  std::vector<Launch> launch[2];
  rb_function* d_fns = nullptr;              // [precision]: function records + plan images
  rb_function* d_fns32 = nullptr;
  rb_member* d_members = nullptr;
  rb_segment* d_segments = nullptr;
  rb_group* d_groups = nullptr;
  int32_t* d_index = nullptr;
  double* d_v64 = nullptr;
  float* d_v32 = nullptr;
  int* h_flags = nullptr;                    // ring of per-call non-finite flags, mapped
  int* d_flags = nullptr;                    // pinned host memory (device alias of h_flags)
  int* d_marks = nullptr;                    // device memory, one word per flag slot (Args::mark)
  std::atomic<uint32_t> next_flag{0};
  std::mutex host_mu;                        // host-pointer API pipeline (evaluate_host_locked)
  void* pin_x[2] = {nullptr, nullptr};       // pinned row chunks
  void* pin_f[2] = {nullptr, nullptr};       // pinned values of a chunk
  void* dev_x[2] = {nullptr, nullptr};
  void* dev_f[2] = {nullptr, nullptr};
  int64_t chunk_rows = 0;                    // capacity of each buffer, in rows
  cudaStream_t copy_stream = nullptr;        // H2D of row chunks
  cudaStream_t d2h_stream = nullptr;         // many-call path: D2H of a chunk's values
  cudaEvent_t computed[2] = {nullptr, nullptr};
  cudaStream_t many_stream2 = nullptr;       // many-call path: every other call of a chunk
  cudaEvent_t computed2[2] = {nullptr, nullptr}, ready2 = nullptr;
  cudaEvent_t x_ready[2] = {nullptr, nullptr}, f_ready[2] = {nullptr, nullptr};
  float* dev_x32 = nullptr;                  // many-call host path: the float32 rows of a chunk
  void* pin_xm[2] = {nullptr, nullptr};      // ... its (larger) row chunks
  void* dev_xm[2] = {nullptr, nullptr};
  int64_t many_rows = 0;
  void* pin_fm[2] = {nullptr, nullptr};      // ... and every call's values of a chunk
  void* dev_fm[2] = {nullptr, nullptr};
  int fm_calls = 0;                          // capacity of pin_fm / dev_fm, in calls
  cudaStream_t host_stream = nullptr;
  std::mutex fork_mu;                        // rb_func_evaluate_many: the fork stream's record/wait pairs
  cudaStream_t fork_stream = nullptr;        // ... every other call of a batch, joined back to the caller's
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
};

// A replica of the engine on each of several devices:
// rows are sharded contiguously, each device evaluates its rows into its own
// full-length f and stores that slice into every peer's f (peer_scatter).
struct rb_sharded {
  std::vector<rb_engine*> eng;
  std::vector<int> dev;
  std::vector<cudaStream_t> streams;         // used when the caller passes none
  bool p2p = true;                           // every distinct pair has peer access
};

namespace {

void release(rb_engine* e) {
  if (!e) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(e->device);
  cudaFree(e->d_fns);
  cudaFree(e->d_fns32);
  cudaFree(e->d_members);
  cudaFree(e->d_segments);
  cudaFree(e->d_groups);
  cudaFree(e->d_index);
  cudaFree(e->d_v64);
  cudaFree(e->d_v32);
  for (int b = 0; b < 2; ++b) {
    cudaFree(e->dev_x[b]);
    cudaFree(e->dev_f[b]);
    if (e->pin_x[b]) cudaFreeHost(e->pin_x[b]);
    if (e->pin_f[b]) cudaFreeHost(e->pin_f[b]);
    if (e->x_ready[b]) cudaEventDestroy(e->x_ready[b]);
    if (e->f_ready[b]) cudaEventDestroy(e->f_ready[b]);
  }
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  if (e->d2h_stream) cudaStreamDestroy(e->d2h_stream);
  for (int b = 0; b < 2; ++b)
    if (e->computed[b]) cudaEventDestroy(e->computed[b]);
  if (e->many_stream2) cudaStreamDestroy(e->many_stream2);
  if (e->fork_stream) cudaStreamDestroy(e->fork_stream);
  if (e->fork_ev) cudaEventDestroy(e->fork_ev);
  if (e->join_ev) cudaEventDestroy(e->join_ev);
  for (int b = 0; b < 2; ++b)
    if (e->computed2[b]) cudaEventDestroy(e->computed2[b]);
  if (e->ready2) cudaEventDestroy(e->ready2);
  cudaFree(e->dev_x32);
  for (int b = 0; b < 2; ++b) {
    cudaFree(e->dev_xm[b]);
    if (e->pin_xm[b]) cudaFreeHost(e->pin_xm[b]);
  }
  for (int b = 0; b < 2; ++b) {
    cudaFree(e->dev_fm[b]);
    if (e->pin_fm[b]) cudaFreeHost(e->pin_fm[b]);
  }
  if (e->h_flags) cudaFreeHost(e->h_flags);
  cudaFree(e->d_marks);
  if (e->host_stream) cudaStreamDestroy(e->host_stream);
  cudaSetDevice(prev);
  delete e;
}

template <class T>
rb::Args<T> make_args(const rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f, int* dflag,
                      const Launch& L) {
  const int pi = sizeof(T) == 8 ? 0 : 1;
  rb::Args<T> a;
  a.x = x;
  a.f = f;
  a.n = n;
  a.dim = e->dim;
  a.fns = pi == 0 ? e->d_fns : e->d_fns32;
  a.members = e->d_members;
  a.segments = e->d_segments;
  a.groups = e->d_groups;
  a.index = e->d_index;
  a.values = reinterpret_cast<const T*>(pi == 0 ? (const void*)e->d_v64 : (const void*)e->d_v32);
  a.fn = fn_id;
  a.flag = dflag;
  a.mark = dflag ? e->d_marks + (dflag - e->d_flags) / kSlotInts : nullptr;
  a.ldz = e->ldz[pi];
  a.ldv = L.ldv;
  a.max_q = L.max_q;
  a.tma = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
  a.nbuf = L.nbuf;
  a.l2pf = l2_prefetch();
  a.neg_zero = -0.0f;
  a.opt_rows = L.opt_rows;
  return a;
}

// float64 re-evaluation of the rows the main kernel marked (fixup_kernel,
// rb_device.cuh exact64_kernel), stream-ordered behind it.
rb_status launch_fixup(rb_engine* e, int32_t fn_id, const double* x, int64_t n, double* f,
                       cudaStream_t stream, int* dflag) {
  const Launch& L = e->launch[0][fn_id];
  rb::Args<double> a = make_args<double>(e, fn_id, x, n, f, dflag, L);
  a.nbuf = 1;
  const int64_t nchunks = (n + rb::TP - 1) / rb::TP;
  const int grid = (int)std::min<int64_t>(nchunks, e->fixup_grid);
  void* args[] = {&a};
  RB_CUDA(cudaLaunchKernel(rb::fixup_f64, dim3(grid), dim3(rb::NT), args, L.smem_nbuf[1], stream));
  g_launches.fetch_add(1);
  return RB_OK;
}

// Validation in the reference's order (engine.py:180-203).
template <class T>
rb_status check_call(rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f) {
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (fn_id < 0 || fn_id >= (int32_t)e->fns.size())
    return fail(RB_E_UNKNOWN_FUNCTION, "function id " + std::to_string(fn_id) + " is not in 0..36");
  if (e->fns[fn_id].category == RB_DISABLED)
    return fail(RB_E_DISABLED_FUNCTION, "function " + std::to_string(fn_id) + " needs dimension >= 10");
  if (n > e->max_concurrency)
    return fail(RB_E_BATCH_TOO_LARGE, "batch of " + std::to_string(n) + " exceeds max_concurrency=" +
                                          std::to_string(e->max_concurrency));
  if (n < 1 || !x || !f) return fail(RB_E_INVALID_ARGUMENT, "empty batch or null pointer");
  const int pi = sizeof(T) == 8 ? 0 : 1;
  if (!e->why[pi][fn_id].empty())
    return fail(RB_E_UNSUPPORTED, "function " + std::to_string(fn_id) + ": " + e->why[pi][fn_id]);
  return RB_OK;
}

// Validation in the reference's order, then the launch on `stream`; the
// caller has made e->device current, synchronises and reads the flags
// (*flag_out: [0] non-finite input, [1] rows marked for the fixup pass).
// fixup_now: also queue the fixup pass of a float64 exact64 function behind
// the kernel (callers that do not inspect the flags before using f).
template <class T>
rb_status launch_eval(rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f,
                      cudaStream_t stream, volatile int** flag_out, bool fixup_now = false,
                      uint32_t* seq_out = nullptr) {
  const rb_status vs = check_call<T>(e, fn_id, x, n, f);
  if (vs != RB_OK) return vs;
  const int pi = sizeof(T) == 8 ? 0 : 1;
  const Launch& L = e->launch[pi][fn_id];

  const uint32_t seq = e->next_flag.fetch_add(1);
  const uint32_t slot = seq & (kFlagSlots - 1);
  if (seq_out) *seq_out = seq;
  // the flags live in mapped pinned memory: cleared by the host, set by the
  // kernel with a plain store over PCIe, read after the stream sync (no
  // memset / D2H copy that would queue behind bulk transfers on the copy
  // engines)
  volatile int* hflag = e->h_flags + kSlotInts * slot;
  hflag[0] = 0;
  hflag[1] = 0;
  hflag[2] = (int)seq;
  int* dflag = e->d_flags + kSlotInts * slot;

  rb::Args<T> a = make_args<T>(e, fn_id, x, n, f, dflag, L);
  const int64_t ntiles = (n + rb::TP - 1) / rb::TP;
  const int grid = (int)std::min<int64_t>(ntiles, L.grid_cap);
  if (L.big) {
    // per-CTA tiles in stream-ordered scratch (the pool caches it across calls)
    unsigned char* scratch = nullptr;
    size_t per_cta = L.per_cta;
    RB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), per_cta * grid, stream));
    void* args[] = {&a, &scratch, &per_cta};
    const cudaError_t err = cudaLaunchKernel(L.func, dim3(grid), dim3(rb::NT), args, L.smem, stream);
    cudaFreeAsync(scratch, stream);
    RB_CUDA(err);
    g_launches.fetch_add(1);
    *flag_out = hflag;
    return RB_OK;
  }
  void* args[] = {&a};
  if (sizeof(T) == 8 && e->fixup[fn_id])   // the kernel may mark rows: a clean word for this call
    RB_CUDA(cudaMemsetAsync(a.mark, 0, sizeof(int), stream));
  RB_CUDA(cudaLaunchKernel(L.func, dim3(grid), dim3(rb::NT), args, L.smem, stream));
  g_launches.fetch_add(1);
  if constexpr (sizeof(T) == 8) {
    if (fixup_now && e->fixup[fn_id]) {
      const rb_status st = launch_fixup(e, fn_id, x, n, f, stream, dflag);
      if (st != RB_OK) return st;
    }
  }
  *flag_out = hflag;
  return RB_OK;
}

rb_status non_finite() {
  return fail(RB_E_NON_FINITE_INPUT, "batch contains NaN or infinity (kernel input not finite)");
}

template <class T>
rb_status evaluate_device(rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f,
                          cudaStream_t stream) {
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  if (prev != e->device) RB_CUDA(cudaSetDevice(e->device));
  volatile int* flag = nullptr;
  rb_status s = launch_eval<T>(e, fn_id, x, n, f, stream, &flag);
  if (s == RB_OK) {
    cudaError_t err = cudaStreamSynchronize(stream);
    if (err == cudaSuccess && !flag[0] && flag[1]) {    // marked rows: the exact-order pass
      if constexpr (sizeof(T) == 8) {
        s = launch_fixup(e, fn_id, x, n, f, stream, const_cast<int*>(e->d_flags + (flag - e->h_flags)));
        if (s == RB_OK) err = cudaStreamSynchronize(stream);
      }
    }
    if (s != RB_OK) {
    } else if (err != cudaSuccess) {
      s = fail(RB_E_CUDA, std::string("cudaStreamSynchronize: ") + cudaGetErrorString(err));
    } else if (flag[0]) {
      s = non_finite();
    }
  }
  if (prev != e->device) cudaSetDevice(prev);
  return s;
}

// Host-pointer call (device current, host_mu held), pipelined in row chunks
// of ~kChunkBytes: while the GPU copies chunk c in (copy stream), evaluates
// it and copies its values out (engine stream), host threads stage chunk
// c+1 into the other pinned buffer -- a copy, or for float64 rows
// evaluated in float32 the rounding engine.py:201 does (astype = round to
// nearest) -- and the values of chunk c-1 leave their pinned buffer for the
// caller's f.  A batch of one chunk is one H2D, one launch, one D2H.  On an
// error the contents of f are unspecified (the reference returns nothing).
constexpr size_t kChunkBytes = size_t(32) << 20;

// Persistent host worker pool for the pipeline's staging copies (spawning
// threads per chunk cost ~0.3 ms per 32 MB chunk).  One job at a time
// (engines serialise on the pool); the calling thread takes part.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return (int)workers_.size() + 1; }
  // fn(lo, hi) over [0, n) split into size() contiguous ranges
  void run(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
    std::lock_guard<std::mutex> job(job_mu_);
    const int parts = size();
    const int64_t per = (n + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      per_ = per;
      pending_ = parts - 1;
      ++generation_;
    }
    cv_.notify_all();
    fn(0, std::min(n, per));
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    const char* v = std::getenv("RB_HOST_THREADS");                // staging threads (default 8)
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nt = std::min(v ? std::max(1, std::atoi(v)) : 8, hw);
    for (int t = 1; t < nt; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int64_t, int64_t)>* fn;
      int64_t lo, hi;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || generation_ != seen; });
        if (stop_) return;
        seen = generation_;
        fn = fn_;
        lo = t * per_;
        hi = std::min(n_, lo + per_);
      }
      if (lo < hi) (*fn)(lo, hi);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int64_t, int64_t)>* fn_ = nullptr;
  int64_t n_ = 0, per_ = 0;
  int pending_ = 0;
  uint64_t generation_ = 0;
  bool stop_ = false;
};

template <class F>
void parallel_rows(int64_t n, int64_t bytes, F&& fn) {
  if (bytes < (int64_t(1) << 21) || n < 16 || HostPool::get().size() <= 1) {
    fn(int64_t(0), n);
    return;
  }
  const std::function<void(int64_t, int64_t)> job = fn;
  HostPool::get().run(n, job);
}

rb_status ensure_pipeline(rb_engine* e) {
  if (e->chunk_rows > 0) return RB_OK;
  static const size_t chunk_bytes = [] {     // RB_CHUNK_MB: pipeline chunk (default 32 MB)
    const char* v = std::getenv("RB_CHUNK_MB");
    return v ? size_t(std::max(1, std::atoi(v))) << 20 : kChunkBytes;
  }();
  const int64_t rows = std::max<int64_t>(1, (int64_t)(chunk_bytes / (sizeof(double) * e->dim)));
  for (int b = 0; b < 2; ++b) {
    RB_CUDA(cudaMallocHost(&e->pin_x[b], sizeof(double) * rows * e->dim));
    RB_CUDA(cudaMallocHost(&e->pin_f[b], sizeof(double) * rows));
    RB_CUDA(cudaMalloc(&e->dev_x[b], sizeof(double) * rows * e->dim));
    RB_CUDA(cudaMalloc(&e->dev_f[b], sizeof(double) * rows));
    RB_CUDA(cudaEventCreateWithFlags(&e->x_ready[b], cudaEventDisableTiming));
    RB_CUDA(cudaEventCreateWithFlags(&e->f_ready[b], cudaEventDisableTiming));
  }
  RB_CUDA(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
  RB_CUDA(cudaStreamCreateWithFlags(&e->d2h_stream, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) RB_CUDA(cudaEventCreateWithFlags(&e->computed[b], cudaEventDisableTiming));
  RB_CUDA(cudaStreamCreateWithFlags(&e->many_stream2, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) RB_CUDA(cudaEventCreateWithFlags(&e->computed2[b], cudaEventDisableTiming));
  RB_CUDA(cudaEventCreateWithFlags(&e->ready2, cudaEventDisableTiming));
  e->chunk_rows = rows;
  return RB_OK;
}

// TI: the caller's element type; T: the evaluation precision
template <class TI, class T>
rb_status evaluate_host_locked(rb_engine* e, int32_t fn_id, const TI* x, int64_t n, T* f) {
  {
    const rb_status st = ensure_pipeline(e);
    if (st != RB_OK) return st;
  }
  const int dim = e->dim;
  const int64_t cap = e->chunk_rows;
  const int64_t nchunks = (n + cap - 1) / cap;
  if (nchunks == 1) {
    // one chunk (every small batch): stage, H2D, launch, D2H on the engine
    // stream and ONE synchronisation; the float64 exact-order pass only when
    // the kernel marked rows (then a second D2H)
    T* px = static_cast<T*>(e->pin_x[0]);
    parallel_rows(n, (int64_t)sizeof(T) * n * dim, [&](int64_t lo, int64_t hi) {
      if constexpr (std::is_same<TI, T>::value) {
        std::memcpy(px + lo * dim, x + lo * dim, sizeof(T) * (hi - lo) * dim);
      } else {
        for (int64_t i = lo * dim; i < hi * dim; ++i) px[i] = static_cast<T>(x[i]);
      }
    });
    RB_CUDA(cudaMemcpyAsync(e->dev_x[0], px, sizeof(T) * n * dim, cudaMemcpyHostToDevice, e->host_stream));
    volatile int* flag = nullptr;
    rb_status st = launch_eval<T>(e, fn_id, static_cast<const T*>(e->dev_x[0]), n,
                                  static_cast<T*>(e->dev_f[0]), e->host_stream, &flag, false);
    if (st != RB_OK) {
      cudaStreamSynchronize(e->host_stream);
      return st;
    }
    RB_CUDA(cudaMemcpyAsync(e->pin_f[0], e->dev_f[0], sizeof(T) * n, cudaMemcpyDeviceToHost, e->host_stream));
    RB_CUDA(cudaStreamSynchronize(e->host_stream));
    if (flag[0]) return non_finite();
    if constexpr (sizeof(T) == 8) {
      if (flag[1]) {
        st = launch_fixup(e, fn_id, static_cast<const double*>(e->dev_x[0]), n,
                          static_cast<double*>(e->dev_f[0]), e->host_stream,
                          const_cast<int*>(e->d_flags + (flag - e->h_flags)));
        if (st != RB_OK) return st;
        RB_CUDA(cudaMemcpyAsync(e->pin_f[0], e->dev_f[0], sizeof(T) * n, cudaMemcpyDeviceToHost,
                                e->host_stream));
        RB_CUDA(cudaStreamSynchronize(e->host_stream));
        if (flag[0]) return non_finite();
      }
    }
    std::memcpy(f, e->pin_f[0], sizeof(T) * n);
    return RB_OK;
  }
  std::vector<volatile int*> flags;
  flags.reserve(nchunks);
  auto drain = [&](int64_t c) -> rb_status {   // chunk c's values into the caller's f
    const int b = (int)(c & 1);
    RB_CUDA(cudaEventSynchronize(e->f_ready[b]));
    const int64_t r0 = c * cap, rows = std::min(cap, n - r0);
    std::memcpy(f + r0, e->pin_f[b], sizeof(T) * rows);
    return RB_OK;
  };
  rb_status st = RB_OK;
  for (int64_t c = 0; c < nchunks && st == RB_OK; ++c) {
    const int b = (int)(c & 1);
    if (c >= 2) {                              // buffers b free: chunk c-2 is done
      st = drain(c - 2);
      if (st != RB_OK) break;
    }
    const int64_t r0 = c * cap, rows = std::min(cap, n - r0);
    T* px = static_cast<T*>(e->pin_x[b]);
    const TI* src = x + r0 * dim;
    parallel_rows(rows, (int64_t)sizeof(T) * rows * dim, [&](int64_t lo, int64_t hi) {
      if constexpr (std::is_same<TI, T>::value) {
        std::memcpy(px + lo * dim, src + lo * dim, sizeof(T) * (hi - lo) * dim);
      } else {
        for (int64_t i = lo * dim; i < hi * dim; ++i) px[i] = static_cast<T>(src[i]);
      }
    });
    if (cudaMemcpyAsync(e->dev_x[b], px, sizeof(T) * rows * dim, cudaMemcpyHostToDevice,
                        e->copy_stream) != cudaSuccess ||
        cudaEventRecord(e->x_ready[b], e->copy_stream) != cudaSuccess ||
        cudaStreamWaitEvent(e->host_stream, e->x_ready[b], 0) != cudaSuccess) {
      st = fail(RB_E_CUDA, "host pipeline: H2D failed");
      break;
    }
    volatile int* flag = nullptr;
    st = launch_eval<T>(e, fn_id, static_cast<const T*>(e->dev_x[b]), rows,
                        static_cast<T*>(e->dev_f[b]), e->host_stream, &flag, true);
    if (st != RB_OK) break;
    flags.push_back(flag);
    if (cudaMemcpyAsync(e->pin_f[b], e->dev_f[b], sizeof(T) * rows, cudaMemcpyDeviceToHost,
                        e->host_stream) != cudaSuccess ||
        cudaEventRecord(e->f_ready[b], e->host_stream) != cudaSuccess)
      st = fail(RB_E_CUDA, "host pipeline: D2H failed");
  }
  if (st == RB_OK)
    for (int64_t c = std::max<int64_t>(0, nchunks - 2); c < nchunks && st == RB_OK; ++c) st = drain(c);
  cudaStreamSynchronize(e->host_stream);
  cudaStreamSynchronize(e->copy_stream);
  if (st != RB_OK) return st;
  for (volatile int* fl : flags)
    if (fl[0]) return non_finite();
  return RB_OK;
}

// Many (function, precision) calls on ONE host population (device current,
// host_mu held): the rows cross PCIe once per chunk, not once per call.
// Per chunk (double-buffered, as evaluate_host_locked): host staging of the
// float64 rows, H2D on the copy stream, then on the engine stream the
// float32 cast (when a call is single precision; engine.py:201), every
// call's kernel (+ the float64 exact-order pass queued behind it) and one
// D2H of all their values; the values of chunk c-2 leave their pinned
// buffer for the callers' arrays meanwhile.
rb_status evaluate_host_many_locked(rb_engine* e, int32_t n_calls, const int32_t* fn_ids,
                                    const int32_t* precisions, const double* x, int64_t n,
                                    void* const* f) {
  {
    const rb_status st = ensure_pipeline(e);
    if (st != RB_OK) return st;
  }
  const int dim = e->dim;
  // chunks of ~128 MB: every chunk launches one kernel per call, so bigger
  // chunks amortise the launches (measured at N = 1e7, 74 calls: 32 MB
  // 343, 64 MB 446, 128 MB 507, 256 MB 548 M evals/s; 128 MB keeps the
  // pinned staging under ~0.5 GB)
  if (!e->many_rows) {
    static const size_t many_bytes = [] {     // RB_MANY_CHUNK_MB (default 128)
      const char* v = std::getenv("RB_MANY_CHUNK_MB");
      return (v ? size_t(std::max(1, std::atoi(v))) : size_t(128)) << 20;
    }();
    const int64_t rows = std::max<int64_t>(1, (int64_t)(many_bytes / (sizeof(double) * dim)));
    for (int b = 0; b < 2; ++b) {
      RB_CUDA(cudaMallocHost(&e->pin_xm[b], sizeof(double) * rows * dim));
      RB_CUDA(cudaMalloc(&e->dev_xm[b], sizeof(double) * rows * dim));
    }
    e->many_rows = rows;
  }
  const int64_t cap = e->many_rows;
  if (n_calls > e->fm_calls) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(e->dev_fm[b]);
      if (e->pin_fm[b]) cudaFreeHost(e->pin_fm[b]);
      e->dev_fm[b] = e->pin_fm[b] = nullptr;
    }
    e->fm_calls = 0;
    for (int b = 0; b < 2; ++b) {
      RB_CUDA(cudaMalloc(&e->dev_fm[b], sizeof(double) * cap * n_calls));
      RB_CUDA(cudaMallocHost(&e->pin_fm[b], sizeof(double) * cap * n_calls));
    }
    e->fm_calls = n_calls;
  }
  bool any32 = false;
  for (int32_t i = 0; i < n_calls; ++i) any32 = any32 || precisions[i] == RB_SINGLE;
  if (any32 && !e->dev_x32) RB_CUDA(cudaMalloc(reinterpret_cast<void**>(&e->dev_x32), sizeof(float) * cap * dim));
  const int64_t nchunks = (n + cap - 1) / cap;
  std::vector<volatile int*> flags;
  flags.reserve((size_t)nchunks * n_calls);
  auto drain = [&](int64_t c) -> rb_status {
    const int b = (int)(c & 1);
    RB_CUDA(cudaEventSynchronize(e->f_ready[b]));
    const int64_t r0 = c * cap, rows = std::min(cap, n - r0);
    const unsigned char* src = static_cast<const unsigned char*>(e->pin_fm[b]);
    parallel_rows(n_calls, (int64_t)sizeof(double) * rows * n_calls, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        const size_t s = precisions[i] == RB_DOUBLE ? sizeof(double) : sizeof(float);
        std::memcpy(static_cast<unsigned char*>(f[i]) + s * r0, src + sizeof(double) * cap * i, s * rows);
      }
    });
    return RB_OK;
  };
  rb_status st = RB_OK;
  for (int64_t c = 0; c < nchunks && st == RB_OK; ++c) {
    const int b = (int)(c & 1);
    if (c >= 2) {
      st = drain(c - 2);
      if (st != RB_OK) break;
    }
    const int64_t r0 = c * cap, rows = std::min(cap, n - r0);
    double* px = static_cast<double*>(e->pin_xm[b]);
    const double* src = x + r0 * dim;
    parallel_rows(rows, (int64_t)sizeof(double) * rows * dim, [&](int64_t lo, int64_t hi) {
      std::memcpy(px + lo * dim, src + lo * dim, sizeof(double) * (hi - lo) * dim);
    });
    if (cudaMemcpyAsync(e->dev_xm[b], px, sizeof(double) * rows * dim, cudaMemcpyHostToDevice,
                        e->copy_stream) != cudaSuccess ||
        cudaEventRecord(e->x_ready[b], e->copy_stream) != cudaSuccess ||
        cudaStreamWaitEvent(e->host_stream, e->x_ready[b], 0) != cudaSuccess) {
      st = fail(RB_E_CUDA, "host pipeline: H2D failed");
      break;
    }
    const double* x64 = static_cast<const double*>(e->dev_xm[b]);
    // dev_x32 is single-buffered: the previous chunk's calls on the second
    // stream read it until they finish
    if (c >= 1 && cudaStreamWaitEvent(e->host_stream, e->computed2[b ^ 1], 0) != cudaSuccess) {
      st = fail(RB_E_CUDA, "host pipeline: event wait failed");
      break;
    }
    if (any32) {
      const int grid = (int)std::min<int64_t>((rows * dim + 255) / 256, 148 * 8);
      rb::cast_rows_kernel<<<grid, 256, 0, e->host_stream>>>(x64, e->dev_x32, rows * dim);
      g_launches.fetch_add(1);
    }
    unsigned char* fb = static_cast<unsigned char*>(e->dev_fm[b]);
    if (c >= 2 && cudaStreamWaitEvent(e->host_stream, e->f_ready[b], 0) != cudaSuccess) {
      st = fail(RB_E_CUDA, "host pipeline: event wait failed");   // dev_fm[b] copied out
      break;
    }
    // the calls alternate between two streams, so one kernel's last wave
    // (a chunk is ~10 waves per launch) overlaps the next kernel's first
    if (cudaEventRecord(e->ready2, e->host_stream) != cudaSuccess ||
        cudaStreamWaitEvent(e->many_stream2, e->ready2, 0) != cudaSuccess) {
      st = fail(RB_E_CUDA, "host pipeline: event wait failed");
      break;
    }
    for (int32_t i = 0; i < n_calls && st == RB_OK; ++i) {
      volatile int* flag = nullptr;
      void* fi = fb + sizeof(double) * cap * i;
      cudaStream_t cs = (i & 1) ? e->many_stream2 : e->host_stream;
      if (precisions[i] == RB_DOUBLE)
        st = launch_eval<double>(e, fn_ids[i], x64, rows, static_cast<double*>(fi), cs, &flag, true);
      else
        st = launch_eval<float>(e, fn_ids[i], e->dev_x32, rows, static_cast<float*>(fi), cs, &flag, true);
      if (st == RB_OK) flags.push_back(flag);
    }
    if (st != RB_OK) break;
    // the values leave on their own stream (PCIe is full duplex), so chunk
    // c+1's kernels start as soon as chunk c's are done
    if (cudaEventRecord(e->computed[b], e->host_stream) != cudaSuccess ||
        cudaEventRecord(e->computed2[b], e->many_stream2) != cudaSuccess ||
        cudaStreamWaitEvent(e->d2h_stream, e->computed[b], 0) != cudaSuccess ||
        cudaStreamWaitEvent(e->d2h_stream, e->computed2[b], 0) != cudaSuccess ||
        cudaMemcpyAsync(e->pin_fm[b], e->dev_fm[b], sizeof(double) * cap * n_calls, cudaMemcpyDeviceToHost,
                        e->d2h_stream) != cudaSuccess ||
        cudaEventRecord(e->f_ready[b], e->d2h_stream) != cudaSuccess)
      st = fail(RB_E_CUDA, "host pipeline: D2H failed");
  }
  if (st == RB_OK)
    for (int64_t c = std::max<int64_t>(0, nchunks - 2); c < nchunks && st == RB_OK; ++c) st = drain(c);
  cudaStreamSynchronize(e->host_stream);
  cudaStreamSynchronize(e->many_stream2);
  cudaStreamSynchronize(e->copy_stream);
  cudaStreamSynchronize(e->d2h_stream);
  if (st != RB_OK) return st;
  for (volatile int* fl : flags)
    if (fl[0]) return non_finite();
  return RB_OK;
}

template <class TI, class T>
rb_status evaluate_host(rb_engine* e, int32_t fn_id, const TI* x, int64_t n, T* f) {
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (n < 1 || n > e->max_concurrency || !x || !f || fn_id < 0 ||
      fn_id >= (int32_t)e->fns.size() || e->fns[fn_id].category == RB_DISABLED)
    return evaluate_device<T>(e, fn_id, reinterpret_cast<const T*>(x), n, f, nullptr);  // the error
  const int pi = sizeof(T) == 8 ? 0 : 1;
  if (!e->why[pi][fn_id].empty())
    return fail(RB_E_UNSUPPORTED, "function " + std::to_string(fn_id) + ": " + e->why[pi][fn_id]);
  std::lock_guard<std::mutex> lock(e->host_mu);
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  RB_CUDA(cudaSetDevice(e->device));
  const rb_status s = evaluate_host_locked<TI, T>(e, fn_id, x, n, f);
  cudaSetDevice(prev);
  return s;
}

// Per-function launch parameters: kernel variant, shared-memory layout.  A
// function that does not fit (shared-memory tile, plan tables, float32
// pairwise stack) is marked unsupported in that precision; the others stay
// usable (the reference has no dimension cap, engine.py:42-44).
rb_status plan_launches(rb_engine* e, const rb_pack* pk, int device) {
  int sms = 0, optin = 0;
  RB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  RB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  int max_d = 1;
  for (int i = 0; i < pk->n_segments; ++i) max_d = std::max(max_d, pk->segments[i].d);
  e->ldz[0] = pad_to(max_d, 16, 8);   // 8 lanes x 4 points read rows: stride 8 (mod 16) doubles
  e->ldz[1] = pad_to(max_d, 32, 8);
  const int nf = pk->n_functions;
  for (int pi = 0; pi < 2; ++pi) {
    e->launch[pi].assign(nf, Launch());
    e->why[pi].assign(nf, std::string());
  }
  e->fixup.assign(nf, 0);
  e->fixup_grid = sms * RB_FIXUP_BLOCKS;
  std::map<const void*, size_t> need;       // dynamic shared memory per kernel
  std::vector<int> variant(nf, rb::N_VARIANTS - 1);
  std::vector<int> spec(nf, -1);            // function-specialised kernel (rb_fnspec.cuh)
  for (int fi = 0; fi < nf; ++fi) {
    const rb_function& fn = pk->functions[fi];
    if (fn.category == RB_DISABLED) continue;
    const rb_member& first = pk->members[fn.member0];
    const rb_member& last = pk->members[fn.member0 + fn.n_members - 1];
    const int s0 = first.segment0, s1 = last.segment0 + last.n_segments;
    const int g0 = pk->segments[s0].group0;
    const int g1 = pk->segments[s1 - 1].group0 + pk->segments[s1 - 1].n_groups;
    if (fn.n_members > rb::MAX_MEMBERS || s1 - s0 > rb::MAX_SEGMENTS || g1 - g0 > rb::MAX_GROUPS) {
      e->why[0][fi] = e->why[1][fi] = "exceeds the plan limits";
      continue;
    }
    int max_q = 0, ldv = 4, units = 0;
    for (int mi = 0; mi < fn.n_members; ++mi) {    // V rows: a member's chunks at once
      const rb_member& mm = pk->members[fn.member0 + mi];
      int q4 = 0;
      bool exact64 = false, deep = false;
      for (int si = mm.segment0; si < mm.segment0 + mm.n_segments; ++si) {
        const rb_segment& sg = pk->segments[si];
        exact64 = exact64 || (rb::exact64_kernel(sg.kernel) && sg.n_groups > 0);
        for (int g = sg.group0; g < sg.group0 + sg.n_groups; ++g) {
          max_q += rb::round8(pk->groups[g].m);
          q4 += (pk->groups[g].m + 3) & ~3;
          units += (rb::TP / 16) * ((pk->groups[g].m + 7) / 8);   // (MT2 kernels: half)
          deep = deep || pk->groups[g].leaf == -2;
        }
      }
      if (deep)
        e->why[1][fi] = "single precision needs rotated segments whose pairwise tree fits the "
                        "device stack (any length <= 968)";
      ldv = std::max(ldv, q4);
      if (exact64 && !deep) e->fixup[fi] |= 1 << mi;   // (deep: float64 keeps the DMMA z)
    }
    const bool many_units = units > rb::MAX_UNITS;   // -> evaluate_big_kernel (on-the-fly units)
    if (fn.category == RB_BASIC && fn.n_members == 1 && first.n_segments == 1)
      variant[fi] = pk->segments[s0].kernel;
    if (fi >= rb::FN_FIRST_SPEC && fi < rb::FN_FIRST_SPEC + rb::FN_COUNT_SPEC) {
      // the pack's jobs must be exactly the compiled catalog's
      const rb::JobList jl = rb::job_list(fi);
      bool match = jl.n == s1 - s0;
      for (int mi = 0, j = 0; match && mi < fn.n_members; ++mi) {
        const rb_member& mm = pk->members[fn.member0 + mi];
        for (int si = 0; si < mm.n_segments; ++si, ++j)
          match = match && j < jl.n && jl.member[j] == mi &&
                  jl.kernel[j] == pk->segments[mm.segment0 + si].kernel &&
                  pk->segments[mm.segment0 + si].n_groups > 0;
      }
      if (match && spec_mode()) spec[fi] = fi - rb::FN_FIRST_SPEC;
    }
    for (int pi = 0; pi < 2; ++pi) {
      Launch& L = e->launch[pi][fi];
      L.func = (pi == 0 ? rb::kernels_f64 : rb::kernels_f32)[variant[fi]];
      if (spec[fi] >= 0) L.func = (pi == 0 ? rb::kernels_spec_f64 : rb::kernels_spec_f32)[spec[fi]];
      // must match rb::mt2_kernel<KID>() of the kernel chosen
      L.mt2 = pi == 0 && (spec[fi] >= 0 ? fi < 29 : variant[fi] < rb::K_COUNT);
      L.max_q = std::max(max_q, 1);
      L.ldv = pi == 0 ? 0 : ldv;             // float64 has no V tile
      L.opt_rows = fn.category == RB_COMPOSITION ? fn.n_members : 0;
      for (int nb = 1; nb <= 2; ++nb)
        L.smem_nbuf[nb] = pi == 0 ? rb::smem_bytes<double>(pk->dim, L.ldv, e->ldz[0], L.max_q, nb, L.opt_rows)
                                  : rb::smem_bytes<float>(pk->dim, L.ldv, e->ldz[1], L.max_q, nb, L.opt_rows);
      if ((int)L.smem_nbuf[1] > optin || (pi == 0 && many_units) || big_mode() == 1) {
        // the tile does not fit: PlanHead in shared memory, the rest in a
        // per-CTA slice of global scratch (evaluate_big_kernel)
        L.big = true;
        L.mt2 = false;
        L.nbuf = 1;
        L.func = pi == 0 ? rb::big_f64 : rb::big_f32;
        L.smem = rb::align16(sizeof(rb::PlanHead));
        L.per_cta = L.smem_nbuf[1] - L.smem;
        need[L.func] = std::max(need[L.func], L.smem);
        continue;
      }
      const size_t top = (int)L.smem_nbuf[2] <= optin ? L.smem_nbuf[2] : L.smem_nbuf[1];
      need[L.func] = std::max(need[L.func], top);
      if (pi == 0 && e->fixup[fi]) need[rb::fixup_f64] = std::max(need[rb::fixup_f64], L.smem_nbuf[1]);
    }
  }
  {
    std::lock_guard<std::mutex> lock(g_attr_mu);
    for (const auto& kv : need) {
      size_t& have = g_attr[std::make_pair(device, kv.first)];
      if (kv.second <= have) continue;
      RB_CUDA(cudaFuncSetAttribute(kv.first, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kv.second));
      have = kv.second;
    }
  }
  for (int fi = 0; fi < nf; ++fi) {
    if (pk->functions[fi].category == RB_DISABLED) continue;
    for (int pi = 0; pi < 2; ++pi) {
      Launch& L = e->launch[pi][fi];
      if (!L.func) continue;
      int occ[3] = {0, 0, 0};
      if (L.big) {
        RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], L.func, rb::NT, L.smem));
        if (occ[1] < 1) {
          e->why[pi][fi] = "kernel does not fit on an SM";
          continue;
        }
        L.grid_cap = sms * std::min(occ[1], 2);     // bounds the scratch (per_cta each)
        continue;
      }
      for (int nb = 1; nb <= 2; ++nb)
        if ((int)L.smem_nbuf[nb] <= optin)
          RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[nb], L.func, rb::NT,
                                                                L.smem_nbuf[nb]));
      if (occ[1] < 1) {
        e->why[pi][fi] = "kernel does not fit on an SM";
        continue;
      }
      const int mode = prefetch_mode();
      L.nbuf = (mode == 1 && occ[2] >= 1) || (mode < 0 && occ[2] >= occ[1]) ? 2 : 1;
      if (pi == 0) L.nbuf = 1;           // fp64 tiles have no second X buffer
      L.smem = L.smem_nbuf[L.nbuf];
      L.grid_cap = sms * occ[L.nbuf];
    }
  }
  return RB_OK;
}

// Every offset of a pack (a public C ABI: hosts other than pack.py may build
// one) is checked with its extent against the tables before anything reads
// through it on the host or the device.
int64_t ctab_len(int kernel, int d) {
  switch (kernel) {
    case rb::K_ELLIPTIC: case rb::K_POWERS: case rb::K_GRIEWANK: return d;
    case rb::K_WEIERSTRASS: return 43;
    case rb::K_KATSUURA: return 2;
    default: return 0;
  }
}

rb_status validate_pack(const rb_pack* pk) {
  const int64_t nv = pk->n_values, ni = pk->n_index;
  auto in_values = [&](int64_t off, int64_t len) { return len == 0 || (off >= 0 && off + len <= nv); };
  auto in_index = [&](int64_t off, int64_t len) { return len == 0 || (off >= 0 && off + len <= ni); };
  auto bad = [](const char* what, int i) {
    return fail(RB_E_INVALID_ARGUMENT, std::string(what) + " " + std::to_string(i) + " out of range");
  };
  if (pk->n_functions > 4096 || pk->n_members < 0 || pk->n_segments < 0 || pk->n_groups < 0 ||
      nv < 0 || ni < 0 || (nv > 0 && (!pk->values_f64 || !pk->values_f32)) || (ni > 0 && !pk->index) ||
      !pk->functions || (pk->n_members > 0 && !pk->members) ||
      (pk->n_segments > 0 && !pk->segments) || (pk->n_groups > 0 && !pk->groups))
    return fail(RB_E_INVALID_ARGUMENT, "malformed pack header");
  const int dim = pk->dim;
  for (int i = 0; i < pk->n_functions; ++i) {
    const rb_function& f = pk->functions[i];
    if (f.category == RB_DISABLED) continue;
    if (f.category < RB_BASIC || f.category > RB_COMPOSITION || f.n_members < 1 || f.member0 < 0 ||
        (int64_t)f.member0 + f.n_members > pk->n_members)
      return bad("function", i);
  }
  for (int i = 0; i < pk->n_members; ++i) {
    const rb_member& m = pk->members[i];
    if (m.n_segments < 1 || m.segment0 < 0 || (int64_t)m.segment0 + m.n_segments > pk->n_segments ||
        !in_values(m.shift, dim) || (m.perm != -1 && !in_index(m.perm, dim)))
      return bad("member", i);
    if (m.perm != -1)
      for (int j = 0; j < dim; ++j)
        if (pk->index[m.perm + j] < 0 || pk->index[m.perm + j] >= dim) return bad("member", i);
    int64_t covered = 0;
    for (int si = m.segment0; si < m.segment0 + m.n_segments; ++si) {
      const rb_segment& sg = pk->segments[si];
      if (sg.src < 0 || sg.d < 1 || (int64_t)sg.src + sg.d > dim) return bad("segment", si);
      covered += sg.d;
    }
    if (covered > dim) return bad("member", i);
  }
  for (int i = 0; i < pk->n_segments; ++i) {
    const rb_segment& s = pk->segments[i];
    if (s.kernel < 0 || s.kernel >= rb::K_COUNT || s.d < 1 || s.d > dim || s.n_groups < 0 ||
        s.group0 < 0 || (int64_t)s.group0 + s.n_groups > pk->n_groups ||
        !in_values(s.ctab, ctab_len(s.kernel, s.d)))
      return bad("segment", i);
    int64_t rows = 0;
    for (int g = s.group0; g < s.group0 + s.n_groups; ++g) {
      const rb_group& G = pk->groups[g];
      const int m = G.m;
      if (m < 1 || m > s.d) return bad("group", g);
      const int64_t m4 = (m + 3) & ~3, nt = (m + 7) / 8, nk = (m + 3) / 4;
      if (!in_index(G.col, m) || !in_index(G.row, m) || !in_index(G.col64, m) ||
          !in_values(G.mat, (int64_t)m * m4) || !in_values(G.frag, nt * nk * 32) || !in_values(G.cz, m))
        return bad("group", g);
      for (int q = 0; q < m; ++q)
        if (pk->index[G.col + q] < 0 || pk->index[G.col + q] >= s.d || pk->index[G.row + q] < 0 ||
            pk->index[G.row + q] >= s.d || pk->index[G.col64 + q] < 0 || pk->index[G.col64 + q] >= s.d)
          return bad("group", g);
      auto qb_ok = [m](const int32_t* qb) {
        for (int k = 0; k < 10; ++k)
          if (qb[k] < 0 || qb[k] > m || (k && qb[k] < qb[k - 1])) return false;
        return true;
      };
      if (G.leaf == -1) {
        if (!qb_ok(G.qb) || G.qb[9] != m) return bad("group", g);
      } else if (G.leaf != -2) {
        if (!in_index(G.leaf, 1)) return bad("group", g);
        const int64_t nl = pk->index[G.leaf];
        if (nl < 1 || nl > 64 || !in_index(G.leaf, 1 + 11 * nl)) return bad("group", g);
        for (int64_t l = 0; l < nl; ++l)
          if (!qb_ok(pk->index + G.leaf + 1 + 11 * l)) return bad("group", g);
      }
      rows += m;
    }
    if (rows > s.d) return bad("segment", i);
  }
  return RB_OK;
}

// Weierstrass series constants (a_k, c_k; pack.py kernel_constants) into
// the kernels' __constant__ tables.  They depend on the dtype only, so every
// Weierstrass segment of the pack must carry the same 42 values.
rb_status upload_series_constants(const rb_pack* pk) {
  int found = -1;
  for (int i = 0; i < pk->n_segments; ++i) {
    const rb_segment& s = pk->segments[i];
    if (s.kernel != rb::K_WEIERSTRASS) continue;
    if (s.ctab < 0 || (int64_t)s.ctab + 43 > pk->n_values)
      return fail(RB_E_INVALID_ARGUMENT, "segment " + std::to_string(i) + ": constant table out of range");
    if (found < 0) {
      found = s.ctab;
      continue;
    }
    for (int k = 0; k < 42; ++k)
      if (pk->values_f64[s.ctab + k] != pk->values_f64[found + k] ||
          pk->values_f32[s.ctab + k] != pk->values_f32[found + k])
        return fail(RB_E_INVALID_ARGUMENT, "Weierstrass constant tables differ between segments");
  }
  if (found < 0) return RB_OK;
  RB_CUDA(rb::set_weier_f64(pk->values_f64 + found));
  RB_CUDA(rb::set_weier_f32(pk->values_f32 + found));
  RB_CUDA(rb::set_weier_f64x(pk->values_f64 + found));
  RB_CUDA(rb::set_weier_f32x(pk->values_f32 + found));
  return RB_OK;
}

// Per precision: the function records (the device copy's `reserved` word
// carries the float64 exact-order members in bits 0-7 and the plan image's
// offset in bits 8+, 16-byte units) followed by one plan image per usable
// function, built on the device by plan_image_kernel with the very Args the
// evaluation launches use (rb_device.cuh enter_plan).
template <class T>
size_t plan_bytes_host(int dim, int max_q, int opt_rows) {
  size_t b = rb::align16(sizeof(rb::PlanHead));
  b += 2 * rb::align16(sizeof(int) * max_q) + rb::align16(sizeof(T) * max_q);
  if (sizeof(T) == 8) b += rb::align16(sizeof(T) * max_q);
  b += rb::align16(sizeof(T) * opt_rows * dim);
  return b;
}

rb_status build_function_tables(rb_engine* e, const rb_pack* pk) {
  const int nf = pk->n_functions;
  static const bool images = [] {
    const char* v = std::getenv("RB_PLAN_IMAGE");
    return !v || std::atoi(v) != 0;
  }();
  for (int pi = 0; pi < 2; ++pi) {
    std::vector<rb_function> fns(pk->functions, pk->functions + nf);
    std::vector<size_t> off(nf, 0), bytes(nf, 0);
    size_t total = (sizeof(rb_function) * nf + 127) & ~size_t(127);
    for (int fi = 0; fi < nf; ++fi) {
      fns[fi].reserved = pi == 0 ? (e->fixup[fi] & 0xff) : 0;
      const Launch& L = e->launch[pi][fi];
      if (!images || fns[fi].category == RB_DISABLED || !L.func || L.big || !e->why[pi][fi].empty())
        continue;
      bytes[fi] = pi == 0 ? plan_bytes_host<double>(pk->dim, L.max_q, L.opt_rows)
                          : plan_bytes_host<float>(pk->dim, L.max_q, L.opt_rows);
      off[fi] = total;
      total += (bytes[fi] + 127) & ~size_t(127);
    }
    if ((total >> 4) >= (size_t(1) << 23)) return fail(RB_E_UNSUPPORTED, "plan images too large");
    rb_function** dst = pi == 0 ? &e->d_fns : &e->d_fns32;
    RB_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), total));
    // records without images first: the image kernel reads them
    RB_CUDA(cudaMemcpy(*dst, fns.data(), sizeof(rb_function) * nf, cudaMemcpyHostToDevice));
    for (int fi = 0; fi < nf; ++fi) {
      if (!bytes[fi]) continue;
      const Launch& L = e->launch[pi][fi];
      uint4* out = reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(*dst) + off[fi]);
      const void* kern = pi == 0 ? rb::plan_image_f64[L.mt2 ? 1 : 0] : rb::plan_image_f32;
      {                                      // only ever raised (engines coexist)
        std::lock_guard<std::mutex> lock(g_attr_mu);
        size_t& have = g_attr[std::make_pair(e->device, kern)];
        if (bytes[fi] > have) {
          RB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes[fi]));
          have = bytes[fi];
        }
      }
      if (pi == 0) {
        rb::Args<double> a = make_args<double>(e, fi, nullptr, 0, nullptr, nullptr, L);
        void* args[] = {&a, &out};
        RB_CUDA(cudaLaunchKernel(kern, dim3(1), dim3(rb::NT), args, bytes[fi], 0));
      } else {
        rb::Args<float> a = make_args<float>(e, fi, nullptr, 0, nullptr, nullptr, L);
        void* args[] = {&a, &out};
        RB_CUDA(cudaLaunchKernel(kern, dim3(1), dim3(rb::NT), args, bytes[fi], 0));
      }
      fns[fi].reserved |= (int32_t)((off[fi] >> 4) << 8);
    }
    RB_CUDA(cudaDeviceSynchronize());
    RB_CUDA(cudaMemcpy(*dst, fns.data(), sizeof(rb_function) * nf, cudaMemcpyHostToDevice));
  }
  return RB_OK;
}

// Stream-ordered call: validation now, the status later (rb_ticket_status).
// float64 functions with exact64 members queue their fixup pass behind the
// kernel, since nobody inspects the flags in between.
template <class T>
rb_status evaluate_async(rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f,
                         cudaStream_t stream, int64_t* ticket) {
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  if (prev != e->device) RB_CUDA(cudaSetDevice(e->device));
  volatile int* flag = nullptr;
  uint32_t seq = 0;
  const rb_status s = launch_eval<T>(e, fn_id, x, n, f, stream, &flag, true, &seq);
  if (s == RB_OK && ticket) *ticket = (int64_t)seq;
  if (prev != e->device) cudaSetDevice(prev);
  return s;
}

rb_status ticket_status(rb_engine* e, int64_t ticket) {
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (ticket < 0) return fail(RB_E_INVALID_ARGUMENT, "bad ticket");
  const uint32_t seq = (uint32_t)ticket;
  const volatile int* hf = e->h_flags + kSlotInts * (seq & (kFlagSlots - 1));
  if ((uint32_t)hf[2] != seq)
    return fail(RB_E_INVALID_ARGUMENT, "ticket expired: more than 4096 calls issued since");
  return hf[0] ? non_finite() : RB_OK;
}

template <class T>
rb_status evaluate_sharded(rb_sharded* sh, int32_t fn_id, const void* const* x_shards, int64_t n_total,
                           void* const* f_full, void* const* streams, int64_t* tickets) {
  const int G = (int)sh->eng.size();
  if (n_total < 1 || !x_shards || !f_full) return fail(RB_E_INVALID_ARGUMENT, "empty batch or null pointer");
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  const int64_t base = n_total / G, extra = n_total % G;
  std::vector<int64_t> start(G + 1, 0);
  for (int g = 0; g < G; ++g) start[g + 1] = start[g] + base + (g < extra ? 1 : 0);
  std::vector<volatile int*> flags(G, nullptr);
  rb_status st = RB_OK;
  for (int g = 0; g < G && st == RB_OK; ++g) {
    const int64_t cnt = start[g + 1] - start[g];
    if (tickets) tickets[g] = -1;
    if (cnt == 0) continue;                  // fewer rows than devices
    cudaStream_t stream = streams ? static_cast<cudaStream_t>(streams[g]) : sh->streams[g];
    if (cudaSetDevice(sh->dev[g]) != cudaSuccess) {
      st = fail(RB_E_CUDA, "cudaSetDevice failed");
      break;
    }
    T* fg = static_cast<T*>(f_full[g]) + start[g];
    uint32_t seq = 0;
    st = launch_eval<T>(sh->eng[g], fn_id, static_cast<const T*>(x_shards[g]), cnt, fg, stream,
                        &flags[g], true, &seq);
    if (st != RB_OK) break;
    if (tickets) tickets[g] = (int64_t)seq;
    if (G == 1) continue;
    if (sh->p2p) {                           // this slice into every peer's f, over NVLink
      rb::PeerDst dst{};
      for (int h = 0; h < G; ++h)
        if (h != g) dst.p[dst.n++] = static_cast<T*>(f_full[h]) + start[g];
      const int grid = (int)std::min<int64_t>((cnt + 255) / 256, 148 * 4);
      rb::peer_scatter_kernel<T><<<grid, 256, 0, stream>>>(fg, cnt, dst);
      g_launches.fetch_add(1);
      const cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) st = fail(RB_E_CUDA, std::string("peer_scatter: ") + cudaGetErrorString(err));
    } else {                                 // no peer access: copy-engine copies
      for (int h = 0; h < G && st == RB_OK; ++h) {
        if (h == g) continue;
        const cudaError_t err = cudaMemcpyPeerAsync(static_cast<T*>(f_full[h]) + start[g], sh->dev[h], fg,
                                                    sh->dev[g], sizeof(T) * cnt, stream);
        if (err != cudaSuccess) st = fail(RB_E_CUDA, std::string("cudaMemcpyPeerAsync: ") + cudaGetErrorString(err));
      }
    }
  }
  if (st == RB_OK && !tickets) {             // synchronous: wait, then the reference's errors
    for (int g = 0; g < G; ++g) {
      if (!flags[g]) continue;
      cudaStream_t stream = streams ? static_cast<cudaStream_t>(streams[g]) : sh->streams[g];
      cudaSetDevice(sh->dev[g]);
      const cudaError_t err = cudaStreamSynchronize(stream);
      if (err != cudaSuccess && st == RB_OK)
        st = fail(RB_E_CUDA, std::string("cudaStreamSynchronize: ") + cudaGetErrorString(err));
    }
    for (int g = 0; g < G && st == RB_OK; ++g)
      if (flags[g] && flags[g][0]) st = non_finite();
  }
  cudaSetDevice(prev);
  return st;
}

// ------------------------------------------------------------ CUDA graphs
// One evaluation (fixed function, precision, device pointers, row count)
// captured once and replayed: a replay is one cudaGraphLaunch instead of
// validation + flag bookkeeping + one or two kernel launches, for callers
// that evaluate the same buffers many times (optimizer loops over small
// populations, BASELINE config 1).  The graph owns its flag words (mapped
// host memory, reset by a memset node at the start of every replay) and its
// device mark word, so replays never touch the engine's call ring.
struct rb_graph_t {
  rb_engine* e = nullptr;
  int device = 0;
  int* h_flag = nullptr;            // [0] non-finite, [1] rows left for fixup, [2] call number (0)
  int* d_flag = nullptr;
  int* d_mark = nullptr;
  unsigned char* scratch = nullptr; // large-dimension kernel tiles
  cudaGraphExec_t exec = nullptr;
};

void release_graph(rb_graph_t* g) {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  cudaFree(g->d_mark);
  cudaFree(g->scratch);
  if (g->h_flag) cudaFreeHost(g->h_flag);
  cudaSetDevice(prev);
  delete g;
}

template <class T>
rb_status capture_graph(rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f, rb_graph_t** out) {
  const rb_status vs = check_call<T>(e, fn_id, x, n, f);
  if (vs != RB_OK) return vs;
  const int pi = sizeof(T) == 8 ? 0 : 1;
  const Launch& L = e->launch[pi][fn_id];
  rb_graph_t* g = new rb_graph_t();
  g->e = e;
  g->device = e->device;
  cudaStream_t cs = nullptr;
  cudaGraph_t graph = nullptr;
  rb_status st = RB_OK;
  auto cuda = [&](cudaError_t err, const char* what) {
    if (err != cudaSuccess && st == RB_OK)
      st = fail(RB_E_CUDA, std::string("graph capture: ") + what + ": " + cudaGetErrorString(err));
    return st == RB_OK;
  };
  const int64_t ntiles = (n + rb::TP - 1) / rb::TP;
  const int grid = (int)std::min<int64_t>(ntiles, L.grid_cap);
  if (cuda(cudaHostAlloc(reinterpret_cast<void**>(&g->h_flag), kSlotInts * sizeof(int),
                         cudaHostAllocMapped | cudaHostAllocPortable), "flag") &&
      cuda(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g->d_flag), g->h_flag, 0), "flag pointer") &&
      cuda(cudaMalloc(reinterpret_cast<void**>(&g->d_mark), sizeof(int)), "mark") &&
      (!L.big || cuda(cudaMalloc(reinterpret_cast<void**>(&g->scratch), L.per_cta * grid), "scratch")) &&
      cuda(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream") &&
      cuda(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin")) {
    std::memset(g->h_flag, 0, kSlotInts * sizeof(int));
    rb::Args<T> a = make_args<T>(e, fn_id, x, n, f, nullptr, L);
    a.flag = g->d_flag;
    a.mark = g->d_mark;
    cuda(cudaMemsetAsync(g->d_flag, 0, kSlotInts * sizeof(int), cs), "flag reset");
    const bool fixup = sizeof(T) == 8 && e->fixup[fn_id] && !L.big;
    if (fixup) cuda(cudaMemsetAsync(g->d_mark, 0, sizeof(int), cs), "mark reset");
    if (L.big) {
      size_t per_cta = L.per_cta;
      void* args[] = {&a, &g->scratch, &per_cta};
      cuda(cudaLaunchKernel(L.func, dim3(grid), dim3(rb::NT), args, L.smem, cs), "kernel");
    } else {
      void* args[] = {&a};
      cuda(cudaLaunchKernel(L.func, dim3(grid), dim3(rb::NT), args, L.smem, cs), "kernel");
      if (fixup) {
        rb::Args<T> b = a;
        b.nbuf = 1;
        const int fgrid = (int)std::min<int64_t>(ntiles, e->fixup_grid);
        void* fargs[] = {&b};
        cuda(cudaLaunchKernel(rb::fixup_f64, dim3(fgrid), dim3(rb::NT), fargs, L.smem_nbuf[1], cs), "fixup");
      }
    }
    const cudaError_t end = cudaStreamEndCapture(cs, &graph);
    cuda(end, "end");
    if (st == RB_OK) cuda(cudaGraphInstantiate(&g->exec, graph, 0), "instantiate");
  }
  if (graph) cudaGraphDestroy(graph);
  if (cs) cudaStreamDestroy(cs);
  if (st != RB_OK) {
    release_graph(g);
    return st;
  }
  *out = g;
  return RB_OK;
}

}  // namespace

extern "C" {

int32_t rb_abi_version(void) { return 1; }

const char* rb_last_error(void) { return g_last_error.c_str(); }

int64_t rb_launch_count(void) { return g_launches.load(); }

/* Diagnostics (not part of the reference interface): per-phase clock sums
 * of the evaluation kernels of one precision (0 = float64, 1 = float32):
 * [load, stage, kernel, tile, tiles] summed over CTAs; zeros unless the
 * library was built with -DRB_PHASE_TIMING (tools/phase_timing.py). */
void rb_debug_phases(int32_t precision, uint64_t out[8], int32_t reset) {
  unsigned long long v[8], w[8];
  if (precision == 0) {
    rb::phase_read_f64(v, reset != 0);
    rb::phase_read_f64x(w, reset != 0);
  } else {
    rb::phase_read_f32(v, reset != 0);
    rb::phase_read_f32x(w, reset != 0);
  }
  for (int i = 0; i < 8; ++i) out[i] = v[i] + w[i];
}

void rb_struct_sizes(int64_t out[5]) {
  out[0] = sizeof(rb_group);
  out[1] = sizeof(rb_segment);
  out[2] = sizeof(rb_member);
  out[3] = sizeof(rb_function);
  out[4] = sizeof(rb_pack);
}

rb_status rb_initialize(const rb_pack* pk, int64_t max_concurrency, int32_t device,
                        rb_engine** out) {
  NvtxRange range("rb_initialize");
  if (!pk || !out) return fail(RB_E_INVALID_ARGUMENT, "null pack or output pointer");
  *out = nullptr;
  if (pk->dim < 2 || pk->n_functions <= 0 || max_concurrency < 1)
    return fail(RB_E_INVALID_ARGUMENT, "malformed pack");
  {
    const rb_status vs = validate_pack(pk);
    if (vs != RB_OK) return vs;
  }
  int ndev = 0;
  RB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return fail(RB_E_INVALID_ARGUMENT, "device " + std::to_string(device) + " not present");
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  RB_CUDA(cudaSetDevice(device));

  rb_engine* e = new rb_engine();
  e->device = device;
  e->dim = pk->dim;
  e->max_concurrency = max_concurrency;
  e->fns.assign(pk->functions, pk->functions + pk->n_functions);
  rb_status s = plan_launches(e, pk, device);
  if (s == RB_OK) s = upload_series_constants(pk);
  if (s == RB_OK) s = upload(&e->d_members, pk->members, pk->n_members);
  if (s == RB_OK) s = upload(&e->d_segments, pk->segments, pk->n_segments);
  if (s == RB_OK) s = upload(&e->d_groups, pk->groups, pk->n_groups);
  if (s == RB_OK) s = upload(&e->d_index, pk->index, pk->n_index);
  if (s == RB_OK) s = upload(&e->d_v64, pk->values_f64, pk->n_values);
  if (s == RB_OK) s = upload(&e->d_v32, pk->values_f32, pk->n_values);
  if (s == RB_OK) s = build_function_tables(e, pk);
  if (s == RB_OK && cudaHostAlloc(reinterpret_cast<void**>(&e->h_flags), kSlotInts * sizeof(int) * kFlagSlots,
                                   cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    s = fail(RB_E_CUDA, "mapped flag allocation failed");
  if (s == RB_OK && cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->d_flags), e->h_flags, 0) !=
                        cudaSuccess)
    s = fail(RB_E_CUDA, "mapped flag pointer failed");
  if (s == RB_OK && (cudaMalloc(reinterpret_cast<void**>(&e->d_marks), sizeof(int) * kFlagSlots) != cudaSuccess ||
                     cudaMemset(e->d_marks, 0, sizeof(int) * kFlagSlots) != cudaSuccess))
    s = fail(RB_E_CUDA, "mark words allocation failed");
  if (s == RB_OK && cudaStreamCreateWithFlags(&e->host_stream, cudaStreamNonBlocking) != cudaSuccess)
    s = fail(RB_E_CUDA, "stream creation failed");
  cudaSetDevice(prev);
  if (s != RB_OK) {
    release(e);
    return s;
  }
  *out = e;
  return RB_OK;
}

rb_status rb_dispose(rb_engine** engine) {
  if (!engine || !*engine) return RB_OK;
  release(*engine);
  *engine = nullptr;
  return RB_OK;
}

rb_status rb_func_evaluate(rb_engine* e, int32_t fn_id, const double* x, int64_t n, double* f,
                           void* stream) {
  NvtxRange range("rb_func_evaluate");
  return evaluate_device<double>(e, fn_id, x, n, f, static_cast<cudaStream_t>(stream));
}

rb_status rb_func_evaluatef(rb_engine* e, int32_t fn_id, const float* x, int64_t n, float* f,
                            void* stream) {
  NvtxRange range("rb_func_evaluatef");
  return evaluate_device<float>(e, fn_id, x, n, f, static_cast<cudaStream_t>(stream));
}

rb_status rb_h_func_evaluate(rb_engine* e, int32_t fn_id, const double* x, int64_t n, double* f) {
  NvtxRange range("rb_h_func_evaluate");
  return evaluate_host<double, double>(e, fn_id, x, n, f);
}

rb_status rb_h_func_evaluatef(rb_engine* e, int32_t fn_id, const float* x, int64_t n, float* f) {
  NvtxRange range("rb_h_func_evaluatef");
  return evaluate_host<float, float>(e, fn_id, x, n, f);
}

rb_status rb_h_func_evaluate_x64(rb_engine* e, int32_t fn_id, int32_t precision, const double* x,
                                 int64_t n, void* f) {
  NvtxRange range("rb_h_func_evaluate_x64");
  if (precision == RB_DOUBLE) return evaluate_host<double, double>(e, fn_id, x, n, static_cast<double*>(f));
  if (precision == RB_SINGLE) return evaluate_host<double, float>(e, fn_id, x, n, static_cast<float*>(f));
  return fail(RB_E_INVALID_ARGUMENT, "precision must be RB_DOUBLE or RB_SINGLE");
}

rb_status rb_func_evaluate_async(rb_engine* e, int32_t fn_id, int32_t precision, const void* x,
                                 int64_t n, void* f, void* stream, int64_t* ticket) {
  NvtxRange range("rb_func_evaluate_async");
  if (precision == RB_DOUBLE)
    return evaluate_async<double>(e, fn_id, static_cast<const double*>(x), n, static_cast<double*>(f),
                                  static_cast<cudaStream_t>(stream), ticket);
  if (precision == RB_SINGLE)
    return evaluate_async<float>(e, fn_id, static_cast<const float*>(x), n, static_cast<float*>(f),
                                 static_cast<cudaStream_t>(stream), ticket);
  return fail(RB_E_INVALID_ARGUMENT, "precision must be RB_DOUBLE or RB_SINGLE");
}

rb_status rb_ticket_status(rb_engine* e, int64_t ticket) { return ticket_status(e, ticket); }

// True when no call's output overlaps another call's output or any call's
// input: then the calls may run concurrently (rb_func_evaluate_many).
static bool outputs_disjoint(rb_engine* e, int32_t k, const int32_t* precisions, const void* const* x,
                      const int64_t* n, void* const* f) {
  std::vector<std::pair<uintptr_t, uintptr_t>> outs, ins;
  for (int32_t i = 0; i < k; ++i) {
    const size_t el = precisions[i] == RB_DOUBLE ? sizeof(double) : sizeof(float);
    if (n[i] < 1) return false;
    const uintptr_t fo = reinterpret_cast<uintptr_t>(f[i]), xo = reinterpret_cast<uintptr_t>(x[i]);
    outs.emplace_back(fo, fo + el * (size_t)n[i]);
    ins.emplace_back(xo, xo + el * (size_t)n[i] * (size_t)e->dim);
  }
  std::sort(outs.begin(), outs.end());
  for (size_t i = 1; i < outs.size(); ++i)
    if (outs[i].first < outs[i - 1].second) return false;
  for (const auto& in : ins) {      // the first output ending after `in` starts must start after it ends
    auto it = std::lower_bound(outs.begin(), outs.end(), in,
                               [](const std::pair<uintptr_t, uintptr_t>& o,
                                  const std::pair<uintptr_t, uintptr_t>& v) { return o.second <= v.first; });
    if (it != outs.end() && it->first < in.second) return false;
  }
  return true;
}

rb_status rb_func_evaluate_many(rb_engine* e, int32_t n_calls, const int32_t* fn_ids,
                                const int32_t* precisions, const void* const* x, const int64_t* n,
                                void* const* f, void* stream, int64_t* tickets) {
  NvtxRange range("rb_func_evaluate_many");
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (n_calls < 0 || (n_calls > 0 && (!fn_ids || !precisions || !x || !n || !f)))
    return fail(RB_E_INVALID_ARGUMENT, "bad arguments");
  if (n_calls > (int32_t)kFlagSlots) return fail(RB_E_INVALID_ARGUMENT, "more than 4096 calls");
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  if (prev != e->device) RB_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rb_status s = RB_OK;
  // calls with disjoint outputs alternate between the caller's stream and
  // an engine-owned one (forked from and joined back to the caller's), so a
  // short kernel's launch latency and any kernel's last partial wave
  // overlap the next call; stream order as seen by the caller is unchanged
  // (only for short calls: at many waves per launch two co-running
  // kernels cost more than the tails they hide -- measured at N = 1e7,
  // D = 100: -6 %; RB_FORK_WAVES sets the limit, 0 disables)
  static const int64_t fork_waves = [] {
    const char* v = std::getenv("RB_FORK_WAVES");
    return v ? (int64_t)std::atoll(v) : int64_t(128);
  }();
  bool fork = n_calls >= 2 && fork_waves > 0;
  for (int32_t i = 0; fork && i < n_calls; ++i) {
    fork = precisions[i] == RB_DOUBLE || precisions[i] == RB_SINGLE;
    if (fork && fn_ids[i] >= 0 && fn_ids[i] < (int32_t)e->fns.size()) {
      const Launch& L = e->launch[precisions[i] == RB_DOUBLE ? 0 : 1][fn_ids[i]];
      fork = L.grid_cap > 0 && (n[i] + rb::TP - 1) / rb::TP <= fork_waves * L.grid_cap;
    }
  }
  fork = fork && outputs_disjoint(e, n_calls, precisions, x, n, f);
  std::unique_lock<std::mutex> lk(e->fork_mu, std::defer_lock);
  if (fork) {
    lk.lock();
    if (!e->fork_stream) {
      RB_CUDA(cudaStreamCreateWithFlags(&e->fork_stream, cudaStreamNonBlocking));
      RB_CUDA(cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming));
      RB_CUDA(cudaEventCreateWithFlags(&e->join_ev, cudaEventDisableTiming));
    }
    RB_CUDA(cudaEventRecord(e->fork_ev, st));
    RB_CUDA(cudaStreamWaitEvent(e->fork_stream, e->fork_ev, 0));
  }
  for (int32_t i = 0; i < n_calls && s == RB_OK; ++i) {
    volatile int* flag = nullptr;
    uint32_t seq = 0;
    cudaStream_t cs = (fork && (i & 1)) ? e->fork_stream : st;
    if (precisions[i] == RB_DOUBLE)
      s = launch_eval<double>(e, fn_ids[i], static_cast<const double*>(x[i]), n[i],
                              static_cast<double*>(f[i]), cs, &flag, true, &seq);
    else if (precisions[i] == RB_SINGLE)
      s = launch_eval<float>(e, fn_ids[i], static_cast<const float*>(x[i]), n[i],
                             static_cast<float*>(f[i]), cs, &flag, true, &seq);
    else
      s = fail(RB_E_INVALID_ARGUMENT, "precision must be RB_DOUBLE or RB_SINGLE");
    if (tickets) tickets[i] = s == RB_OK ? (int64_t)seq : -1;
  }
  if (fork) {                       // join (also after a failed call: what was queued completes)
    if (cudaEventRecord(e->join_ev, e->fork_stream) != cudaSuccess ||
        cudaStreamWaitEvent(st, e->join_ev, 0) != cudaSuccess)
      if (s == RB_OK) s = fail(RB_E_CUDA, "fork stream join failed");
  }
  if (prev != e->device) cudaSetDevice(prev);
  return s;
}

rb_status rb_h_func_evaluate_many(rb_engine* e, int32_t n_calls, const int32_t* fn_ids,
                                  const int32_t* precisions, const double* x, int64_t n,
                                  void* const* f) {
  NvtxRange range("rb_h_func_evaluate_many");
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (n_calls < 0 || (n_calls > 0 && (!fn_ids || !precisions || !f)))
    return fail(RB_E_INVALID_ARGUMENT, "bad arguments");
  if (n_calls == 0) return RB_OK;
  if (n_calls > 1024) return fail(RB_E_INVALID_ARGUMENT, "more than 1024 calls");
  // every call's arguments in the reference's order before any work
  for (int32_t i = 0; i < n_calls; ++i) {
    const int32_t fn = fn_ids[i];
    if (fn < 0 || fn >= (int32_t)e->fns.size())
      return fail(RB_E_UNKNOWN_FUNCTION, "function id " + std::to_string(fn) + " is not in 0..36");
    if (e->fns[fn].category == RB_DISABLED)
      return fail(RB_E_DISABLED_FUNCTION, "function " + std::to_string(fn) + " needs dimension >= 10");
    if (n > e->max_concurrency)
      return fail(RB_E_BATCH_TOO_LARGE, "batch of " + std::to_string(n) + " exceeds max_concurrency=" +
                                            std::to_string(e->max_concurrency));
    if (precisions[i] != RB_DOUBLE && precisions[i] != RB_SINGLE)
      return fail(RB_E_INVALID_ARGUMENT, "precision must be RB_DOUBLE or RB_SINGLE");
    const int pi = precisions[i] == RB_DOUBLE ? 0 : 1;
    if (!e->why[pi][fn].empty())
      return fail(RB_E_UNSUPPORTED, "function " + std::to_string(fn) + ": " + e->why[pi][fn]);
    if (!f[i]) return fail(RB_E_INVALID_ARGUMENT, "null output pointer");
  }
  if (n < 1 || !x) return fail(RB_E_INVALID_ARGUMENT, "empty batch or null pointer");
  std::lock_guard<std::mutex> lock(e->host_mu);
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  RB_CUDA(cudaSetDevice(e->device));
  const rb_status s = evaluate_host_many_locked(e, n_calls, fn_ids, precisions, x, n, f);
  cudaSetDevice(prev);
  return s;
}

rb_status rb_initialize_sharded(const rb_pack* pk, int64_t max_concurrency, const int32_t* devices,
                                int32_t n_devices, rb_sharded** out) {
  if (!out) return fail(RB_E_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (!devices || n_devices < 1 || n_devices > rb::kMaxDevices)
    return fail(RB_E_INVALID_ARGUMENT, "1..16 devices required");
  rb_sharded* sh = new rb_sharded();
  int prev = 0;
  cudaGetDevice(&prev);
  rb_status st = RB_OK;
  for (int g = 0; g < n_devices && st == RB_OK; ++g) {
    rb_engine* e = nullptr;
    st = rb_initialize(pk, max_concurrency, devices[g], &e);
    if (st != RB_OK) break;
    sh->eng.push_back(e);
    sh->dev.push_back(devices[g]);
    cudaStream_t s = nullptr;
    cudaSetDevice(devices[g]);
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
      st = fail(RB_E_CUDA, "stream creation failed");
    sh->streams.push_back(s);
  }
  // peer access for the P2P all-gather stores (NVLink / NVSwitch)
  for (int g = 0; g < n_devices && st == RB_OK; ++g)
    for (int h = 0; h < n_devices; ++h) {
      if (devices[g] == devices[h]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[g], devices[h]);
      if (!can) {
        sh->p2p = false;
        continue;
      }
      cudaSetDevice(devices[g]);
      const cudaError_t err = cudaDeviceEnablePeerAccess(devices[h], 0);
      if (err == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (err != cudaSuccess) sh->p2p = false;
    }
  cudaSetDevice(prev);
  if (st != RB_OK) {
    rb_dispose_sharded(&sh);
    return st;
  }
  *out = sh;
  return RB_OK;
}

rb_status rb_dispose_sharded(rb_sharded** sh) {
  if (!sh || !*sh) return RB_OK;
  rb_sharded* s = *sh;
  for (size_t g = 0; g < s->eng.size(); ++g) {
    if (g < s->streams.size() && s->streams[g]) {
      cudaSetDevice(s->dev[g]);
      cudaStreamDestroy(s->streams[g]);
    }
    rb_dispose(&s->eng[g]);
  }
  delete s;
  *sh = nullptr;
  return RB_OK;
}

rb_status rb_func_evaluate_sharded(rb_sharded* sh, int32_t fn_id, int32_t precision,
                                   const void* const* x_shards, int64_t n_total, void* const* f_full,
                                   void* const* streams, int64_t* tickets) {
  NvtxRange range("rb_func_evaluate_sharded");
  if (!sh) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (precision == RB_DOUBLE)
    return evaluate_sharded<double>(sh, fn_id, x_shards, n_total, f_full, streams, tickets);
  if (precision == RB_SINGLE)
    return evaluate_sharded<float>(sh, fn_id, x_shards, n_total, f_full, streams, tickets);
  return fail(RB_E_INVALID_ARGUMENT, "precision must be RB_DOUBLE or RB_SINGLE");
}

rb_status rb_sharded_ticket_status(rb_sharded* sh, int32_t device_index, int64_t ticket) {
  if (!sh) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (device_index < 0 || device_index >= (int32_t)sh->eng.size())
    return fail(RB_E_INVALID_ARGUMENT, "device index out of range");
  if (ticket == -1) return RB_OK;            // that device had no rows
  return ticket_status(sh->eng[device_index], ticket);
}

rb_status rb_uniform_population(uint64_t key0, uint64_t key1, uint64_t first_element,
                                int64_t n_elements, double low, double high, double* out64,
                                float* out32, void* stream) {
  if (n_elements < 0 || (n_elements > 0 && !out64 && !out32))
    return fail(RB_E_INVALID_ARGUMENT, "bad arguments");
  if (n_elements == 0) return RB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (n_elements + 3) / 4 + 1;
  const int grid = (int)std::min<int64_t>((blocks + 255) / 256, 148 * 32);
  rb::uniform_population_kernel<<<grid, 256, 0, st>>>(key0, key1, first_element, n_elements, low,
                                                        high, out64, out32);
  g_launches.fetch_add(1);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

rb_status rb_np_powf(const float* x, const float* y, float* out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y || !out))) return fail(RB_E_INVALID_ARGUMENT, "bad arguments");
  if (n == 0) return RB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  rb::np_powf_kernel<<<grid, 256, 0, st>>>(x, y, out, n);
  g_launches.fetch_add(1);
  RB_CUDA(cudaGetLastError());
  RB_CUDA(cudaStreamSynchronize(st));
  return RB_OK;
}

rb_status rb_graph_capture(rb_engine* e, int32_t fn_id, int32_t precision, const void* x, int64_t n,
                           void* f, rb_graph** out) {
  NvtxRange range("rb_graph_capture");
  if (!out) return fail(RB_E_INVALID_ARGUMENT, "null graph handle");
  *out = nullptr;
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  if (prev != e->device) RB_CUDA(cudaSetDevice(e->device));
  rb_graph_t* g = nullptr;
  rb_status s;
  if (precision == RB_DOUBLE)
    s = capture_graph<double>(e, fn_id, static_cast<const double*>(x), n, static_cast<double*>(f), &g);
  else if (precision == RB_SINGLE)
    s = capture_graph<float>(e, fn_id, static_cast<const float*>(x), n, static_cast<float*>(f), &g);
  else
    s = fail(RB_E_INVALID_ARGUMENT, "precision must be RB_DOUBLE or RB_SINGLE");
  if (prev != e->device) cudaSetDevice(prev);
  if (s == RB_OK) *out = reinterpret_cast<rb_graph*>(g);
  return s;
}

rb_status rb_graph_launch(rb_graph* graph, void* stream) {
  rb_graph_t* g = reinterpret_cast<rb_graph_t*>(graph);
  if (!g) return fail(RB_E_USE_AFTER_DISPOSE, "graph was destroyed");
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  if (prev != g->device) RB_CUDA(cudaSetDevice(g->device));
  const cudaError_t err = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream));
  if (prev != g->device) cudaSetDevice(prev);
  if (err != cudaSuccess) return fail(RB_E_CUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(err));
  g_launches.fetch_add(1);
  return RB_OK;
}

rb_status rb_graph_status(rb_graph* graph) {
  rb_graph_t* g = reinterpret_cast<rb_graph_t*>(graph);
  if (!g) return fail(RB_E_USE_AFTER_DISPOSE, "graph was destroyed");
  return reinterpret_cast<volatile int*>(g->h_flag)[0] ? non_finite() : RB_OK;
}

rb_status rb_graph_destroy(rb_graph** graph) {
  if (!graph || !*graph) return RB_OK;
  release_graph(reinterpret_cast<rb_graph_t*>(*graph));
  *graph = nullptr;
  return RB_OK;
}

}  // extern "C"
