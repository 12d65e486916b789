// robench_b200: batched evaluation of the 37 suite functions on sm_100a.
//
// One CTA evaluates tiles of TP = 32 points (persistent grid-stride loop).
// Per tile, everything stays in shared memory:
//   XS[p][j]   the X rows of the tile (read from HBM once)
//   V          the shifted/scaled coordinates of one segment, in q-order
//   ZS[p][i]   the rotated vector z of one segment
// and the phases are
//   gather     v = scale*(x - o)[perm] + pre              (engine.py:96-100, hybrid.py:103-110)
//   rotate     z = R v + post per diagonal block           (transforms.py:42-48)
//                fp64: DMMA  mma.sync.m16n8k4.f64  (tensor pipe)
//                fp32: SIMT FMUL+FADD in NumPy's pairwise order (bit-exact z)
//   kernel     8 lanes per point, NumPy-order reductions   (kernels.py:52-228)
//   blend      composition weights and sum                 (composition.py:114-166)
// The reference's per-point Python loop (engine.py:205-213) becomes 8 lanes
// per point x 32 points per tile x (2..n) tiles per SM.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/robench_b200.h"
#include "rb_kernels.cuh"

namespace rb {

constexpr int TP = 32;        // points per tile
constexpr int NT = 256;       // threads per CTA = 8 lanes x TP
constexpr int MAX_MEMBERS = 5;

template <class T>
struct Args {
  const T* x;
  T* f;
  int64_t n;
  int dim;
  const rb_function* fns;
  const rb_member* members;
  const rb_segment* segments;
  const rb_group* groups;
  const int32_t* index;
  const T* values;
  int fn;
  int* flag;       // bit 0: non-finite x, bit 1: non-finite kernel input
  int ldx, ldv, ldz;
};

__device__ __forceinline__ int round4(int v) { return (v + 3) & ~3; }

// ------------------------------------------------------------ rotate fp64
// Z[p][row] = sum_q V[p][q] * B[q][r]  on the tensor pipe.  A = V (16 points
// x 4 q, row-major in smem), B = block (4 q x 8 rows), C in registers.
// Fragment layouts (PTX m16n8k4 .f64): a_i: (gid + 8i, tig); b: (tig, gid);
// c_i: (gid + 8*(i>>1), 2*tig + (i&1)).
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ void rotate_segment(const Args<double>& a, const rb_segment& seg, const double* VS,
                               double* ZS) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const double post = seg.post;
  // flatten (group, m-tile, n-tile) tasks over the 8 warps
  int total = 0;
  for (int g = 0; g < seg.n_groups; ++g) total += (TP / 16) * ((a.groups[seg.group0 + g].m + 7) >> 3);
  for (int t = warp; t < total; t += NT / 32) {
    int g = 0, rem = t, vq = 0;
    rb_group G = a.groups[seg.group0];
    for (;;) {
      const int cnt = (TP / 16) * ((G.m + 7) >> 3);
      if (rem < cnt) break;
      rem -= cnt;
      vq += round4(G.m);
      G = a.groups[seg.group0 + (++g)];
    }
    const int ntn = (G.m + 7) >> 3;
    const int mt = rem / ntn, nt = rem - mt * ntn;
    const int m = G.m, kp = round4(m);
    const double* B = a.values + G.mat;
    const double* A0 = VS + (mt * 16 + gid) * a.ldv + vq + tig;
    const double* A1 = A0 + 8 * a.ldv;
    const int r = nt * 8 + gid;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < kp; k0 += 4) {
      const int q = k0 + tig;
      const double b = (q < m && r < m) ? __ldg(B + q * m + r) : 0.0;
      dmma_16x8x4(c, A0[k0], A1[k0], b);
    }
    const int32_t* rows = a.index + G.row;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = nt * 8 + 2 * tig + (i & 1);
      const int pp = mt * 16 + gid + ((i >> 1) << 3);
      if (rr < m) {
        const double zv = post != 0.0 ? c[i] + post : c[i];
        ZS[pp * a.ldz + rows[rr]] = zv;
      }
    }
  }
}

// ------------------------------------------------------------ rotate fp32
// Exact NumPy order (transforms.py:42-48): every product rounded, each
// output's terms accumulated per pairwise-sum slot in q-order, slots folded
// ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)), tail appended in order.  A thread
// owns 4 points x 4 rows.  VT is [q][TP] (4 points = one 16-byte load).
__device__ void rotate_segment(const Args<float>& a, const rb_segment& seg, const float* VT,
                               float* ZS) {
  const float post = (float)seg.post;
  int total = 0;
  for (int g = 0; g < seg.n_groups; ++g) total += (TP / 4) * ((a.groups[seg.group0 + g].m + 3) >> 2);
  for (int t = threadIdx.x; t < total; t += NT) {
    int g = 0, rem = t, vq = 0;
    rb_group G = a.groups[seg.group0];
    for (;;) {
      const int cnt = (TP / 4) * ((G.m + 3) >> 2);
      if (rem < cnt) break;
      rem -= cnt;
      vq += round4(G.m);
      G = a.groups[seg.group0 + (++g)];
    }
    const int pq = rem & 7, rq = rem >> 3;   // TP/4 == 8 point-quads
    const int m = G.m;
    const float* B = a.values + G.mat;
    const int r0 = rq * 4;
    float t0[4][4], t1[4][4], t2[4][4], acc[4][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
      for (int q = G.qb[s]; q < G.qb[s + 1]; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(VT + (vq + q) * TP + pq * 4);
        float b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = (r0 + j < m) ? __ldg(B + q * m + r0 + j) : 0.0f;
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(vv[i], b[j]));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float x = acc[i][j];
          switch (s) {
            case 0: t0[i][j] = x; break;
            case 1: t0[i][j] = __fadd_rn(t0[i][j], x); break;
            case 2: t1[i][j] = x; break;
            case 3: t1[i][j] = __fadd_rn(t1[i][j], x); t0[i][j] = __fadd_rn(t0[i][j], t1[i][j]); break;
            case 4: t1[i][j] = x; break;
            case 5: t1[i][j] = __fadd_rn(t1[i][j], x); break;
            case 6: t2[i][j] = x; break;
            default:
              t2[i][j] = __fadd_rn(t2[i][j], x);
              t1[i][j] = __fadd_rn(t1[i][j], t2[i][j]);
              t0[i][j] = __fadd_rn(t0[i][j], t1[i][j]);
          }
        }
    }
    for (int q = G.qb[8]; q < G.qb[9]; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(VT + (vq + q) * TP + pq * 4);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float b = (r0 + j < m) ? __ldg(B + q * m + r0 + j) : 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) t0[i][j] = __fadd_rn(t0[i][j], __fmul_rn(vv[i], b));
      }
    }
    const int32_t* rows = a.index + G.row;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (r0 + j >= m) break;
      const int row = rows[r0 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float zv = post != 0.0f ? __fadd_rn(t0[i][j], post) : t0[i][j];
        ZS[(pq * 4 + i) * a.ldz + row] = zv;
      }
    }
  }
}

// V layout helpers: fp64 [p][ldv] (DMMA A operand), fp32 [q][TP].
__device__ __forceinline__ int v_at(const Args<double>& a, int p, int q) { return p * a.ldv + q; }
__device__ __forceinline__ int v_at(const Args<float>& a, int p, int q) { return q * TP + p; }

// ------------------------------------------------------------ one segment
// Gather + transform into V (or straight into ZS when not rotated), rotate.
template <class T>
__device__ void stage_segment(const Args<T>& a, const rb_member& mem, const rb_segment& seg,
                              const T* XS, T* VS, T* ZS) {
  const T* o = a.values + mem.shift;
  const int32_t* perm = mem.perm >= 0 ? a.index + mem.perm + seg.src : nullptr;
  const T scale = (T)seg.scale, pre = (T)seg.pre, post = (T)seg.post;
  if (seg.n_groups == 0) {
    const int d = seg.d;
    for (int e = threadIdx.x; e < TP * d; e += NT) {
      const int p = e / d, j = e - p * d;
      const int src = perm ? perm[j] : j;
      T v = scale * (XS[p * a.ldx + src] - o[src]);
      if (pre != T(0)) v = v + pre;
      if (post != T(0)) v = v + post;
      ZS[p * a.ldz + j] = v;
    }
    __syncthreads();
    return;
  }
  int vq = 0;
  for (int g = 0; g < seg.n_groups; ++g) {
    const rb_group G = a.groups[seg.group0 + g];
    const int kp = round4(G.m);
    const int32_t* cols = a.index + G.col;
    for (int e = threadIdx.x; e < TP * kp; e += NT) {
      int p, q;
      if (sizeof(T) == 8) { p = e / kp; q = e - p * kp; }   // q fastest: row-major V
      else { q = e / TP; p = e - q * TP; }                   // p fastest: [q][p] V
      T v = T(0);
      if (q < G.m) {
        const int pos = cols[q];
        const int src = perm ? perm[pos] : pos;
        v = scale * (XS[p * a.ldx + src] - o[src]);
        if (pre != T(0)) v = v + pre;
      }
      VS[v_at(a, p, vq + q)] = v;
    }
    vq += kp;
  }
  __syncthreads();
  rotate_segment(a, seg, VS, ZS);
  __syncthreads();
}

// Value of one member (a basic function, a hybrid, or a composition member)
// for the calling lane's point; `live` masks the finiteness check.
template <class T>
__device__ T member_value(const Args<T>& a, const rb_member& mem, const T* XS, T* VS, T* ZS,
                          bool live) {
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  T total = T(0);
  for (int s = 0; s < mem.n_segments; ++s) {
    const rb_segment seg = a.segments[mem.segment0 + s];
    stage_segment(a, mem, seg, XS, VS, ZS);
    const T* z = ZS + p * a.ldz;
    bool bad = false;
    for (int j = l8; j < seg.d; j += 8) bad |= !M<T>::finite(z[j]);   // kernels.py:45-49
    if (bad && live) atomicOr(a.flag, 2);
    const Pt<T> P{z, seg.d, l8, a.values + seg.ctab};
    const T v = kernel_value<T>(seg.kernel, P);
    total = (s == 0) ? v : total + v;   // hybrid.py:105-115: 0 + K_0 + K_1 + ...
    __syncthreads();                     // ZS / VS are rewritten by the next segment
  }
  return total;
}

template <class T>
__global__ void __launch_bounds__(NT, 2) evaluate_kernel(const Args<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* XS = reinterpret_cast<T*>(smem_raw);
  T* VS = XS + TP * a.ldx;
  T* ZS = VS + TP * a.ldv;
  const rb_function fn = a.fns[a.fn];
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int64_t ntiles = (a.n + TP - 1) / TP;
  const int D = a.dim;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * TP;
    const int64_t left = a.n - row0;
    const int nv = left < TP ? (int)left : TP;
    // -- load the tile's rows (coalesced per row) and check finiteness
    {
      bool bad = false;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int r = warp; r < TP; r += NT / 32) {
        T* dst = XS + r * a.ldx;
        if (r < nv) {
          const T* src = a.x + (row0 + r) * D;
          for (int j = lane; j < D; j += 32) {
            const T v = src[j];
            bad |= !M<T>::finite(v);
            dst[j] = v;
          }
        } else {
          for (int j = lane; j < D; j += 32) dst[j] = T(0);
        }
      }
      if (bad) atomicOr(a.flag, 1);                                    // engine.py:202-203
    }
    __syncthreads();

    T result;
    const bool valid = p < nv;
    if (fn.category != RB_COMPOSITION) {
      result = member_value(a, a.members[fn.member0], XS, VS, ZS, valid);
    } else {
      // composition.py:114-141 — weights from squared distances to the optima
      const int nm = fn.n_members;
      T d2[MAX_MEMBERS], om[MAX_MEMBERS];
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k) {
        d2[k] = T(0);
        om[k] = T(0);
        if (k < nm) {
          const T* o = a.values + a.members[fn.member0 + k].shift;
          const T* x = XS + p * a.ldx;
          d2[k] = pw8<T>(0, D, [&](int j) { const T t = x[j] - o[j]; return t * t; }, l8);
        }
      }
      T mn = d2[0];
      int am = 0;
#pragma unroll
      for (int k = 1; k < MAX_MEMBERS; ++k)
        if (k < nm && d2[k] < mn) { mn = d2[k]; am = k; }
      if (mn < C<T>(1.0000000000000002e-24)) {          // 1e-12**2, an exact optimum
#pragma unroll
        for (int k = 0; k < MAX_MEMBERS; ++k) om[k] = (k == am) ? T(1) : T(0);
      } else {
        T w[MAX_MEMBERS], tot = T(0);
#pragma unroll
        for (int k = 0; k < MAX_MEMBERS; ++k) {
          w[k] = T(0);
          if (k < nm) {
            const T sg = (T)a.members[fn.member0 + k].sigma;
            w[k] = apow<T>(d2[k], C<T>(-0.5)) * M<T>::exp(-d2[k] / (C<T>(2.0 * D) * (sg * sg)));
            tot = tot + w[k];
          }
        }
#pragma unroll
        for (int k = 0; k < MAX_MEMBERS; ++k)
          if (k < nm) om[k] = (tot == T(0)) ? C<T>(1.0 / nm) : w[k] / tot;
      }
      // composition.py:157-166 — members with a zero weight are skipped
      T total = T(0);
#pragma unroll 1
      for (int k = 0; k < nm; ++k) {
        T omk = T(0);
#pragma unroll
        for (int kk = 0; kk < MAX_MEMBERS; ++kk) if (kk == k) omk = om[kk];
        const bool use = valid && omk != T(0);
        if (!__syncthreads_or(use)) continue;
        const rb_member mem = a.members[fn.member0 + k];
        const T g = member_value(a, mem, XS, VS, ZS, use);
        if (omk != T(0)) total = total + omk * ((T)mem.height * g + (T)mem.bias);
      }
      result = total;
    }
    if (l8 == 0 && valid) a.f[row0 + p] = result + C<T>(100.0);     // engine.py:209
    __syncthreads();
  }
}

__global__ void np_powf_kernel(const float* x, const float* y, float* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rb_svml::powf_np(x[i], y[i]);
}

}  // namespace rb

// =====================================================================
//                               host side
// =====================================================================

namespace {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

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

constexpr int kFlagSlots = 4096;

}  // namespace

struct rb_engine {
  int device = 0;
  int dim = 0;
  int64_t max_concurrency = 0;
  int max_exact_len = 0;
  std::vector<rb_function> fns;              // host copy for validation
  rb_function* d_fns = nullptr;
  rb_member* d_members = nullptr;
  rb_segment* d_segments = nullptr;
  rb_group* d_groups = nullptr;
  int32_t* d_index = nullptr;
  double* d_v64 = nullptr;
  float* d_v32 = nullptr;
  int* d_flags = nullptr;                    // kFlagSlots ring (concurrent calls)
  int* h_flags = nullptr;                    // pinned mirror
  std::atomic<int> next_flag{0};
  int ldx[2], ldv[2], ldz[2];                // [0] fp64, [1] fp32
  size_t smem[2];
  int grid_cap[2];
  std::mutex host_mu;                        // host-pointer API staging
  void* h_stage_x = nullptr;
  void* h_stage_f = nullptr;
  size_t stage_bytes_x = 0, stage_bytes_f = 0;
  cudaStream_t host_stream = nullptr;
};

namespace {

int pad_to(int v, int mod, int rem) {        // smallest u >= v with u % mod == rem
  int u = v;
  while (u % mod != rem) ++u;
  return u;
}

void release(rb_engine* e) {
  if (!e) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(e->device);
  cudaFree(e->d_fns);
  cudaFree(e->d_members);
  cudaFree(e->d_segments);
  cudaFree(e->d_groups);
  cudaFree(e->d_index);
  cudaFree(e->d_v64);
  cudaFree(e->d_v32);
  cudaFree(e->d_flags);
  cudaFree(e->h_stage_x);
  cudaFree(e->h_stage_f);
  if (e->h_flags) cudaFreeHost(e->h_flags);
  if (e->host_stream) cudaStreamDestroy(e->host_stream);
  cudaSetDevice(prev);
  delete e;
}

template <class T>
rb_status evaluate_device(rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f,
                          cudaStream_t stream) {
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (fn_id < 0 || fn_id >= (int32_t)e->fns.size())
    return fail(RB_E_UNKNOWN_FUNCTION, "function id " + std::to_string(fn_id) + " is not in 0..36");
  const rb_function& fn = e->fns[fn_id];
  if (fn.category == RB_DISABLED)
    return fail(RB_E_DISABLED_FUNCTION,
                "function " + std::to_string(fn_id) + " needs dimension >= 10");
  if (n > e->max_concurrency)
    return fail(RB_E_BATCH_TOO_LARGE, "batch of " + std::to_string(n) +
                                          " exceeds max_concurrency=" +
                                          std::to_string(e->max_concurrency));
  if (n < 1 || !x || !f) return fail(RB_E_INVALID_ARGUMENT, "empty batch or null pointer");
  const int pi = sizeof(T) == 8 ? 0 : 1;
  if (pi == 1 && e->max_exact_len > 128)
    return fail(RB_E_UNSUPPORTED, "single precision needs rotated segments of length <= 128");

  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  if (prev != e->device) RB_CUDA(cudaSetDevice(e->device));
  const int slot = e->next_flag.fetch_add(1) % kFlagSlots;
  int* dflag = e->d_flags + slot;
  RB_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), stream));

  rb::Args<T> a;
  a.x = x;
  a.f = f;
  a.n = n;
  a.dim = e->dim;
  a.fns = e->d_fns;
  a.members = e->d_members;
  a.segments = e->d_segments;
  a.groups = e->d_groups;
  a.index = e->d_index;
  a.values = reinterpret_cast<const T*>(pi == 0 ? (const void*)e->d_v64 : (const void*)e->d_v32);
  a.fn = fn_id;
  a.flag = dflag;
  a.ldx = e->ldx[pi];
  a.ldv = e->ldv[pi];
  a.ldz = e->ldz[pi];
  const int64_t ntiles = (n + rb::TP - 1) / rb::TP;
  const int grid = (int)std::min<int64_t>(ntiles, e->grid_cap[pi]);
  rb::evaluate_kernel<T><<<grid, rb::NT, e->smem[pi], stream>>>(a);
  g_launches.fetch_add(1);
  RB_CUDA(cudaGetLastError());
  RB_CUDA(cudaMemcpyAsync(e->h_flags + slot, dflag, sizeof(int), cudaMemcpyDeviceToHost, stream));
  RB_CUDA(cudaStreamSynchronize(stream));
  const int flag = e->h_flags[slot];
  if (prev != e->device) cudaSetDevice(prev);
  if (flag & 1) return fail(RB_E_NON_FINITE_INPUT, "batch contains NaN or infinity");
  if (flag & 2) return fail(RB_E_NON_FINITE_INPUT, "kernel input contains NaN or infinity");
  return RB_OK;
}

template <class T>
rb_status evaluate_host(rb_engine* e, int32_t fn_id, const T* x, int64_t n, T* f) {
  if (!e) return fail(RB_E_USE_AFTER_DISPOSE, "engine was disposed");
  if (n < 1 || n > e->max_concurrency || !x || !f)   // let the device path report the error
    return evaluate_device<T>(e, fn_id, x, n, f, nullptr);
  std::lock_guard<std::mutex> lock(e->host_mu);
  int prev = 0;
  RB_CUDA(cudaGetDevice(&prev));
  RB_CUDA(cudaSetDevice(e->device));
  const size_t bx = sizeof(T) * (size_t)n * e->dim, bf = sizeof(T) * (size_t)n;
  if (bx > e->stage_bytes_x) {
    cudaFree(e->h_stage_x);
    e->h_stage_x = nullptr;
    RB_CUDA(cudaMalloc(&e->h_stage_x, bx));
    e->stage_bytes_x = bx;
  }
  if (bf > e->stage_bytes_f) {
    cudaFree(e->h_stage_f);
    e->h_stage_f = nullptr;
    RB_CUDA(cudaMalloc(&e->h_stage_f, bf));
    e->stage_bytes_f = bf;
  }
  RB_CUDA(cudaMemcpyAsync(e->h_stage_x, x, bx, cudaMemcpyHostToDevice, e->host_stream));
  const rb_status s = evaluate_device<T>(e, fn_id, static_cast<const T*>(e->h_stage_x), n,
                                         static_cast<T*>(e->h_stage_f), e->host_stream);
  if (s == RB_OK)
    RB_CUDA(cudaMemcpyAsync(f, e->h_stage_f, bf, cudaMemcpyDeviceToHost, e->host_stream));
  RB_CUDA(cudaStreamSynchronize(e->host_stream));
  cudaSetDevice(prev);
  return s;
}

}  // namespace

extern "C" {

int32_t rb_abi_version(void) { return 1; }

const char* rb_last_error(void) { return g_last_error.c_str(); }

int64_t rb_launch_count(void) { return g_launches.load(); }

void rb_struct_sizes(int64_t out[5]) {
  out[0] = sizeof(rb_group);
  out[1] = sizeof(rb_segment);
  out[2] = sizeof(rb_member);
  out[3] = sizeof(rb_function);
  out[4] = sizeof(rb_pack);
}

rb_status rb_initialize(const rb_pack* pk, int64_t max_concurrency, int32_t device,
                        rb_engine** out) {
  if (!pk || !out) return fail(RB_E_INVALID_ARGUMENT, "null pack or output pointer");
  *out = nullptr;
  if (pk->dim < 2 || pk->n_functions <= 0 || max_concurrency < 1)
    return fail(RB_E_INVALID_ARGUMENT, "malformed pack");
  // structural validation of the pack (offsets in range)
  for (int i = 0; i < pk->n_functions; ++i) {
    const rb_function& f = pk->functions[i];
    if (f.category == RB_DISABLED) continue;
    if (f.n_members < 1 || f.n_members > rb::MAX_MEMBERS || f.member0 < 0 ||
        f.member0 + f.n_members > pk->n_members)
      return fail(RB_E_INVALID_ARGUMENT, "function " + std::to_string(i) + ": bad members");
  }
  int max_exact = 0, max_q = 0, max_d = 0;
  for (int i = 0; i < pk->n_segments; ++i) {
    const rb_segment& s = pk->segments[i];
    if (s.kernel < 0 || s.kernel >= rb::K_COUNT || s.d < 1 || s.d > pk->dim ||
        s.group0 + s.n_groups > pk->n_groups)
      return fail(RB_E_INVALID_ARGUMENT, "segment " + std::to_string(i) + " malformed");
    int q = 0;
    for (int g = 0; g < s.n_groups; ++g) q += (pk->groups[s.group0 + g].m + 3) & ~3;
    max_q = std::max(max_q, q);
    max_d = std::max(max_d, s.d);
    if (s.n_groups) max_exact = std::max(max_exact, s.d);
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
  e->max_exact_len = max_exact;
  e->fns.assign(pk->functions, pk->functions + pk->n_functions);
  rb_status s = RB_OK;
  if (s == RB_OK) s = upload(&e->d_fns, pk->functions, pk->n_functions);
  if (s == RB_OK) s = upload(&e->d_members, pk->members, pk->n_members);
  if (s == RB_OK) s = upload(&e->d_segments, pk->segments, pk->n_segments);
  if (s == RB_OK) s = upload(&e->d_groups, pk->groups, pk->n_groups);
  if (s == RB_OK) s = upload(&e->d_index, pk->index, pk->n_index);
  if (s == RB_OK) s = upload(&e->d_v64, pk->values_f64, pk->n_values);
  if (s == RB_OK) s = upload(&e->d_v32, pk->values_f32, pk->n_values);
  if (s == RB_OK && cudaMalloc(&e->d_flags, sizeof(int) * kFlagSlots) != cudaSuccess)
    s = fail(RB_E_CUDA, "flag allocation failed");
  if (s == RB_OK && cudaMallocHost(&e->h_flags, sizeof(int) * kFlagSlots) != cudaSuccess)
    s = fail(RB_E_CUDA, "pinned flag allocation failed");
  if (s == RB_OK && cudaStreamCreateWithFlags(&e->host_stream, cudaStreamNonBlocking) != cudaSuccess)
    s = fail(RB_E_CUDA, "stream creation failed");
  if (s == RB_OK) {
    const int D = pk->dim;
    // fp64: rows of XS / ZS read by 8 lanes x 4 points -> stride = 8 (mod 16)
    // doubles; V is the DMMA A operand -> stride = 4 (mod 16) doubles.
    e->ldx[0] = pad_to(D, 16, 8);
    e->ldz[0] = pad_to(std::max(max_d, 1), 16, 8);
    e->ldv[0] = pad_to(std::max(max_q, 4), 16, 4);
    // fp32: XS rows odd (conflict-free column gathers), ZS = 8 (mod 32), V is [q][TP].
    e->ldx[1] = D | 1;
    e->ldz[1] = pad_to(std::max(max_d, 1), 32, 8);
    e->ldv[1] = std::max(max_q, 4);
    e->smem[0] = sizeof(double) * (size_t)rb::TP * (e->ldx[0] + e->ldv[0] + e->ldz[0]);
    e->smem[1] = sizeof(float) * (size_t)rb::TP * (e->ldx[1] + e->ldv[1] + e->ldz[1]);
    int sms = 0, optin = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    for (int pi = 0; pi < 2 && s == RB_OK; ++pi) {
      if ((int)e->smem[pi] > optin) {
        s = fail(RB_E_UNSUPPORTED, "dimension too large for the shared-memory tile");
        break;
      }
      cudaError_t err = pi == 0 ? cudaFuncSetAttribute(rb::evaluate_kernel<double>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)e->smem[0])
                                : cudaFuncSetAttribute(rb::evaluate_kernel<float>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)e->smem[1]);
      if (err != cudaSuccess) { s = fail(RB_E_CUDA, cudaGetErrorString(err)); break; }
      int per_sm = 0;
      err = pi == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                          &per_sm, rb::evaluate_kernel<double>, rb::NT, e->smem[0])
                    : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                          &per_sm, rb::evaluate_kernel<float>, rb::NT, e->smem[1]);
      if (err != cudaSuccess || per_sm < 1) {
        s = fail(RB_E_UNSUPPORTED, "kernel does not fit on an SM");
        break;
      }
      e->grid_cap[pi] = sms * per_sm;
    }
  }
  cudaSetDevice(prev);
  if (s != RB_OK) {
    release(e);
    return s;
  }
  *out = e;
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

rb_status rb_dispose(rb_engine** engine) {
  if (!engine || !*engine) return RB_OK;
  release(*engine);
  *engine = nullptr;
  return RB_OK;
}

rb_status rb_func_evaluate(rb_engine* e, int32_t fn_id, const double* x, int64_t n, double* f,
                           void* stream) {
  return evaluate_device<double>(e, fn_id, x, n, f, static_cast<cudaStream_t>(stream));
}

rb_status rb_func_evaluatef(rb_engine* e, int32_t fn_id, const float* x, int64_t n, float* f,
                            void* stream) {
  return evaluate_device<float>(e, fn_id, x, n, f, static_cast<cudaStream_t>(stream));
}

rb_status rb_h_func_evaluate(rb_engine* e, int32_t fn_id, const double* x, int64_t n,
                             double* f) {
  return evaluate_host<double>(e, fn_id, x, n, f);
}

rb_status rb_h_func_evaluatef(rb_engine* e, int32_t fn_id, const float* x, int64_t n,
                              float* f) {
  return evaluate_host<float>(e, fn_id, x, n, f);
}

}  // extern "C"
