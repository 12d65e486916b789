// The evaluation kernel (device side), shared by the per-precision
// instantiation units rb_kern_f64.cu / rb_kern_f32.cu.
//
// Persistent grid; one CTA (256 threads) walks tiles of TP = 32 points:
//   load     X tile -> XS via one TMA bulk copy (cp.async.bulk + mbarrier),
//            double-buffered when shared memory allows (next tile in flight)
//   rotate   z = R (scale*(x - o)[perm] + pre) + post per diagonal block
//              fp64: mma.sync.m16n8k4.f64 (DMMA) on the tensor pipe.  The
//                    segment's (m-tile, n-tile) units are split into 8 equal
//                    contiguous ranges, one per warp; A fragments are built in
//                    registers from XS (shift/scale fused), B fragments come
//                    pre-swizzled from the pack (one 256-byte load each)
//              fp32: SIMT FMUL+FADD in NumPy's pairwise order (bit-exact z),
//                    4 points x 4 rows per thread from a q-ordered V tile
//            the epilogue scatters z into ZS and checks it is finite (the
//            reference's NonFiniteInput, engine.py:202-203, kernels.py:45-49)
//   kernel   8 lanes per point, NumPy-order reductions (rb_kernels.cuh)
//   blend    composition weights / member sum (composition.py:114-166)
// The function's descriptors and per-column gather tables live in shared
// memory for the CTA's lifetime ("plan").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/robench_b200.h"
#include "rb_kernels.cuh"

#ifndef RB_NTC
#define RB_NTC 2
#endif
#ifndef RB_MIN_BLOCKS_F64
#define RB_MIN_BLOCKS_F64 3
#endif
#ifndef RB_MIN_BLOCKS_F32
#define RB_MIN_BLOCKS_F32 2
#endif
#ifndef RB_F32_ROWS
#define RB_F32_ROWS 4             // rows per pass of the float32 rotate tile (4 or 2)
#endif

namespace rb {

constexpr int TP = 32;          // points per tile
constexpr int NT = 256;         // threads per CTA = 8 lanes x TP
constexpr int NWARPS = NT / 32;
constexpr int MAX_MEMBERS = 5;
constexpr int MAX_SEGMENTS = 16;
constexpr int MAX_GROUPS = 16;
constexpr int NTC = RB_NTC;     // DMMA n-tiles (8 rows) accumulated per pass
constexpr int GENERIC = -1;     // kernel template id for hybrids / compositions

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
  int* flag;        // set to 2 when a kernel input is not finite
  int ldz;          // ZS row stride (elements)
  int ldv;          // fp32 V tile rows (sum of 4-padded group sizes)
  int max_q;        // capacity of the plan's per-column tables
  int tma;          // x is 16-byte aligned: bulk-copy full tiles
  int nbuf;         // 2: prefetch the next tile while computing this one
};

struct PlanHead {
  rb_function fn;
  int seg_base, grp_base, n_seg, n_grp;
  rb_member mem[MAX_MEMBERS];
  rb_segment seg[MAX_SEGMENTS];
  rb_group grp[MAX_GROUPS];
  int gq0[MAX_GROUPS];            // group g's slice of the per-column tables (8-aligned)
  unsigned long long mbar[2];     // TMA completion barriers, one per X buffer
  uint32_t live;                  // points of the tile whose kernel inputs are checked
};

__host__ __device__ inline int round8(int v) { return (v + 7) & ~7; }

// dynamic shared memory:
//   [PlanHead][qsrc int[max_q]][prow int[max_q]][qo T[max_q]][XB0 (XB1)][V][ZS]
template <class T>
struct Smem {
  PlanHead* P;
  int* qsrc;      // x column feeding the group's q-th column (split perm applied)
  int* prow;      // z position of the group's r-th block row
  T* qo;          // the optimum at the q-th column
  T* XS;          // [TP][dim], the current tile (one of XB)
  T* XB[2];       // X tile buffers (XB[1] == XB[0] without prefetch)
  T* VS;          // fp32 only: [ldv][TP]
  T* ZS;          // [TP][ldz]
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

template <class T>
__host__ __device__ inline size_t smem_bytes(int dim, int ldv, int ldz, int max_q, int nbuf) {
  size_t b = align16(sizeof(PlanHead));
  b += 2 * align16(sizeof(int) * max_q) + align16(sizeof(T) * max_q);
  b += nbuf * align16(sizeof(T) * TP * dim);
  if (sizeof(T) == 4) b += align16(sizeof(T) * TP * ldv);
  b += align16(sizeof(T) * TP * ldz);
  return b;
}

template <class T>
__device__ inline Smem<T> carve(unsigned char* base, const Args<T>& a) {
  Smem<T> s;
  size_t off = 0;
  s.P = reinterpret_cast<PlanHead*>(base);
  off += align16(sizeof(PlanHead));
  s.qsrc = reinterpret_cast<int*>(base + off);
  off += align16(sizeof(int) * a.max_q);
  s.prow = reinterpret_cast<int*>(base + off);
  off += align16(sizeof(int) * a.max_q);
  s.qo = reinterpret_cast<T*>(base + off);
  off += align16(sizeof(T) * a.max_q);
  s.XB[0] = reinterpret_cast<T*>(base + off);
  off += align16(sizeof(T) * TP * a.dim);
  s.XB[1] = s.XB[0];
  if (a.nbuf == 2) {
    s.XB[1] = reinterpret_cast<T*>(base + off);
    off += align16(sizeof(T) * TP * a.dim);
  }
  s.XS = s.XB[0];
  s.VS = reinterpret_cast<T*>(base + off);
  if (sizeof(T) == 4) off += align16(sizeof(T) * TP * a.ldv);
  s.ZS = reinterpret_cast<T*>(base + off);
  return s;
}

__device__ __forceinline__ int round4(int v) { return (v + 3) & ~3; }
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ plan
// Copy the function's descriptors (contiguous in the pack) into shared
// memory and build the per-column gather tables (padded to 8 columns with
// column 0 and optimum 0: finite values times zero B entries) and the
// per-row scatter table.
template <class T>
__device__ void load_plan(const Args<T>& a, const Smem<T>& s) {
  PlanHead& P = *s.P;
  if (threadIdx.x == 0) {
    const rb_function fn = a.fns[a.fn];
    P.fn = fn;
    const rb_member first = a.members[fn.member0];
    const rb_member last = a.members[fn.member0 + fn.n_members - 1];
    P.seg_base = first.segment0;
    P.n_seg = last.segment0 + last.n_segments - first.segment0;
    const rb_segment s0 = a.segments[first.segment0];
    const rb_segment sl = a.segments[last.segment0 + last.n_segments - 1];
    P.grp_base = s0.group0;
    P.n_grp = sl.group0 + sl.n_groups - s0.group0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P.fn.n_members; i += NT) P.mem[i] = a.members[P.fn.member0 + i];
  for (int i = threadIdx.x; i < P.n_seg; i += NT) P.seg[i] = a.segments[P.seg_base + i];
  for (int i = threadIdx.x; i < P.n_grp; i += NT) P.grp[i] = a.groups[P.grp_base + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int q = 0;
    for (int g = 0; g < P.n_grp; ++g) {
      P.gq0[g] = q;
      q += round8(P.grp[g].m);
    }
  }
  __syncthreads();
  for (int mi = 0; mi < P.fn.n_members; ++mi) {
    const rb_member& mem = P.mem[mi];
    const T* o = a.values + mem.shift;
    for (int si = 0; si < mem.n_segments; ++si) {
      const rb_segment& seg = P.seg[mem.segment0 - P.seg_base + si];
      for (int gi = 0; gi < seg.n_groups; ++gi) {
        const int g = seg.group0 - P.grp_base + gi;
        const rb_group& G = P.grp[g];
        const int32_t* cols = a.index + G.col;
        const int32_t* rows = a.index + G.row;
        for (int q = threadIdx.x; q < round8(G.m); q += NT) {
          int src = 0, row = 0;
          T ov = T(0);
          if (q < G.m) {
            const int pos = cols[q];
            src = mem.perm >= 0 ? a.index[mem.perm + seg.src + pos] : pos;
            ov = o[src];
            row = rows[q];
          }
          s.qsrc[P.gq0[g] + q] = src;
          s.qo[P.gq0[g] + q] = ov;
          s.prow[P.gq0[g] + q] = row;
        }
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------- X tile load
// A tile is 32 consecutive rows = one contiguous span of X, so one
// cp.async.bulk (TMA bulk copy, completion on an mbarrier) moves it.
template <class T>
__device__ __forceinline__ bool tile_is_bulk(const Args<T>& a, int nv) {
  return a.tma && ((sizeof(T) * (size_t)nv * a.dim) & 15u) == 0;
}

template <class T>
__device__ __forceinline__ int tile_rows(const Args<T>& a, int64_t tile) {
  const int64_t left = a.n - tile * TP;
  return left < TP ? (int)left : TP;
}

// thread 0 only
template <class T>
__device__ __forceinline__ void issue_tile(const Args<T>& a, T* dst, unsigned long long* mbar,
                                           int64_t tile, int nv) {
  const uint32_t bytes = (uint32_t)(sizeof(T) * (size_t)nv * a.dim);
  const uint32_t bar = smem_u32(mbar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(a.x + tile * TP * a.dim), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void wait_tile(unsigned long long* mbar, uint32_t phase) {
  const uint32_t bar = smem_u32(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}

// z value into ZS; flags a non-finite value of a live point (kernels.py:45-49)
template <class T>
__device__ __forceinline__ void put_z(const Args<T>& a, const Smem<T>& s, int p, int pos, T v,
                                      bool& bad) {
  s.ZS[p * a.ldz + pos] = v;
  bad |= !M<T>::finite(v) && ((s.P->live >> p) & 1u);
}

// ------------------------------------------------------------ rotate fp64
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// z[p][row] = post + sum_q (scale*(x[p][src_q] - o_q) + pre) * B[q][r]
// Units = (group, 16-point m-tile, 8-row n-tile), ordered group-major; warp
// w owns units [w*U/8, (w+1)*U/8) and walks them in runs of <= NTC n-tiles
// that share (group, m-tile), so one A fragment per k-step feeds the run.
// Fragment layouts (PTX m16n8k4 .f64): a_i = (gid + 8i, tig), b = (tig, gid),
// c_i = (gid + 8*(i>>1), 2*tig + (i&1)).
__device__ inline bool rotate(const Args<double>& a, const Smem<double>& s, const rb_segment& seg) {
  const PlanHead& P = *s.P;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const double scale = seg.scale, pre = seg.pre, post = seg.post;
  const int g0 = seg.group0 - P.grp_base;
  int total = 0;
  for (int g = 0; g < seg.n_groups; ++g) total += (TP / 16) * ((P.grp[g0 + g].m + 7) >> 3);
  const int end = (warp + 1) * total / NWARPS;
  bool bad = false;
  for (int u = warp * total / NWARPS; u < end;) {
    int g = g0, rem = u;
    for (;;) {
      const int cnt = (TP / 16) * ((P.grp[g].m + 7) >> 3);
      if (rem < cnt) break;
      rem -= cnt;
      ++g;
    }
    const rb_group& G = P.grp[g];
    const int m = G.m, ntn = (m + 7) >> 3, nks = (m + 3) >> 2;
    const int mt = rem / ntn, nt0 = rem - mt * ntn;
    const int run = min(min(NTC, ntn - nt0), end - u);
    const double* F = a.values + G.frag + (size_t)nt0 * nks * 32 + lane;
    const int* qs = s.qsrc + P.gq0[g];
    const double* qo = s.qo + P.gq0[g];
    const double* X0 = s.XS + (mt * 16 + gid) * a.dim;
    const double* X1 = X0 + 8 * a.dim;
    double acc[NTC][4];
#pragma unroll
    for (int c = 0; c < NTC; ++c)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[c][i] = 0.0;
#pragma unroll 2
    for (int ks = 0; ks < nks; ++ks) {
      const int q = ks * 4 + tig;               // padded columns read x[.][0] * B = 0
      const int col = qs[q];
      const double o = qo[q];
      const double a0 = scale * (X0[col] - o) + pre;
      const double a1 = scale * (X1[col] - o) + pre;
#pragma unroll
      for (int c = 0; c < NTC; ++c)
        if (c < run) dmma_16x8x4(acc[c], a0, a1, __ldg(F + (c * nks + ks) * 32));
    }
    const int* prow = s.prow + P.gq0[g];
#pragma unroll
    for (int c = 0; c < NTC; ++c) {
      if (c >= run) break;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rr = (nt0 + c) * 8 + 2 * tig + (i & 1);
        if (rr < m) put_z(a, s, mt * 16 + gid + ((i >> 1) << 3), prow[rr], acc[c][i] + post, bad);
      }
    }
    u += run;
  }
  return bad;
}

// ------------------------------------------------------------ rotate fp32
// Exact NumPy order (transforms.py:42-48): rounded products, per-slot
// accumulation in q-order, slot fold ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)),
// ordered tail.  VS is [q][TP]; B rows are 4-padded (one float4 per q).
__device__ inline bool rotate(const Args<float>& a, const Smem<float>& s, const rb_segment& seg) {
  const PlanHead& P = *s.P;
  const int g0 = seg.group0 - P.grp_base;
  const float scale = (float)seg.scale, pre = (float)seg.pre, post = (float)seg.post;
  // gather: V[vq + q][p] = scale*(x[p][src_q] - o_q) + pre   (engine.py:97-100)
  {
    int vq = 0;
    for (int g = 0; g < seg.n_groups; ++g) {
      const int kp = round4(P.grp[g0 + g].m);
      const int* qs = s.qsrc + P.gq0[g0 + g];
      const float* qo = s.qo + P.gq0[g0 + g];
      for (int e = threadIdx.x; e < TP * kp; e += NT) {
        const int q = e / TP, p = e - q * TP;
        float v = scale * (s.XS[p * a.dim + qs[q]] - qo[q]);
        if (pre != 0.0f) v = v + pre;
        s.VS[(vq + q) * TP + p] = v;
      }
      vq += kp;
    }
  }
  __syncthreads();
  int total = 0;
  for (int g = 0; g < seg.n_groups; ++g) total += (TP / 4) * ((P.grp[g0 + g].m + 3) >> 2);
  bool bad = false;
  for (int t = threadIdx.x; t < total; t += NT) {
    int g = g0, rem = t, vq = 0;
    for (;;) {
      const int cnt = (TP / 4) * ((P.grp[g].m + 3) >> 2);
      if (rem < cnt) break;
      rem -= cnt;
      vq += round4(P.grp[g].m);
      ++g;
    }
    const rb_group& G = P.grp[g];
    const int pq = rem & 7, rq = rem >> 3;
    const int m = G.m, m4 = round4(m);
    const int* prow = s.prow + P.gq0[g];
    constexpr int RR = RB_F32_ROWS;
#pragma unroll 1
    for (int pass = 0; pass < 4 / RR; ++pass) {
      const int r0 = rq * 4 + pass * RR;
      if (r0 >= m) break;
      const float* B = a.values + G.mat + r0;
      float t0[4][RR], t1[4][RR], t2[4][RR], acc[4][RR];
#pragma unroll
      for (int sl = 0; sl < 8; ++sl) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < RR; ++j) acc[i][j] = 0.0f;
        for (int q = G.qb[sl]; q < G.qb[sl + 1]; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(s.VS + (vq + q) * TP + pq * 4);
          float bb[RR];
          if constexpr (RR == 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(B + q * m4));
            bb[0] = b.x; bb[1] = b.y; bb[2] = b.z; bb[3] = b.w;
          } else {
            const float2 b = __ldg(reinterpret_cast<const float2*>(B + q * m4));
            bb[0] = b.x; bb[1] = b.y;
          }
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < RR; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(vv[i], bb[j]));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < RR; ++j) {
            const float x = acc[i][j];
            switch (sl) {
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
        const float4 v = *reinterpret_cast<const float4*>(s.VS + (vq + q) * TP + pq * 4);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < RR; ++j) {
          const float b = __ldg(B + q * m4 + j);
#pragma unroll
          for (int i = 0; i < 4; ++i) t0[i][j] = __fadd_rn(t0[i][j], __fmul_rn(vv[i], b));
        }
      }
#pragma unroll
      for (int j = 0; j < RR; ++j) {
        if (r0 + j >= m) break;
        const int row = prow[r0 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          put_z(a, s, pq * 4 + i, row, post != 0.0f ? __fadd_rn(t0[i][j], post) : t0[i][j], bad);
      }
    }
  }
  return bad;
}

// ---------------------------------------------------------- one segment
// z of one segment into ZS (all points of the tile), then barrier.
template <class T>
__device__ void stage_segment(const Args<T>& a, const Smem<T>& s, const rb_member& mem,
                              const rb_segment& seg) {
  bool bad;
  if (seg.n_groups == 0) {                 // shift-only ids 10 and 15 (engine.py:96-104)
    const T* o = a.values + mem.shift;
    const int32_t* perm = mem.perm >= 0 ? a.index + mem.perm + seg.src : nullptr;
    const T scale = (T)seg.scale, pre = (T)seg.pre, post = (T)seg.post;
    const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
    bad = false;
    for (int j = l8; j < seg.d; j += 8) {
      const int src = perm ? perm[j] : j;
      T v = scale * (s.XS[p * a.dim + src] - o[src]);
      if (pre != T(0)) v = v + pre;
      if (post != T(0)) v = v + post;
      put_z(a, s, p, j, v, bad);
    }
  } else {
    bad = rotate(a, s, seg);
  }
  if (bad) atomicOr(a.flag, 2);
  __syncthreads();
}

// Value of one member (basic function, hybrid, or composition member) for
// the calling lane's point.
template <class T, int KID>
__device__ T member_value(const Args<T>& a, const Smem<T>& s, const rb_member& mem) {
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const PlanHead& P = *s.P;
  T total = T(0);
  for (int si = 0; si < mem.n_segments; ++si) {
    const rb_segment& seg = P.seg[mem.segment0 - P.seg_base + si];
    stage_segment(a, s, mem, seg);
    const Pt<T> pt{s.ZS + p * a.ldz, seg.d, l8, a.values + seg.ctab};
    T v;
    if constexpr (KID >= 0) v = kernel_value_k<T, KID>(pt);
    else v = kernel_value<T>(seg.kernel, pt);
    total = (si == 0) ? v : total + v;   // hybrid.py:105-115: 0 + K_0 + K_1 + ...
    __syncthreads();                      // ZS is rewritten by the next segment
  }
  return total;
}

// Resident CTAs per SM the register budget is sized for.
template <class T, int KID>
constexpr int min_blocks() {
  return sizeof(T) == 8 ? RB_MIN_BLOCKS_F64 : RB_MIN_BLOCKS_F32;
}

template <class T, int KID>
__global__ void __launch_bounds__(NT, (min_blocks<T, KID>()))
    evaluate_kernel(const Args<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Smem<T> s = carve<T>(smem_raw, a);
  load_plan(a, s);
  PlanHead& P = *s.P;
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int64_t ntiles = (a.n + TP - 1) / TP;
  uint32_t phase0 = 0u, phase1 = 0u;
  const int64_t first = blockIdx.x;
  if (a.nbuf == 2 && threadIdx.x == 0 && first < ntiles && tile_is_bulk(a, tile_rows(a, first)))
    issue_tile(a, s.XB[0], &P.mbar[0], first, tile_rows(a, first));

  int it = 0;
  for (int64_t tile = first; tile < ntiles; tile += gridDim.x, ++it) {
    const int b = (a.nbuf == 2) ? (it & 1) : 0;
    Smem<T> st = s;
    st.XS = b ? s.XB[1] : s.XB[0];
    const int64_t row0 = tile * TP;
    const int nv = tile_rows(a, tile);
    const uint32_t valid_mask = nv == 32 ? 0xffffffffu : ((1u << nv) - 1u);
    const int64_t next = tile + gridDim.x;
    if (threadIdx.x == 0) {
      if (a.nbuf == 2 && next < ntiles && tile_is_bulk(a, tile_rows(a, next)))
        issue_tile(a, b ? s.XB[0] : s.XB[1], b ? &P.mbar[0] : &P.mbar[1], next,
                   tile_rows(a, next));
      if (a.nbuf == 1 && tile_is_bulk(a, nv)) issue_tile(a, st.XS, &P.mbar[0], tile, nv);
      P.live = valid_mask;
    }
    if (tile_is_bulk(a, nv)) {
      if (b) {
        wait_tile(&P.mbar[1], phase1);
        phase1 ^= 1u;
      } else {
        wait_tile(&P.mbar[0], phase0);
        phase0 ^= 1u;
      }
    } else {
      const T* src = a.x + row0 * a.dim;
      for (int e = threadIdx.x; e < nv * a.dim; e += NT) st.XS[e] = src[e];
    }
    __syncthreads();
    // A non-finite x reaches some z of every evaluated member, so the z
    // checks cover the batch check of engine.py:202-203 as well.
    const bool valid = p < nv;
    T result;
    if constexpr (KID >= 0) {
      result = member_value<T, KID>(a, st, P.mem[0]);
    } else if (P.fn.category != RB_COMPOSITION) {
      result = member_value<T, GENERIC>(a, st, P.mem[0]);
    } else {
      // composition.py:114-141: weights from the squared distances
      const int nm = P.fn.n_members;
      const T* x = st.XS + p * a.dim;
      T d2[MAX_MEMBERS], om[MAX_MEMBERS];
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k) {
        d2[k] = T(0);
        om[k] = T(0);
        if (k < nm) {
          const T* o = a.values + P.mem[k].shift;
          d2[k] = pw8<T>(0, a.dim, [&](int j) { const T t = x[j] - o[j]; return t * t; }, l8);
        }
      }
      T mn = d2[0];
      int am = 0;
#pragma unroll
      for (int k = 1; k < MAX_MEMBERS; ++k)
        if (k < nm && d2[k] < mn) { mn = d2[k]; am = k; }
      if (mn < C<T>(1.0000000000000002e-24)) {          // 1e-12**2: on an optimum
#pragma unroll
        for (int k = 0; k < MAX_MEMBERS; ++k) om[k] = (k == am) ? T(1) : T(0);
      } else {
        T w[MAX_MEMBERS], tot = T(0);
#pragma unroll
        for (int k = 0; k < MAX_MEMBERS; ++k) {
          w[k] = T(0);
          if (k < nm) {
            const T sg = (T)P.mem[k].sigma;
            w[k] = apow<T>(d2[k], C<T>(-0.5)) *
                   M<T>::exp(-d2[k] / (C<T>(2.0 * a.dim) * (sg * sg)));
            tot = tot + w[k];
          }
        }
#pragma unroll
        for (int k = 0; k < MAX_MEMBERS; ++k)
          if (k < nm) om[k] = (tot == T(0)) ? C<T>(1.0 / nm) : w[k] / tot;
      }
      // composition.py:157-166: zero weights are skipped (and not checked)
      T total = T(0);
#pragma unroll 1
      for (int k = 0; k < nm; ++k) {
        T omk = T(0);
#pragma unroll
        for (int kk = 0; kk < MAX_MEMBERS; ++kk)
          if (kk == k) omk = om[kk];
        const bool use = valid && omk != T(0);
        __syncthreads();                                   // previous member done with P.live
        if (threadIdx.x == 0) P.live = 0u;
        __syncthreads();
        if (l8 == 0 && use) atomicOr(&P.live, 1u << p);
        if (!__syncthreads_or(use)) continue;
        const rb_member& mem = P.mem[k];
        const T g = member_value<T, GENERIC>(a, st, mem);
        if (omk != T(0)) total = total + omk * ((T)mem.height * g + (T)mem.bias);
      }
      result = total;
    }
    if (l8 == 0 && valid) a.f[row0 + p] = result + C<T>(100.0);     // engine.py:209
    __syncthreads();                                                 // XS reused by next TMA
  }
}

// Host-visible table of instantiations: [0..20] basic kernels, [21] generic.
constexpr int N_VARIANTS = K_COUNT + 1;

}  // namespace rb
