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

#ifndef RB_MIN_BLOCKS_F64
#define RB_MIN_BLOCKS_F64 3
#endif
#ifndef RB_MIN_BLOCKS_F32
#define RB_MIN_BLOCKS_F32 2
#endif
#ifndef RB_F32_UNROLL
#define RB_F32_UNROLL 2           // column-loop unroll of the float32 rotate slots
#endif
constexpr int kF32Unroll = RB_F32_UNROLL;
#ifndef RB_F32_FAST_WEIGHTS
#define RB_F32_FAST_WEIGHTS 1
#endif
#ifndef RB_F32_ROWS
#define RB_F32_ROWS 4             // rows per pass of the float32 rotate tile (4 or 2)
#endif

namespace rb {

#ifndef RB_TP
#define RB_TP 32
#endif
constexpr int TP = RB_TP;       // points per tile (16 or 32)

// Optional phase timing (tools/phase_timing.py): thread 0 of every CTA adds
// the clock64() spent per tile in load / z staging / kernel phases.
#ifdef RB_PHASE_TIMING
static __device__ unsigned long long g_phase[8];
#define RB_PHASE_MARK(var) const long long var = clock64()
#define RB_PHASE_ADD(i, dt) if (threadIdx.x == 0) atomicAdd(&g_phase[i], (unsigned long long)(dt))
#else
#define RB_PHASE_MARK(var)
#define RB_PHASE_ADD(i, dt)
#endif
constexpr int NT = 8 * TP;      // threads per CTA = 8 lanes x TP
constexpr int NWARPS = NT / 32;
constexpr int MAX_MEMBERS = 5;
constexpr int MAX_SEGMENTS = 16;
constexpr int MAX_GROUPS = 16;
constexpr int MAX_UNITS = 512;  // fp64 DMMA units (m-tile x n-tile of a group) per function
// MT2 (float64 DMMA rotate): one unit covers both 16-point m-tiles of the
// tile, so each B fragment load feeds twice the DMMAs (half the B traffic
// from L1 / L2).  Measured: basic functions +0-4 %, hybrids +5-8 %;
// compositions -10-20 % (the extra accumulators spill at their register
// budget), which keep one m-tile per unit.
static_assert(TP == 32, "MT2 units cover the tile's two m-tiles");
template <int KID>
__host__ __device__ constexpr bool mt2_kernel() { return KID >= 0 && KID < 100 + 29; }   // basic + hybrids 23-28
constexpr int NTC = 2;          // DMMA n-tiles (8 rows) sharing one A fragment per k-step
                                // (3 measured: +1-3% basic, -10-18% compositions: spills)
constexpr int GENERIC = -1;     // kernel template id for hybrids / compositions
constexpr int FIXUP = -2;       // member_value mode of fixup_kernel (exact-order float64)
constexpr int BIGDIM = -3;      // member_value mode of evaluate_big_kernel (tiles in global memory)
// modes that evaluate exact64 members in NumPy's order directly (no marks)
__host__ __device__ constexpr bool exact_mode(int kid) { return kid == FIXUP || kid == BIGDIM; }

// Kernel arguments: 128 bytes.  Measured: 4-16 more bytes (unused) cost
// the float64 composition kernels 8-16 % at N = 10^7 (code generation), so
// anything new must fit inside them.
template <class T>
struct Args {
  const T* x;
  T* f;
  int64_t n;
  int dim;
  int fn;
  const rb_function* fns;
  const rb_member* members;
  const rb_segment* segments;
  const rb_group* groups;
  const int32_t* index;
  const T* values;
  int* flag;        // set to 2 when a kernel input is not finite (mapped host memory)
  int* mark;        // float64: the call's word in device memory (zeroed before the launch),
                    // 1 once a row is left for fixup_kernel (read there, not over PCIe)
  int ldz;          // ZS row stride (elements)
  int ldv;          // fp32 V tile rows (sum of 4-padded group sizes)
  int max_q;        // capacity of the plan's per-column tables
  int tma;          // x is 16-byte aligned: bulk-copy full tiles
  int nbuf;         // 2: prefetch the next tile while computing this one
  int l2pf;         // 1: also pull the tile after the next in-flight one into L2
  int opt_rows;     // member optima staged in shared memory (compositions)
  float neg_zero;   // -0.0f, opaque to ptxas (see f32_leaf)
};
static_assert(sizeof(Args<double>) == 128 && sizeof(Args<float>) == 128,
              "kernel arguments outgrew 128 bytes (see the note above)");

// every writer stores the same value: a plain store (the flag is in mapped
// host memory, where device atomics need not be supported)
template <class T>
__device__ __forceinline__ void raise_flag(const Args<T>& a) {
  *reinterpret_cast<volatile int*>(a.flag) = 2;
}
// a.flag[1]: some row's value was left for fixup_kernel (float64 exact64
// members next to the HappyCat / HGBat residual); the row holds fixup_mark
// until the fixup pass overwrites it
// (points next to an optimum; in a converged population, every row): two
// plain stores, no reads -- the device word for fixup_kernel, the host flag
// for the blocking callers.
template <class T>
__device__ __forceinline__ void mark_fixup(const Args<T>& a) {
  *reinterpret_cast<volatile int*>(a.mark) = 1;
  reinterpret_cast<volatile int*>(a.flag)[1] = 1;
}
// a signalling-NaN payload no arithmetic produces (NaN results are quiet)
constexpr unsigned long long kFixupBits = 0x7ff4f1c5ed0ddba1ull;
template <class T> __device__ __forceinline__ T fixup_mark() { return (T)__longlong_as_double(kFixupBits); }
__device__ __forceinline__ bool is_fixup_mark(double v) {
  return (unsigned long long)__double_as_longlong(v) == kFixupBits;
}

struct PlanHead {
  rb_function fn;
  int seg_base, grp_base, n_seg, n_grp;
  rb_member mem[MAX_MEMBERS];
  rb_segment seg[MAX_SEGMENTS];
  rb_group grp[MAX_GROUPS];
  int gq0[MAX_GROUPS];            // group g's slice of the per-column tables (8-aligned)
  int8_t grp_seg[MAX_GROUPS];     // plan segment owning group g
  unsigned long long mbar[2];     // TMA completion barriers, one per X buffer
  uint32_t live;                  // valid points of the current tile
  uint32_t livek[MAX_MEMBERS];    // compositions: valid points with a nonzero weight, per member
  int n_jobs;                     // (member, segment) pairs per tile, in evaluation order
  int8_t job_mem[MAX_SEGMENTS];
  int8_t job_seg[MAX_SEGMENTS];   // index into seg[]
  int unit_off[MAX_SEGMENTS + 1];  // fp64 rotate: segment si's units are unit[unit_off[si] ..)
  uint32_t exact_mem;             // fp64: members with an exact-order path (exact64_kernel)
  uint32_t marked;                // fixup_kernel: marked points of the current chunk
  int icum[MAX_GROUPS + 1];       // fp32 rotate: items (4 points x 4 rows) before plan group g
  int vcum[MAX_GROUPS + 1];       // fp32: V rows (4-padded group sizes) before plan group g
  float gsc32[MAX_GROUPS], gpre32[MAX_GROUPS], gpost32[MAX_GROUPS];  // fp32: group's segment constants
  uint32_t unit[MAX_UNITS];       // (group | m-tile << 8 | n-tile << 16), group-major per segment
};

// float64 kernels whose value amplifies the last ulp of z beyond the parity
// bar next to an optimum: HappyCat's |sum z^2 - d|^0.25 and HGBat's
// sqrt(|r2^2 - sz^2|) are not differentiable where the residual vanishes
// (kernels.py:204-217), and the residual vanishes exactly at the optimum
// (z = -1).  Members containing them keep the DMMA rotate; a tile in which
// some point's residual is small relative to its terms (ill64) re-stages the
// member with z in NumPy's exact order -- rounded products, the pairwise
// slots of transforms.py:42-48 -- and sums r2 and sz in NumPy's order too,
// so the residual carries the reference's bits (rotate_exact_f64).
__host__ __device__ constexpr bool exact64_kernel(int k) { return k == K_HAPPYCAT || k == K_HGBAT; }

__host__ __device__ inline int round8(int v) { return (v + 7) & ~7; }

// dynamic shared memory:
//   fp32: [PlanHead][qsrc int[max_q]][prow int[max_q]][qo T[max_q]][XB0 (XB1)][V][ZS]
//   fp64: [PlanHead][qsrc int[max_q]][prow int[max_q]][qo T[max_q]][cz T[max_q]][XS][ZS]
template <class T>
struct Smem {
  PlanHead* P;
  int* qsrc;      // x column feeding the group's q-th column (split perm applied)
  int* prow;      // z position of the group's r-th block row
  T* qo;          // the optimum at the q-th column
  T* cz;          // fp64: offset constant of the r-th block row (pack.py group())
  T* opt;         // compositions: member optima [n_members][dim]
  T* XS;          // [TP][dim], the current tile (one of XB)
  T* XB[2];       // X tile buffers (XB[1] == XB[0] without prefetch)
  T* VS;          // fp32 only: [ldv][TP]
  T* ZS;          // [TP][ldz]
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

__host__ __device__ inline int imax(int a, int b) { return a > b ? a : b; }

template <class T>
__host__ __device__ inline size_t smem_bytes(int dim, int ldv, int ldz, int max_q, int nbuf,
                                             int opt_rows) {
  size_t b = align16(sizeof(PlanHead));
  b += 2 * align16(sizeof(int) * max_q) + align16(sizeof(T) * max_q);
  if (sizeof(T) == 8) b += align16(sizeof(T) * max_q);
  b += align16(sizeof(T) * opt_rows * dim);
  b += nbuf * align16(sizeof(T) * TP * dim);
  if (sizeof(T) == 4) b += align16(sizeof(T) * TP * ldv);
  b += align16(sizeof(T) * TP * ldz);
  return b;
}

// plan_base: the PlanHead (shared memory); rest: everything after it --
// shared memory as well, or for the large-dimension kernel a per-CTA slice
// of global scratch (evaluate_big_kernel)
template <class T>
__device__ inline Smem<T> carve2(unsigned char* plan_base, unsigned char* rest, const Args<T>& a) {
  Smem<T> s;
  s.P = reinterpret_cast<PlanHead*>(plan_base);
  unsigned char* base = rest;
  size_t off = 0;
  s.qsrc = reinterpret_cast<int*>(base + off);
  off += align16(sizeof(int) * a.max_q);
  s.prow = reinterpret_cast<int*>(base + off);
  off += align16(sizeof(int) * a.max_q);
  s.qo = reinterpret_cast<T*>(base + off);
  off += align16(sizeof(T) * a.max_q);
  s.cz = s.qo;
  if (sizeof(T) == 8) {
    s.cz = reinterpret_cast<T*>(base + off);
    off += align16(sizeof(T) * a.max_q);
  }
  s.opt = reinterpret_cast<T*>(base + off);
  off += align16(sizeof(T) * a.opt_rows * a.dim);
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

template <class T>
__device__ inline Smem<T> carve(unsigned char* base, const Args<T>& a) {
  return carve2<T>(base, base + align16(sizeof(PlanHead)), a);
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
template <class T, bool MT2 = false>
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
    int nj = 0;
    for (int mi = 0; mi < fn.n_members; ++mi) {
      const rb_member mm = a.members[fn.member0 + mi];
      for (int si = 0; si < mm.n_segments && nj < MAX_SEGMENTS; ++si, ++nj) {
        P.job_mem[nj] = (int8_t)mi;
        P.job_seg[nj] = (int8_t)(mm.segment0 - first.segment0 + si);
      }
    }
    P.n_jobs = nj;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nth = blockDim.x;
  for (int i = threadIdx.x; i < P.fn.n_members; i += nth) P.mem[i] = a.members[P.fn.member0 + i];
  for (int i = threadIdx.x; i < P.n_seg; i += nth) P.seg[i] = a.segments[P.seg_base + i];
  for (int i = threadIdx.x; i < P.n_grp; i += nth) P.grp[i] = a.groups[P.grp_base + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int q = 0;
    for (int g = 0; g < P.n_grp; ++g) {
      P.gq0[g] = q;
      q += round8(P.grp[g].m);
    }
    int nu = 0;                              // fp64 DMMA units, group-major per segment
    for (int si = 0; si < P.n_seg; ++si) {
      P.unit_off[si] = nu;
      const int g0 = P.seg[si].group0 - P.grp_base;
      for (int g = g0; g < g0 + P.seg[si].n_groups; ++g) P.grp_seg[g] = (int8_t)si;
      for (int g = g0; g < g0 + P.seg[si].n_groups; ++g)
        for (int mt = 0; mt < TP / 16; mt += (MT2 ? 2 : 1))
          for (int nt = 0; nt < (P.grp[g].m + 7) >> 3 && nu < MAX_UNITS; ++nt)
            P.unit[nu++] = (uint32_t)g | ((uint32_t)mt << 8) | ((uint32_t)nt << 16);
    }
    P.unit_off[P.n_seg] = nu;
    int ic = 0, vc = 0;
    for (int g = 0; g < P.n_grp; ++g) {
      P.icum[g] = ic;
      P.vcum[g] = vc;
      ic += (TP / 4) * ((P.grp[g].m + 3) >> 2);
      vc += round4(P.grp[g].m);
      const rb_segment& sg = P.seg[P.grp_seg[g]];
      P.gsc32[g] = (float)sg.scale;
      P.gpre32[g] = (float)sg.pre;
      P.gpost32[g] = (float)sg.post;
    }
    P.icum[P.n_grp] = ic;
    P.vcum[P.n_grp] = vc;
    // members with an exact-order path, decided by rb_initialize (plan_launches)
    // and carried in the device copy of the function record
    P.exact_mem = sizeof(T) == 8 ? (uint32_t)P.fn.reserved & 0xffu : 0u;
  }
  __syncthreads();
  for (int mi = 0; mi < a.opt_rows && mi < P.fn.n_members; ++mi)
    for (int j = threadIdx.x; j < a.dim; j += nth) s.opt[mi * a.dim + j] = a.values[P.mem[mi].shift + j];
  for (int mi = 0; mi < P.fn.n_members; ++mi) {
    const rb_member& mem = P.mem[mi];
    const T* o = a.values + mem.shift;
    for (int si = 0; si < mem.n_segments; ++si) {
      const rb_segment& seg = P.seg[mem.segment0 - P.seg_base + si];
      for (int gi = 0; gi < seg.n_groups; ++gi) {
        const int g = seg.group0 - P.grp_base + gi;
        const rb_group& G = P.grp[g];
        const int32_t* cols = a.index + (sizeof(T) == 8 ? G.col64 : G.col);
        const int32_t* rows = a.index + G.row;
        for (int q = threadIdx.x; q < round8(G.m); q += nth) {
          int src = 0, row = 0;
          T ov = T(0), cv = T(0);
          if (q < G.m) {
            const int pos = cols[q];
            src = mem.perm >= 0 ? a.index[mem.perm + seg.src + pos] : pos;
            ov = o[src];
            row = rows[q] + seg.src;       // chunk k's z at offset src_k (hybrid members)
            if (sizeof(T) == 8) cv = a.values[G.cz + q];     // indexed by block row q
          }
          s.qsrc[P.gq0[g] + q] = src;
          s.qo[P.gq0[g] + q] = ov;
          s.prow[P.gq0[g] + q] = row;
          if (sizeof(T) == 8) s.cz[P.gq0[g] + q] = cv;
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

// thread 0 only: warm L2 with a future tile (no shared memory needed), so
// its TMA copy is served from L2 instead of HBM
template <class T>
__device__ __forceinline__ void prefetch_tile_l2(const Args<T>& a, int64_t tile) {
  const int64_t ntiles = (a.n + TP - 1) / TP;
  if (tile >= ntiles) return;
  const uint32_t bytes = (uint32_t)(sizeof(T) * (size_t)tile_rows(a, tile) * a.dim) & ~15u;
  if (!bytes || !a.tma) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.x + tile * TP * a.dim), "r"(bytes)
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

// NaN or infinity, by the exponent bits (integer pipe, not the FP64 pipe)
__device__ __forceinline__ bool not_finite(double v) {
  return (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
}
__device__ __forceinline__ bool not_finite(float v) {
  return (__float_as_int(v) & 0x7f800000) == 0x7f800000;
}

// z value into ZS; records point p in `nf` when the value is not finite
// (kernels.py:45-49).  stage_segment masks nf with the live points.
template <bool CHECK, class T>
__device__ __forceinline__ void put_z(const Args<T>& a, const Smem<T>& s, int p, int pos, T v,
                                      uint32_t& nf) {
  s.ZS[p * a.ldz + pos] = v;
  if (CHECK && not_finite(v)) nf |= 1u << p;
}

// |x| bound below which z = R(scale (x - o) + pre) + post cannot overflow
// (|scale| <= 10, rows of R have unit norm, D < 10^6): 2^960 in float64,
// 2^100 in float32.  Tiles whose x all lie below it skip the per-z
// finiteness test, which the X scan in evaluate_kernel then proves.

// ------------------------------------------------------------ rotate fp64
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// z[p][row_r] = sum_q (scale B)[q][r] (x[p][src_q] - o_q) - cz[r]
//             = R (scale (x - o) + pre) + post   (engine.py:97-103, hybrid.py:103-114)
// with the scale folded into the pack's B fragments and pre / post into one
// constant per block row (pack.py group()), so an A element is one
// subtraction -- exactly zero at the optimum, where z is then exactly post
// as in the reference (HappyCat's |r2 - d|^0.25 would amplify any residue).
// Summation order differs from NumPy's (float64 parity is to tolerance,
// DESIGN.md section 3).
// Units = (group, 16-point m-tile, 8-row n-tile), group-major (P.unit);
// warp w owns units [w*U/NW, (w+1)*U/NW) and walks them in runs of <= NTC
// n-tiles sharing (group, m-tile), so one A fragment per k-step feeds the
// run.  Fragment layouts (PTX m16n8k4 .f64): a_i = (gid + 8i, tig),
// b = (tig, gid), c_i = (gid + 8*(i>>1), 2*tig + (i&1)).
// R (1 or 2) n-tiles of one (group, m-tile) over all k-steps: A = x - o
// gathered through the column table, B pre-swizzled from the pack.
#ifndef RB_DMMA_UNROLL
#define RB_DMMA_UNROLL 4                 // A/B: 3 -> 4 +1-2 % on float64 compositions, 2 worse
#endif
constexpr int kDmmaUnroll = RB_DMMA_UNROLL;

template <int R>
__device__ __forceinline__ void dmma_run(const double* X0, const double* X1, const int* qs,
                                         const double* qo, const double* F, int nks,
                                         double (&acc)[2][4]) {
#pragma unroll kDmmaUnroll
  for (int ks = 0; ks < nks; ++ks) {
    const int col = qs[ks * 4];
    const double o = qo[ks * 4];
    const double a0 = X0[col] - o;
    const double a1 = X1[col] - o;
    const double b0 = __ldg(F + ks * 32);
    dmma_16x8x4(acc[0], a0, a1, b0);
    if constexpr (R == 2) {
      const double b1 = __ldg(F + (nks + ks) * 32);
      dmma_16x8x4(acc[1], a0, a1, b1);
    }
  }
}

// epilogue of one m-tile: z = acc - cz, scattered to the rows' z positions;
// rows come in pairs (2 tig, 2 tig + 1), so the tables are read as pairs
template <bool CHECK>
__device__ __forceinline__ void dmma_epilogue(const Args<double>& a, const Smem<double>& s,
                                              const rb_group& G, const double (&acc)[2][4], int mt,
                                              int nt0, int run, int gid, int tig, uint32_t& nf) {
  const PlanHead& P = *s.P;
  const int g = (int)(&G - P.grp);
  const int m = G.m;
  const int* prow = s.prow + P.gq0[g];
  const double* cz = s.cz + P.gq0[g];
  const int p0 = mt * 16 + gid;
  double* Z0 = s.ZS + p0 * a.ldz;
  double* Z1 = Z0 + 8 * a.ldz;
  uint32_t e0 = 0u, e1 = 0u;                  // max exponent field per point
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int rr = (nt0 + c) * 8 + 2 * tig;
    if (c < run && rr < m) {
      const int2 pr = *reinterpret_cast<const int2*>(prow + rr);
      const double2 cc = *reinterpret_cast<const double2*>(cz + rr);
      const double z00 = acc[c][0] - cc.x, z10 = acc[c][2] - cc.x;
      Z0[pr.x] = z00;
      Z1[pr.x] = z10;
      double z01 = 0.0, z11 = 0.0;
      if (rr + 1 < m) {
        z01 = acc[c][1] - cc.y;
        z11 = acc[c][3] - cc.y;
        Z0[pr.y] = z01;
        Z1[pr.y] = z11;
      }
      if (CHECK) {
        e0 = max(e0, max((uint32_t)__double2hiint(z00), (uint32_t)__double2hiint(z01)) & 0x7ff00000u);
        e1 = max(e1, max((uint32_t)__double2hiint(z10), (uint32_t)__double2hiint(z11)) & 0x7ff00000u);
      }
    }
  }
  if (CHECK && e0 == 0x7ff00000u) nf |= 1u << p0;      // NaN or infinity (kernels.py:45-49)
  if (CHECK && e1 == 0x7ff00000u) nf |= 1u << (p0 + 8);
}

// Both m-tiles of the tile (MT2): each B fragment load feeds 2 x R
// DMMAs (the two 16-point m-tiles), halving the B traffic from L1 / L2.
#ifndef RB_DMMA_UNROLL_MT2
#define RB_DMMA_UNROLL_MT2 3            // A/B: 2 -> 3 +3 % on float64 basic functions, 4 no better
#endif
constexpr int kDmmaUnrollMt2 = RB_DMMA_UNROLL_MT2;
template <int R>
__device__ __forceinline__ void dmma_run_mt2(const double* X0, const double* X1, const double* X2,
                                             const double* X3, const int* qs, const double* qo,
                                             const double* F, int nks, double (&acc)[2][2][4]) {
#pragma unroll kDmmaUnrollMt2
  for (int ks = 0; ks < nks; ++ks) {
    const int col = qs[ks * 4];
    const double o = qo[ks * 4];
    const double b0 = __ldg(F + ks * 32);
    const double a0 = X0[col] - o, a1 = X1[col] - o;
    const double a2 = X2[col] - o, a3 = X3[col] - o;
    dmma_16x8x4(acc[0][0], a0, a1, b0);
    dmma_16x8x4(acc[1][0], a2, a3, b0);
    if constexpr (R == 2) {
      const double b1 = __ldg(F + (nks + ks) * 32);
      dmma_16x8x4(acc[0][1], a0, a1, b1);
      dmma_16x8x4(acc[1][1], a2, a3, b1);
    }
  }
}

// BIG (evaluate_big_kernel): the units of plan segments [s_first, s_end)
// are enumerated on the fly (group-major, as load_plan's table) instead of
// read from the fixed-size PlanHead table
__device__ __forceinline__ uint32_t unit_at(const PlanHead& P, int g, int u) {
  for (;;) {
    const int cnt = (TP / 16) * ((P.grp[g].m + 7) >> 3);
    if (u < cnt) break;
    u -= cnt;
    ++g;
  }
  const int ntn = (P.grp[g].m + 7) >> 3;
  return (uint32_t)g | ((uint32_t)(u / ntn) << 8) | ((uint32_t)(u % ntn) << 16);
}

template <int NW, bool CHECK, bool MT2, bool BIG = false>
__device__ inline uint32_t rotate_f64(const Args<double>& a, const Smem<double>& s, int s_first,
                                      int s_end, int warp) {
  const PlanHead& P = *s.P;
  const int lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  int u0 = 0, total = 0;
  const int gb = P.seg[s_first].group0 - P.grp_base;
  if constexpr (BIG) {
    const int ge = P.seg[s_end - 1].group0 + P.seg[s_end - 1].n_groups - P.grp_base;
    for (int g = gb; g < ge; ++g) total += (TP / 16) * ((P.grp[g].m + 7) >> 3);
  } else {
    u0 = P.unit_off[s_first];
    total = P.unit_off[s_end] - u0;
  }
  const int end = (warp + 1) * total / NW;
  uint32_t nf = 0u;
  for (int u = warp * total / NW; u < end;) {
    const uint32_t ud = BIG ? unit_at(P, gb, u) : P.unit[u0 + u];
    const int g = ud & 0xff, mt = (ud >> 8) & 0xff, nt0 = ud >> 16;
    const rb_group& G = P.grp[g];
    const int m = G.m, ntn = (m + 7) >> 3, nks = (m + 3) >> 2;
    const int run = min(min(NTC, ntn - nt0), end - u);
    const double* F = a.values + G.frag + (size_t)nt0 * nks * 32 + lane;
    const int* qs = s.qsrc + P.gq0[g] + tig;    // padded columns read x[.][0] * B = 0
    const double* qo = s.qo + P.gq0[g] + tig;
    const double* X0 = s.XS + (mt * 16 + gid) * a.dim;
    const double* X1 = X0 + 8 * a.dim;
    if constexpr (MT2) {
    double acc2[2][2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc2[i][j][k] = 0.0;
    if (run == 2) dmma_run_mt2<2>(X0, X1, X0 + 16 * a.dim, X1 + 16 * a.dim, qs, qo, F, nks, acc2);
    else dmma_run_mt2<1>(X0, X1, X0 + 16 * a.dim, X1 + 16 * a.dim, qs, qo, F, nks, acc2);
#pragma unroll
    for (int mh = 0; mh < 2; ++mh) dmma_epilogue<CHECK>(a, s, G, acc2[mh], mt + mh, nt0, run, gid, tig, nf);
    } else {
    double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    // the run length is warp-uniform: unpredicated mma.sync in both loops
    if (run == 2) dmma_run<2>(X0, X1, qs, qo, F, nks, acc);
    else dmma_run<1>(X0, X1, qs, qo, F, nks, acc);
    dmma_epilogue<CHECK>(a, s, G, acc, mt, nt0, run, gid, tig, nf);
    }
    u += run;
  }
  return nf;
}

// z of plan segments [s_first, s_end) (the chunks of one member, side by side)
template <bool CHECK, bool MT2 = false, bool BIG = false>
__device__ inline uint32_t rotate(const Args<double>& a, const Smem<double>& s, int s_first,
                                  int s_end) {
  return rotate_f64<NWARPS, CHECK, MT2, BIG>(a, s, s_first, s_end, threadIdx.x >> 5);
}

// ------------------------------------------------------------ rotate fp32
// Exact NumPy order (transforms.py:42-48): rounded products, per-slot
// accumulation in q-order, slot fold ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)),
// ordered tail.  VS is [q][TP] with point p at word vslot(p); B rows are
// 4-padded (one float4 per q).  A rotate item owns points pq + 8i (i < 4),
// one float4 of V: the 8 items of a warp's z store then cover 4 residues of
// p mod 4, i.e. 4 distinct banks at ldz = 8 (mod 32) (2-way instead of 8-way
// conflicts; the pack orders block rows so the warp's 4 rows differ mod 8).
__device__ __forceinline__ int vslot(int p) { return (p & 7) * 4 + (p >> 3); }

// gather: V[vq + q][p] = scale*(x[p][src_q] - o_q) + pre   (engine.py:97-100)
// for the groups of plan segments [s_first, s_end).  Every x of the tile is
// read here once per member, so it also returns the max |x| bit pattern over
// the valid points (the X scan of evaluate_kernel, folded in; nv = 0: skip).
__device__ inline uint32_t gather_v(const Args<float>& a, const Smem<float>& s, int s_first,
                                    int s_end, int nv) {
  const PlanHead& P = *s.P;
  const int g0 = P.seg[s_first].group0 - P.grp_base;
  const int ng = P.seg[s_end - 1].group0 + P.seg[s_end - 1].n_groups - P.seg[s_first].group0;
  uint32_t mx = 0u;
  int vq = 0;
  for (int g = 0; g < ng; ++g) {
    const float scale = P.gsc32[g0 + g], pre = P.gpre32[g0 + g];
    const int kp = round4(P.grp[g0 + g].m);
    const int* qs = s.qsrc + P.gq0[g0 + g];
    const float* qo = s.qo + P.gq0[g0 + g];
    // item (q, p0): points p0 + 8i (i < 4), which vslot places side by side:
    // one float4 store, one column-table read for four elements
    for (int e = threadIdx.x; e < (TP / 4) * kp; e += NT) {
      const int q = e >> 3, p0 = e & 7;
      const int src = qs[q];
      const float o = qo[q];
      float4 v4;
      float* v = reinterpret_cast<float*>(&v4);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int p = p0 + 8 * i;
        const float x = s.XS[p * a.dim + src];
        if (p < nv) mx = max(mx, __float_as_uint(x) & 0x7fffffffu);
        float t = scale * (x - o);
        if (pre != 0.0f) t = t + pre;
        v[i] = t;
      }
      *reinterpret_cast<float4*>(s.VS + (vq + q) * TP + p0 * 4) = v4;
    }
    vq += kp;
  }
  return mx;
}

// One pairwise leaf of the float32 exact-order rotate for RR block rows and
// the 4 points of a float4 V column: slot s walks q in [qb[s], qb[s+1]) with
// a rounded product and a rounded add (NumPy's r[s] += a[i] per slot), the
// 8 slots fold as ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)) and the tail adds in
// order.  bp: B row qb[0] (rows r0.., stride m4).
//
// Packed FP32 (sm_100 FFMA2/FADD2): a pair of rows per register pair, the
// point's v broadcast.  The product is fma(v, b, -0) -- bit-identical to
// the rounded product -- with -0 taken from the kernel arguments: ptxas
// contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 (12.9, even with
// --fmad=false), which it cannot do to an fma with an unknown addend.
template <int RR>
__device__ __forceinline__ void f32_leaf(const float4* Vq, const float* bp, int bstride,
                                         const int (&qb)[10], float nz, float (&t0)[4][RR]) {
  constexpr int vstride = TP / 4;
  constexpr int RP = RR / 2;                     // row pairs
  const float2 Z = make_float2(nz, nz);
  float2 u0[4][RP], u1[4][RP], u2[4][RP], acc[4][RP];
  auto load_b = [&](const float* b, float2 (&bb)[RP]) {
    if constexpr (RR == 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(b));
      bb[0] = make_float2(v.x, v.y); bb[1] = make_float2(v.z, v.w);
    } else {
      bb[0] = __ldg(reinterpret_cast<const float2*>(b));
    }
  };
#pragma unroll
  for (int sl = 0; sl < 8; ++sl) {
    // a slot starts from its first product (NumPy's r[k] = a[k]), not 0 + a[k]
    int q = qb[sl];
    if (q < qb[sl + 1]) {
      const float4 v = Vq[q * vstride];
      float2 bb[RP];
      load_b(bp, bb);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < RP; ++j) acc[i][j] = __ffma2_rn(make_float2(vv[i], vv[i]), bb[j], Z);
      ++q;
      bp += bstride;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < RP; ++j) acc[i][j] = make_float2(0.0f, 0.0f);
    }
#pragma unroll kF32Unroll
    for (; q < qb[sl + 1]; ++q, bp += bstride) {
      const float4 v = Vq[q * vstride];
      float2 bb[RP];
      load_b(bp, bb);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < RP; ++j)
          acc[i][j] = __fadd2_rn(acc[i][j], __ffma2_rn(make_float2(vv[i], vv[i]), bb[j], Z));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const float2 x = acc[i][j];
        switch (sl) {
          case 0: u0[i][j] = x; break;
          case 1: u0[i][j] = __fadd2_rn(u0[i][j], x); break;
          case 2: u1[i][j] = x; break;
          case 3: u1[i][j] = __fadd2_rn(u1[i][j], x); u0[i][j] = __fadd2_rn(u0[i][j], u1[i][j]); break;
          case 4: u1[i][j] = x; break;
          case 5: u1[i][j] = __fadd2_rn(u1[i][j], x); break;
          case 6: u2[i][j] = x; break;
          default:
            u2[i][j] = __fadd2_rn(u2[i][j], x);
            u1[i][j] = __fadd2_rn(u1[i][j], u2[i][j]);
            u0[i][j] = __fadd2_rn(u0[i][j], u1[i][j]);
        }
      }
  }
  for (int q = qb[8]; q < qb[9]; ++q, bp += bstride) {
    const float4 v = Vq[q * vstride];
    const float vv[4] = {v.x, v.y, v.z, v.w};
    float2 bb[RP];
    load_b(bp, bb);
#pragma unroll
    for (int j = 0; j < RP; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        u0[i][j] = __fadd2_rn(u0[i][j], __ffma2_rn(make_float2(vv[i], vv[i]), bb[j], Z));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < RP; ++j) {
      t0[i][2 * j] = u0[i][j].x;
      t0[i][2 * j + 1] = u0[i][j].y;
    }
}

// the V tile is in place (gather_v + barrier)
template <bool CHECK, bool MT2 = false, bool BIG = false>
__device__ inline uint32_t rotate(const Args<float>& a, const Smem<float>& s, int s_first,
                                  int s_end) {
  const PlanHead& P = *s.P;
  const int g0 = P.seg[s_first].group0 - P.grp_base;
  const int ng = P.seg[s_end - 1].group0 + P.seg[s_end - 1].n_groups - P.seg[s_first].group0;
  const int i0 = P.icum[g0];
  const int total = P.icum[g0 + ng] - i0;
  uint32_t nf = 0u;
  for (int t = threadIdx.x; t < total; t += NT) {
    int g = g0;
    while (P.icum[g + 1] <= i0 + t) ++g;
    const int rem = i0 + t - P.icum[g], vq = P.vcum[g] - P.vcum[g0];
    const rb_group& G = P.grp[g];
    const float post = P.gpost32[g];
    const int pq = rem % (TP / 4), rq = rem / (TP / 4);
    const int m = G.m, m4 = round4(m);
    const int* prow = s.prow + P.gq0[g];
    // column q: V row vq + q (4 points, one float4) and B row q
    const float4* Vq = reinterpret_cast<const float4*>(s.VS + vq * TP + pq * 4);
    if (G.leaf < 0) {                          // one pairwise leaf (segment rows <= 128)
      constexpr int RR = RB_F32_ROWS;
      int qb[10];
#pragma unroll
      for (int k = 0; k < 10; ++k) qb[k] = G.qb[k];
#pragma unroll 1
      for (int pass = 0; pass < 4 / RR; ++pass) {
        const int r0 = rq * 4 + pass * RR;
        if (r0 >= m) break;
        float z[4][RR];
        f32_leaf<RR>(Vq, a.values + G.mat + r0, m4, qb, a.neg_zero, z);
#pragma unroll
        for (int j = 0; j < RR; ++j) {
          if (r0 + j >= m) break;
          const int row = prow[r0 + j];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            put_z<CHECK>(a, s, pq + 8 * i, row, post != 0.0f ? __fadd_rn(z[i][j], post) : z[i][j], nf);
        }
      }
    } else {
      // rows longer than 128: NumPy's pairwise tree over the leaves, run as
      // a post-order program (pack.py pairwise_program): each leaf's sum is
      // pushed, then the given number of (left + right) additions pop the
      // stack.  Stack slots are registers (static indices under sp tests).
      constexpr int RR = 2;
      constexpr int SD = 4;                    // pack.py EXACT_ORDER_STACK
      const int* L = a.index + G.leaf;
      const int nl = __ldg(L);
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const int r0 = rq * 4 + pass * RR;
        if (r0 >= m) break;
        const float* B = a.values + G.mat + r0;
        float st[SD][4][RR];
        int sp = 0;
#pragma unroll 1
        for (int lf = 0; lf < nl; ++lf) {
          const int* E = L + 1 + 11 * lf;
          int qb[10];
#pragma unroll
          for (int k = 0; k < 10; ++k) qb[k] = __ldg(E + k);
          float z[4][RR];
          f32_leaf<RR>(Vq, B + qb[0] * m4, m4, qb, a.neg_zero, z);
#pragma unroll
          for (int d = 0; d < SD; ++d)
            if (d == sp) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < RR; ++j) st[d][i][j] = z[i][j];
            }
          ++sp;
          for (int c = __ldg(E + 10); c > 0; --c) {
#pragma unroll
            for (int d = 1; d < SD; ++d)
              if (d == sp - 1) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                  for (int j = 0; j < RR; ++j) st[d - 1][i][j] = __fadd_rn(st[d - 1][i][j], st[d][i][j]);
              }
            --sp;
          }
        }
#pragma unroll
        for (int j = 0; j < RR; ++j) {
          if (r0 + j >= m) break;
          const int row = prow[r0 + j];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float zz = st[0][i][j];
            put_z<CHECK>(a, s, pq + 8 * i, row, post != 0.0f ? __fadd_rn(zz, post) : zz, nf);
          }
        }
      }
    }
  }
  return nf;
}

// ------------------------------------------ float64 exact-order fallback
// One pairwise leaf for RR block rows and the item's 4 points in NumPy's
// order (f32_leaf's slot walk in double, DMUL + DADD, each rounded): slot s
// walks q in [qb[s], qb[s+1]), the slots fold ((s0+s1)+(s2+s3))+((s4+s5)+
// (s6+s7)), the tail adds in order.  load_v(q, v[4]) supplies the column.
template <int RR, class VL>
__device__ __forceinline__ void f64_leaf(VL& load_v, const double* bp, int bstride,
                                         const int (&qb)[10], double (&t0)[4][RR]) {
  double u0[4][RR], u1[4][RR], u2[4][RR], acc[4][RR];
#pragma unroll
  for (int sl = 0; sl < 8; ++sl) {
    int q = qb[sl];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < RR; ++j) acc[i][j] = 0.0;
    if (q < qb[sl + 1]) {                 // NumPy's r[k] = a[k]: the slot's first product
      double vv[4];
      load_v(q, vv);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < RR; ++j) acc[i][j] = __dmul_rn(vv[i], __ldg(bp + j));
      ++q;
      bp += bstride;
    }
#pragma unroll 1
    for (; q < qb[sl + 1]; ++q, bp += bstride) {
      double vv[4];
      load_v(q, vv);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < RR; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(vv[i], __ldg(bp + j)));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < RR; ++j) {
        const double x = acc[i][j];
        switch (sl) {
          case 0: u0[i][j] = x; break;
          case 1: u0[i][j] = __dadd_rn(u0[i][j], x); break;
          case 2: u1[i][j] = x; break;
          case 3: u1[i][j] = __dadd_rn(u1[i][j], x); u0[i][j] = __dadd_rn(u0[i][j], u1[i][j]); break;
          case 4: u1[i][j] = x; break;
          case 5: u1[i][j] = __dadd_rn(u1[i][j], x); break;
          case 6: u2[i][j] = x; break;
          default:
            u2[i][j] = __dadd_rn(u2[i][j], x);
            u1[i][j] = __dadd_rn(u1[i][j], u2[i][j]);
            u0[i][j] = __dadd_rn(u0[i][j], u1[i][j]);
        }
      }
  }
#pragma unroll 1
  for (int q = qb[8]; q < qb[9]; ++q, bp += bstride) {
    double vv[4];
    load_v(q, vv);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < RR; ++j) u0[i][j] = __dadd_rn(u0[i][j], __dmul_rn(vv[i], __ldg(bp + j)));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < RR; ++j) t0[i][j] = u0[i][j];
}

// z of member `mem` (plan segments [s_first, s_end)) in NumPy's exact order:
// v = scale * (x - o)[perm] (+ pre) recomputed from the X tile per column
// (engine.py:97-100, hybrid.py:103-110; no V tile, so the rare fallback
// costs no shared memory), z = matvec(R, v) (transforms.py:42-48) in q-order
// with the block in the pack's `mat` layout, + post.  Items as in the
// float32 rotate: 4 points (pq + 8i) x one block row per pass.
template <bool CHECK>
__device__ __noinline__ uint32_t rotate_exact_f64(const Args<double>& a, const Smem<double>& s,
                                     const rb_member& mem, int s_first, int s_end) {
  const PlanHead& P = *s.P;
  const int g0 = P.seg[s_first].group0 - P.grp_base;
  const int ng = P.seg[s_end - 1].group0 + P.seg[s_end - 1].n_groups - P.seg[s_first].group0;
  int total = 0;
  for (int g = 0; g < ng; ++g) total += (TP / 4) * ((P.grp[g0 + g].m + 3) >> 2);
  const double* o = a.values + mem.shift;
  uint32_t nf = 0u;
  for (int t = threadIdx.x; t < total; t += NT) {
    int g = g0, rem = t;
    for (;;) {
      const int cnt = (TP / 4) * ((P.grp[g].m + 3) >> 2);
      if (rem < cnt) break;
      rem -= cnt;
      ++g;
    }
    const rb_group& G = P.grp[g];
    const rb_segment& seg = P.seg[P.grp_seg[g]];
    const double scale = seg.scale, pre = seg.pre, post = seg.post;
    const int pq = rem % (TP / 4), rq = rem / (TP / 4);
    const int m = G.m, m4 = round4(m);
    const int32_t* col = a.index + G.col;
    const int32_t* perm = mem.perm >= 0 ? a.index + mem.perm + seg.src : nullptr;
    const double* X0 = s.XS + pq * a.dim;
    auto load_v = [&](int q, double (&vv)[4]) {
      const int pos = __ldg(col + q);
      const int src = perm ? __ldg(perm + pos) : pos;
      const double ov = __ldg(o + src);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double v = __dmul_rn(scale, __dsub_rn(X0[8 * i * a.dim + src], ov));
        if (pre != 0.0) v = __dadd_rn(v, pre);
        vv[i] = v;
      }
    };
    const int* prow = a.index + G.row;
    auto store = [&](int r, const double (&z)[4]) {
      const int row = __ldg(prow + r) + seg.src;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        put_z<CHECK>(a, s, pq + 8 * i, row, post != 0.0 ? __dadd_rn(z[i], post) : z[i], nf);
    };
#pragma unroll 1
    for (int r = rq * 4; r < min(rq * 4 + 4, m); ++r) {
      const double* B = a.values + G.mat + r;
      double z[4];
      if (G.leaf < 0) {                         // one pairwise leaf (rows <= 128)
        int qb[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) qb[k] = G.qb[k];
        double zz[4][1];
        f64_leaf<1>(load_v, B, m4, qb, zz);
#pragma unroll
        for (int i = 0; i < 4; ++i) z[i] = zz[i][0];
      } else {                                  // NumPy's pairwise tree (pack.py pairwise_program)
        constexpr int SD = 4;
        const int* L = a.index + G.leaf;
        const int nl = __ldg(L);
        double st[SD][4];
        int sp = 0;
#pragma unroll 1
        for (int lf = 0; lf < nl; ++lf) {
          const int* E = L + 1 + 11 * lf;
          int qb[10];
#pragma unroll
          for (int k = 0; k < 10; ++k) qb[k] = __ldg(E + k);
          double zz[4][1];
          f64_leaf<1>(load_v, B + qb[0] * m4, m4, qb, zz);
#pragma unroll
          for (int d = 0; d < SD; ++d)
            if (d == sp) {
#pragma unroll
              for (int i = 0; i < 4; ++i) st[d][i] = zz[i][0];
            }
          ++sp;
          for (int c = __ldg(E + 10); c > 0; --c) {
#pragma unroll
            for (int d = 1; d < SD; ++d)
              if (d == sp - 1) {
#pragma unroll
                for (int i = 0; i < 4; ++i) st[d - 1][i] = __dadd_rn(st[d - 1][i], st[d][i]);
              }
            --sp;
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) z[i] = st[0][i];
      }
      store(r, z);
    }
  }
  return nf;
}

// ------------------------------------------------------------ tile state
// The tile being evaluated, tracked identically by every thread of the CTA.
struct TileCtx {
  int64_t tile;
  int nv;             // valid rows
  uint32_t phase;     // parity of mbar[0] (fp64 loads / refetches)
  bool check_z;       // some valid x of the tile is huge or not finite: test every z
  bool scanned;       // the tile's X scan is done (fp32: folded into the first gather)
  uint32_t live;      // points whose z of the current member are checked
  bool next_issued;   // single-buffered: the next tile's X copy is already in flight
};

// X tile into XS (buffer A for fp64); all threads; ends with a barrier.
// The caller has passed a barrier since the last read of the buffer.
template <class T>
__device__ void fetch_x(const Args<T>& a, const Smem<T>& s, TileCtx& t) {
  PlanHead& P = *s.P;
  if (tile_is_bulk(a, t.nv)) {
    if (threadIdx.x == 0 && !t.next_issued) issue_tile(a, s.XS, &P.mbar[0], t.tile, t.nv);
    t.next_issued = false;
    wait_tile(&P.mbar[0], t.phase);
    t.phase ^= 1u;
  } else {
    const T* src = a.x + t.tile * TP * a.dim;
    for (int e = threadIdx.x; e < t.nv * a.dim; e += NT) s.XS[e] = src[e];
  }
  __syncthreads();
}

// Single-buffered X: once the tile's last member is staged (every read of
// XS is behind the staging barrier) the next tile's copy is started, so it
// lands while this tile's kernels run.  All threads call it (uniform).
template <class T>
__device__ __forceinline__ void issue_next_x(const Args<T>& a, const Smem<T>& s, TileCtx& t) {
  if (a.nbuf != 1) return;
  const int64_t ntiles = (a.n + TP - 1) / TP;
  const int64_t nxt = t.tile + gridDim.x;
  if (nxt >= ntiles || !tile_is_bulk(a, tile_rows(a, nxt))) return;
  if (threadIdx.x == 0) issue_tile(a, s.XS, &s.P->mbar[0], nxt, tile_rows(a, nxt));
  t.next_issued = true;
}

// ----------------------------------------------------------- one member
// z of every segment of one member for all points of the tile, then one
// barrier: the chunks of a hybrid member are rotated in the same pass and
// their z laid side by side (chunk k at offset src_k, pack.py).  Returns
// where z lives (row stride ldz).
// EXACT (float64, fixup_kernel): members with an exact-order path
// (P.exact_mem) rotate in NumPy's order instead of by DMMA.
template <class T, bool EXACT = false, bool MT2 = false, bool BIG = false>
__device__ const T* stage_member(const Args<T>& a, const Smem<T>& s, const rb_member& mem,
                                 TileCtx& t) {
  const PlanHead& P = *s.P;
  uint32_t nf = 0u;
  const int s_first = mem.segment0 - P.seg_base, s_end = s_first + mem.n_segments;
  const rb_segment& seg = P.seg[s_first];
  if (seg.n_groups == 0) {                 // shift-only ids 10 and 15 (engine.py:96-104)
    T* zw = s.ZS;
    const T* o = a.values + mem.shift;
    const int32_t* perm = mem.perm >= 0 ? a.index + mem.perm + seg.src : nullptr;
    const T scale = (T)seg.scale, pre = (T)seg.pre, post = (T)seg.post;
    const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
    for (int j = l8; j < seg.d; j += 8) {
      const int src = perm ? perm[j] : j;
      T v = scale * (s.XS[p * a.dim + src] - o[src]);
      if (pre != T(0)) v = v + pre;
      if (post != T(0)) v = v + post;
      zw[p * a.ldz + j] = v;
      if (t.check_z && not_finite(v)) nf |= 1u << p;
    }
  } else {
    if constexpr (sizeof(T) == 4) {
      const uint32_t mx = gather_v(a, s, s_first, s_end, t.scanned ? 0 : t.nv);
      if (!t.scanned) {                    // X scan of this tile (see evaluate_kernel)
        if (mx >= 0x7f800000u) raise_flag(a);
        t.check_z = __syncthreads_or(mx >= 0x71800000u) != 0;
        t.scanned = true;
      } else {
        __syncthreads();
      }
    }
    if constexpr (EXACT && sizeof(T) == 8) {
      if ((P.exact_mem >> (int)(&mem - P.mem)) & 1u)
        nf = t.check_z ? rotate_exact_f64<true>(a, s, mem, s_first, s_end)
                       : rotate_exact_f64<false>(a, s, mem, s_first, s_end);
      else
        nf = t.check_z ? rotate<true, false, BIG>(a, s, s_first, s_end)
                       : rotate<false, false, BIG>(a, s, s_first, s_end);
    } else {
      nf = t.check_z ? rotate<true, MT2>(a, s, s_first, s_end) : rotate<false, MT2>(a, s, s_first, s_end);
    }
  }
  if (nf & t.live) raise_flag(a);
  __syncthreads();
  return s.ZS;
}

// Value of one member (basic function, hybrid, or composition member) for
// the calling lane's point: one staging pass, then the chunk kernels in
// order (hybrid.py:105-115: 0 + K_0 + K_1 + ...).
// KID: basic kernel id, GENERIC (run-time kernel dispatch), or FIXUP (the
// exact-order re-evaluation of marked points, fixup_kernel).  `ill`: float64
// HappyCat / HGBat members of the main kernels set it when the point's value
// needs the exact-order z (mark_ill, rb_kernels.cuh).
template <class T, int KID>
__device__ T member_value(const Args<T>& a, const Smem<T>& s, const rb_member& mem, TileCtx& t,
                          bool last, bool* ill = nullptr) {
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const PlanHead& P = *s.P;
  RB_PHASE_MARK(c0);
  const T* zb = stage_member<T, exact_mode(KID), mt2_kernel<KID>(), KID == BIGDIM>(a, s, mem, t);
  if (last) issue_next_x(a, s, t);
  RB_PHASE_MARK(c1);
  // compile-time: can this kernel meet a float64 exact64 member at all?
  constexpr bool kMark = sizeof(T) == 8 && (KID == GENERIC || (KID >= 0 && exact64_kernel(KID)));
  bool* mark = (kMark && ((P.exact_mem >> (int)(&mem - P.mem)) & 1u)) ? ill : nullptr;
  T total = T(0);
  for (int si = 0; si < mem.n_segments; ++si) {
    const rb_segment& seg = P.seg[mem.segment0 - P.seg_base + si];
    const Pt<T> pt{zb + p * a.ldz + seg.src, seg.d, l8, a.values + seg.ctab, mark};
    T v;
    if constexpr (KID >= 0) v = kernel_value_k<T, KID>(pt);
    else v = kernel_value<T, exact_mode(KID)>(seg.kernel, pt);
    total = (si == 0) ? v : total + v;
  }
  __syncthreads();                      // z is rewritten by the next member / tile
  RB_PHASE_MARK(c2);
  RB_PHASE_ADD(1, c1 - c0);
  RB_PHASE_ADD(2, c2 - c1);
  return total;
}

// composition.py:114-141: the normalised weights om[k] of the calling
// lane's point (row x of the X tile) from its squared distances to every
// member optimum: one-hot on an optimum (d2 < 1e-24), uniform if all
// weights underflow.
// NM > 0: member count known at compile time (function-specialised kernels).
template <class T, int NM = 0>
__device__ __forceinline__ void composition_weights(const Args<T>& a, const PlanHead& P, const T* x,
                                                    const T* opt, int l8, T (&om)[MAX_MEMBERS]) {
  const int nm = NM > 0 ? NM : P.fn.n_members;
  const int dim = a.dim;
  T d2[MAX_MEMBERS];
#pragma unroll
  for (int k = 0; k < MAX_MEMBERS; ++k) {
    d2[k] = T(0);
    om[k] = T(0);
  }
  if (dim <= 128) {
    // every member's sum((x - o)**2) in one pass over x (5 independent
    // chains per lane), in pw8's single-leaf order: lane k takes j = k (mod 8)
    // below the last multiple of 8, xor butterfly, then the tail in order
    const int main_len = (sizeof(T) == 8 || dim < 8) ? (sizeof(T) == 8 ? dim : 0) : dim - (dim & 7);
    T r[MAX_MEMBERS];
#pragma unroll
    for (int k = 0; k < MAX_MEMBERS; ++k) r[k] = T(0);
    for (int j = l8; j < main_len; j += 8) {
      const T xj = x[j];
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k)
        if (k < nm) {
          const T u = xj - opt[k * dim + j];
          r[k] = r[k] + u * u;
        }
    }
#pragma unroll
    for (int k = 0; k < MAX_MEMBERS; ++k) {
      if (main_len) {
        r[k] = r[k] + __shfl_xor_sync(RB_FULL, r[k], 1, 8);
        r[k] = r[k] + __shfl_xor_sync(RB_FULL, r[k], 2, 8);
        r[k] = r[k] + __shfl_xor_sync(RB_FULL, r[k], 4, 8);
      }
      const int tail = dim - main_len;
      if (tail) {
        T v = T(0);
        if (k < nm && l8 < tail) {
          const T u = x[main_len + l8] - opt[k * dim + main_len + l8];
          v = u * u;
        }
        for (int q = 0; q < tail; ++q) r[k] = r[k] + __shfl_sync(RB_FULL, v, q, 8);
      }
      d2[k] = k < nm ? r[k] : T(0);
    }
  } else {
#pragma unroll
    for (int k = 0; k < MAX_MEMBERS; ++k)
      if (k < nm) {
        const T* o = opt + k * dim;
        d2[k] = pw8<T>(0, dim, [&](int j) { const T u = x[j] - o[j]; return u * u; }, l8);
      }
  }
  T mn = d2[0];
  int am = 0;
#pragma unroll
  for (int k = 1; k < MAX_MEMBERS; ++k)
    if (k < nm && d2[k] < mn) { mn = d2[k]; am = k; }
  // lane k of the point computes member k's Gaussian weight, then all lanes
  // gather them (the 8 lanes would otherwise repeat 5 pow/exp each); done
  // before the branch below: the points of a warp may take different ones
  T dk = d2[0], sgk = (T)P.mem[0].sigma;
#pragma unroll
  for (int k = 1; k < MAX_MEMBERS; ++k)
    if (l8 == k && k < nm) { dk = d2[k]; sgk = (T)P.mem[k].sigma; }
  // d2 ** -0.5 and the Gaussian factor, to tolerance in both precisions: the
  // weights enter the value linearly (omega * (lambda G + bias)), so an ulp
  // in w is an ulp-level relative change of the value (float32: rsqrtf and
  // expf on the FP32 / XU pipes, not NumPy's SVML powf and a double exp)
#if RB_F32_FAST_WEIGHTS
  T ih, wk;
  if constexpr (sizeof(T) == 8) {
    ih = (T)::rsqrt((double)dk);
    wk = ih * M<T>::exp(-dk / (C<T>(2.0 * dim) * (sgk * sgk)));
  } else {
    ih = ::rsqrtf((float)dk);
    wk = ih * ::expf(-dk / (C<T>(2.0 * dim) * (sgk * sgk)));
  }
#else
  const T ih = sizeof(T) == 8 ? (T)::rsqrt((double)dk) : apow<T>(dk, C<T>(-0.5));
  const T wk = ih * M<T>::exp(-dk / (C<T>(2.0 * dim) * (sgk * sgk)));
#endif
  T w[MAX_MEMBERS];
#pragma unroll
  for (int k = 0; k < MAX_MEMBERS; ++k) w[k] = __shfl_sync(RB_FULL, wk, k, 8);
  if (mn < C<T>(1.0000000000000002e-24)) {          // 1e-12**2: on an optimum
#pragma unroll
    for (int k = 0; k < MAX_MEMBERS; ++k) om[k] = (k == am) ? T(1) : T(0);
  } else {
    T tot = T(0);
#pragma unroll
    for (int k = 0; k < MAX_MEMBERS; ++k)
      if (k < nm) tot = tot + w[k];
    // w / tot per member: a reciprocal 1 / tot overflows when the weights are
    // subnormal (float32 exp of a large negative argument) and 0 * inf = NaN
#pragma unroll
    for (int k = 0; k < MAX_MEMBERS; ++k)
      if (k < nm) om[k] = (tot == T(0)) ? C<T>(1.0 / nm) : w[k] / tot;
  }
}

// composition.py:114-166 for the calling lane's point: weights from the
// squared distances to every member optimum (X tile in XS), then the
// sigma-weighted, biased member values, skipping zero weights.
template <class T, int MODE = GENERIC>
__device__ T composition_value(const Args<T>& a, const Smem<T>& s, TileCtx& t, bool valid,
                               bool* ill = nullptr) {
  PlanHead& P = *s.P;
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int nm = P.fn.n_members;
  T om[MAX_MEMBERS];
  composition_weights<T>(a, P, s.XS + p * a.dim, s.opt, l8, om);
  // composition.py:157-166: zero weights are skipped (and not checked):
  // member k runs for the tile's points with a nonzero weight (P.livek[k],
  // zeroed at the tile start) and is skipped when there are none
  if (l8 == 0 && valid) {
#pragma unroll
    for (int k = 0; k < MAX_MEMBERS; ++k)
      if (k < nm && om[k] != T(0)) atomicOr(&P.livek[k], 1u << p);
  }
  __syncthreads();
  T total = T(0);
#pragma unroll 1
  for (int k = 0; k < nm; ++k) {
    T omk = T(0);
#pragma unroll
    for (int kk = 0; kk < MAX_MEMBERS; ++kk)
      if (kk == k) omk = om[kk];
    t.live = P.livek[k];
    if (!t.live) continue;
    const rb_member& mem = P.mem[k];
    const T g = member_value<T, MODE>(a, s, mem, t, !exact_mode(MODE) && k == nm - 1, ill);
    if (omk != T(0)) total = total + omk * ((T)mem.height * g + (T)mem.bias);
  }
  return total;
}

// Function-specialised hybrids / compositions (rb_fnspec.cuh), kernel ids
// SPEC_BASE + fid.
constexpr int SPEC_BASE = 100;
template <class T, int FID>
__device__ T spec_value(const Args<T>& a, const Smem<T>& s, TileCtx& t, bool valid, bool* ill);

// Resident CTAs per SM the register budget is sized for.
template <class T, int KID>
constexpr int min_blocks() {
  return sizeof(T) == 8 ? RB_MIN_BLOCKS_F64 : RB_MIN_BLOCKS_F32;
}

// Plan images: a function's shared-memory plan (PlanHead, the per-column and
// per-row tables, composition optima: everything carve() places before the
// X tile) is built once per engine and precision on the device
// (plan_image_kernel, rb_initialize) and stored behind the function table;
// the device copy of the function record carries its offset (bits 8+ of
// `reserved`, 16-byte units from the table start).  Every CTA then copies
// it in one coalesced pass instead of walking the descriptors through
// dependent global loads (small batches: launch latency).  The kernel
// arguments are unchanged (Args stays at 128 bytes).
template <class T>
__device__ __forceinline__ size_t plan_bytes(const Smem<T>& s) {
  return (size_t)(reinterpret_cast<const unsigned char*>(s.XB[0]) -
                  reinterpret_cast<const unsigned char*>(s.P));
}

template <class T, bool MT2>
__device__ __forceinline__ void enter_plan(const Args<T>& a, const Smem<T>& s) {
  const uint32_t img = (uint32_t)a.fns[a.fn].reserved >> 8;
  if (img == 0u) {
    load_plan<T, MT2>(a, s);
    return;
  }
  const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned char*>(a.fns) +
                                                    (size_t)img * 16);
  uint4* dst = reinterpret_cast<uint4*>(s.P);
  const int n16 = (int)(plan_bytes(s) / 16);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
  __syncthreads();
  if (threadIdx.x == 0) {                  // barriers are objects, not bytes: init afresh
    PlanHead& P = *s.P;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

template <class T, bool MT2>
__global__ void __launch_bounds__(NT, 1) plan_image_kernel(const Args<T> a, uint4* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Smem<T> s = carve<T>(smem_raw, a);
  load_plan<T, MT2>(a, s);
  const uint4* src = reinterpret_cast<const uint4*>(s.P);
  const int n16 = (int)(plan_bytes(s) / 16);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) out[i] = src[i];
}

template <class T, int KID>
__global__ void __launch_bounds__(NT, (min_blocks<T, KID>()))
    evaluate_kernel(const Args<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Smem<T> s = carve<T>(smem_raw, a);
  enter_plan<T, mt2_kernel<KID>()>(a, s);
  PlanHead& P = *s.P;
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int64_t ntiles = (a.n + TP - 1) / TP;
  TileCtx t{0, 0, 0u, false, false, 0u, false};
  uint32_t phase1 = 0u;
  const int64_t first = blockIdx.x;
  const bool f64 = sizeof(T) == 8;
  if (!f64 && a.nbuf == 2 && threadIdx.x == 0 && first < ntiles &&
      tile_is_bulk(a, tile_rows(a, first)))
    issue_tile(a, s.XB[0], &P.mbar[0], first, tile_rows(a, first));

  int it = 0;
  bool cta_marked = false;            // thread 0: mark_fixup already done by this CTA
  for (int64_t tile = first; tile < ntiles; tile += gridDim.x, ++it) {
    const int b = (!f64 && a.nbuf == 2) ? (it & 1) : 0;
    Smem<T> st = s;
    st.XS = b ? s.XB[1] : s.XB[0];
    RB_PHASE_MARK(c_tile);
    const int64_t row0 = tile * TP;
    const int nv = tile_rows(a, tile);
    t.tile = tile;
    t.nv = nv;
    const uint32_t valid_mask = nv == 32 ? 0xffffffffu : ((1u << nv) - 1u);
    const int64_t next = tile + gridDim.x;
    t.live = valid_mask;
    if (threadIdx.x == 0) {
      P.live = valid_mask;
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k) P.livek[k] = 0u;
      if (a.l2pf) prefetch_tile_l2(a, next + (a.nbuf == 2 ? (int64_t)gridDim.x : 0));
    }
    if constexpr (sizeof(T) == 8) {
      fetch_x(a, st, t);          // barrier inside also publishes P.live
    } else {
      if (threadIdx.x == 0) {
        if (a.nbuf == 2 && next < ntiles && tile_is_bulk(a, tile_rows(a, next)))
          issue_tile(a, b ? s.XB[0] : s.XB[1], b ? &P.mbar[0] : &P.mbar[1], next,
                     tile_rows(a, next));
        if (a.nbuf == 1 && tile_is_bulk(a, nv) && !t.next_issued)
          issue_tile(a, st.XS, &P.mbar[0], tile, nv);
      }
      t.next_issued = false;
      if (tile_is_bulk(a, nv)) {
        if (b) {
          wait_tile(&P.mbar[1], phase1);
          phase1 ^= 1u;
        } else {
          wait_tile(&P.mbar[0], t.phase);
          t.phase ^= 1u;
        }
      } else {
        const T* src = a.x + row0 * a.dim;
        for (int e = threadIdx.x; e < nv * a.dim; e += NT) st.XS[e] = src[e];
      }
      __syncthreads();
    }
    // engine.py:202-203: a non-finite x anywhere in the batch raises; a
    // finite but huge x can still overflow z (kernels.py:45-49), so such
    // tiles test every z they produce.
    const bool valid = p < nv;
    // fp32 functions whose first stage is rotated fold the scan into that
    // stage's V gather (gather_v), which reads every x anyway
    t.scanned = !(sizeof(T) == 4 && P.seg[0].n_groups > 0);
    if (t.scanned) {
      // max of |x| bit patterns (high word for float64) over the point's row
      uint32_t mx = 0u;
      if (valid) {
        const uint32_t* xw = reinterpret_cast<const uint32_t*>(st.XS + p * a.dim);
        constexpr int W = sizeof(T) / 4;          // 32-bit words per element
#pragma unroll 4
        for (int j = l8; j < a.dim; j += 8) mx = max(mx, xw[j * W + W - 1] & 0x7fffffffu);
      }
      const bool big = sizeof(T) == 8 ? mx >= 0x7bf00000u : mx >= 0x71800000u;   // x_large
      if (sizeof(T) == 8 ? mx >= 0x7ff00000u : mx >= 0x7f800000u) raise_flag(a);
      t.check_z = __syncthreads_or(big) != 0;
    }
    RB_PHASE_MARK(c_loaded);
    RB_PHASE_ADD(0, c_loaded - c_tile);
    T result;
    bool ill = false;                   // float64: value needs the exact-order z (fixup_kernel)
    if constexpr (KID >= SPEC_BASE) {
      result = spec_value<T, KID - SPEC_BASE>(a, st, t, valid, &ill);
    } else if constexpr (KID >= 0) {
      result = member_value<T, KID>(a, st, P.mem[0], t, true, &ill);
    } else if (P.fn.category != RB_COMPOSITION) {
      result = member_value<T, GENERIC>(a, st, P.mem[0], t, true, &ill);
    } else {
      result = composition_value<T>(a, st, t, valid, &ill);
    }
    const bool ill_row = sizeof(T) == 8 && l8 == 0 && valid && ill;
    if (l8 == 0 && valid) a.f[row0 + p] = ill_row ? fixup_mark<T>() : result + C<T>(100.0);  // engine.py:209
    // XS is reused by the next TMA; the CTA announces its first marked
    // tile once (two stores, one of them over PCIe)
    if constexpr (sizeof(T) == 8) {
      if (__syncthreads_or(ill_row) && threadIdx.x == 0 && !cta_marked) {
        mark_fixup(a);
        cta_marked = true;
      }
    } else {
      __syncthreads();
    }
    RB_PHASE_MARK(c_end);
    RB_PHASE_ADD(3, c_end - c_tile);
    RB_PHASE_ADD(4, 1);
  }
}

// float64 re-evaluation of the rows the main kernel marked (fixup_mark):
// points next to a HappyCat / HGBat residual, whose value needs z in NumPy's
// exact order (exact64_kernel).  Each CTA scans 32-row chunks of f, gathers
// a chunk's marked rows into one tile (X rows copied by index), evaluates
// the whole function for them -- weights and every member, the exact64
// members rotated by rotate_exact_f64 -- and writes their values.  Chunks
// without marks cost one read of their f words.  One CTA per SM with the
// full register file: the path is rare and not tuned for speed.
template <class T>
#ifndef RB_FIXUP_BLOCKS
#define RB_FIXUP_BLOCKS 2           // resident fixup CTAs per SM (A/B: 1 -> 2 +40 % on converged populations at D=100)
#endif
__global__ void __launch_bounds__(NT, RB_FIXUP_BLOCKS) fixup_kernel(const Args<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Smem<T> s = carve<T>(smem_raw, a);
  // queued behind its kernel by callers that do not read the flags first
  // (rb_func_evaluate_async): nothing marked -> done, before any plan work.
  // The test reads device memory: one PCIe read of the host flag per CTA
  // serialised to ~150 us per launch.
  if (threadIdx.x == 0) s.P->marked = *reinterpret_cast<volatile const int*>(a.mark) != 0 ? 1u : 0u;
  __syncthreads();
  if (!s.P->marked) return;
  load_plan(a, s);
  PlanHead& P = *s.P;
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int64_t nchunks = (a.n + TP - 1) / TP;
  TileCtx t{0, 0, 0u, false, true, 0u, false};
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t row0 = c * TP;
    const int nrow = tile_rows(a, c);
    if (threadIdx.x == 0) P.marked = 0u;
    __syncthreads();
    if (l8 == 0 && p < nrow && is_fixup_mark((double)a.f[row0 + p])) atomicOr(&P.marked, 1u << p);
    __syncthreads();
    const uint32_t marked = P.marked;
    if (!marked) continue;                     // (P.marked is reset behind the next barrier)
    const int nv = __popc(marked);
    // tile point q <- the chunk's q-th marked row
    for (int e = threadIdx.x; e < nv * a.dim; e += NT) {
      const int q = e / a.dim, j = e - q * a.dim;
      const int r = (int)__fns(marked, 0, q + 1);
      s.XS[e] = a.x[(row0 + r) * a.dim + j];
    }
    if (threadIdx.x == 0) {
      P.live = nv == 32 ? 0xffffffffu : ((1u << nv) - 1u);
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k) P.livek[k] = 0u;
    }
    __syncthreads();
    const bool valid = p < nv;
    t.tile = c;
    t.nv = nv;
    t.live = nv == 32 ? 0xffffffffu : ((1u << nv) - 1u);
    uint32_t mx = 0u;                          // X scan as in evaluate_kernel
    if (valid) {
      const uint32_t* xw = reinterpret_cast<const uint32_t*>(s.XS + p * a.dim);
      for (int j = l8; j < a.dim; j += 8) mx = max(mx, xw[j * 2 + 1] & 0x7fffffffu);
    }
    if (mx >= 0x7ff00000u) raise_flag(a);
    t.check_z = __syncthreads_or(mx >= 0x7bf00000u) != 0;
    const T result = P.fn.category == RB_COMPOSITION ? composition_value<T, FIXUP>(a, s, t, valid)
                                                     : member_value<T, FIXUP>(a, s, P.mem[0], t, false);
    if (l8 == 0 && valid) a.f[row0 + (int)__fns(marked, 0, p + 1)] = result + C<T>(100.0);
    __syncthreads();
  }
}

// Dimensions whose tile does not fit in shared memory (or whose DMMA units
// overflow the PlanHead table): the same evaluation with only the PlanHead
// in shared memory and the per-column tables, optima, X / V / z tiles in a
// per-CTA slice of global scratch (`per_cta` bytes from `scratch`, carve2),
// served by L1 / L2.  Tiles are loaded with plain coalesced loads; float64
// exact64 members rotate in NumPy's order directly (no marks, no fixup
// pass); DMMA units are enumerated on the fly (unit_at).  Values equal the
// shared-memory kernels' (float32: bit-identical; float64: the fixup pass's
// values for every row).
template <class T>
__global__ void __launch_bounds__(NT, 1)
    evaluate_big_kernel(const Args<T> a, unsigned char* scratch, size_t per_cta) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Smem<T> s = carve2<T>(smem_raw, scratch + (size_t)blockIdx.x * per_cta, a);
  load_plan(a, s);
  PlanHead& P = *s.P;
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int64_t ntiles = (a.n + TP - 1) / TP;
  TileCtx t{0, 0, 0u, false, true, 0u, false};
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * TP;
    const int nv = tile_rows(a, tile);
    const T* src = a.x + row0 * a.dim;
    for (int64_t e = threadIdx.x; e < (int64_t)nv * a.dim; e += NT) s.XS[e] = src[e];
    // rows past a ragged end: defined values (the DMMA tiles read all 32)
    for (int64_t e = (int64_t)nv * a.dim + threadIdx.x; e < (int64_t)TP * a.dim; e += NT) s.XS[e] = T(0);
    const uint32_t valid_mask = nv == 32 ? 0xffffffffu : ((1u << nv) - 1u);
    if (threadIdx.x == 0) {
      P.live = valid_mask;
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k) P.livek[k] = 0u;
    }
    __syncthreads();
    const bool valid = p < nv;
    t.tile = tile;
    t.nv = nv;
    t.live = valid_mask;
    uint32_t mx = 0u;                          // X scan as in evaluate_kernel
    if (valid) {
      const uint32_t* xw = reinterpret_cast<const uint32_t*>(s.XS + p * a.dim);
      constexpr int W = sizeof(T) / 4;
      for (int j = l8; j < a.dim; j += 8) mx = max(mx, xw[j * W + W - 1] & 0x7fffffffu);
    }
    if (sizeof(T) == 8 ? mx >= 0x7ff00000u : mx >= 0x7f800000u) raise_flag(a);
    t.check_z = __syncthreads_or(sizeof(T) == 8 ? mx >= 0x7bf00000u : mx >= 0x71800000u) != 0;
    const T result = P.fn.category == RB_COMPOSITION ? composition_value<T, BIGDIM>(a, s, t, valid)
                                                     : member_value<T, BIGDIM>(a, s, P.mem[0], t, false);
    if (l8 == 0 && valid) a.f[row0 + p] = result + C<T>(100.0);    // engine.py:209
    __syncthreads();
  }
}

// Host-visible table of instantiations: [0..20] basic kernels, [21] generic.
constexpr int N_VARIANTS = K_COUNT + 1;

}  // namespace rb
