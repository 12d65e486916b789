// Compile-time specialisation of the hybrid (23-28) and composition (29-36)
// functions: their segment kernels are fixed by the catalog (catalog.py:
// 147-211; paper_1407_7737_b200/catalog.py _HYBRIDS / _COMPOSITIONS), so each
// function gets its own kernel whose job loop dispatches over its own member
// kernels only (not the 21-way switch of the generic kernel): smaller code,
// registers sized for the members it has.  rb_initialize checks the pack's
// segment kernels against these tables and falls back to the generic kernel
// on any mismatch (RB_SPEC=0 forces the fallback).
#pragma once
#include "rb_device.cuh"

namespace rb {

constexpr int FN_FIRST_SPEC = 23;
constexpr int FN_COUNT_SPEC = 14;       // functions 23..36

// Jobs (member, segment) of function fid in evaluation order: kernel id and
// member index.  Hybrid members (compositions 35, 36) contribute one job per
// chunk.
struct JobList {
  int n;
  int kernel[MAX_SEGMENTS];
  int member[MAX_SEGMENTS];
};

__host__ __device__ constexpr JobList job_list(int fid) {
  // hybrid chunk kernels (catalog.py:147-164)
  constexpr int H[6][5] = {
      {K_SCHWEFEL, K_RASTRIGIN, K_ELLIPTIC, -1, -1},
      {K_CIGAR, K_HGBAT, K_RASTRIGIN, -1, -1},
      {K_GRIEWANK, K_WEIERSTRASS, K_ROSENBROCK, K_SCHAFFERS_F6, -1},
      {K_HGBAT, K_DISCUS, K_GRIE_ROSEN, K_RASTRIGIN, -1},
      {K_SCHAFFERS_F6, K_HGBAT, K_ROSENBROCK, K_SCHWEFEL, K_ELLIPTIC},
      {K_KATSUURA, K_HAPPYCAT, K_GRIE_ROSEN, K_SCHWEFEL, K_ACKLEY}};
  // composition member kernels (catalog.py:165-211); -2 = hybrid member
  constexpr int CM[6][5] = {
      {K_ROSENBROCK, K_ELLIPTIC, K_CIGAR, K_DISCUS, K_ELLIPTIC},
      {K_SCHWEFEL, K_RASTRIGIN, K_HGBAT, -1, -1},
      {K_SCHWEFEL, K_RASTRIGIN, K_ELLIPTIC, -1, -1},
      {K_SCHWEFEL, K_HAPPYCAT, K_ELLIPTIC, K_WEIERSTRASS, K_GRIEWANK},
      {K_HGBAT, K_RASTRIGIN, K_ELLIPTIC, K_WEIERSTRASS, K_SCHWEFEL},
      {K_GRIE_ROSEN, K_HAPPYCAT, K_SCHWEFEL, K_SCHAFFERS_F6, K_ELLIPTIC}};
  JobList L{};
  L.n = 0;
  auto add = [&L](int k, int m) {
    L.kernel[L.n] = k;
    L.member[L.n] = m;
    ++L.n;
  };
  if (fid >= 23 && fid <= 28) {
    for (int j = 0; j < 5; ++j)
      if (H[fid - 23][j] >= 0) add(H[fid - 23][j], 0);
  } else if (fid >= 29 && fid <= 34) {
    for (int j = 0; j < 5; ++j)
      if (CM[fid - 29][j] >= 0) add(CM[fid - 29][j], j);
  } else if (fid == 35 || fid == 36) {        // compositions of hybrids 23-25 / 26-28
    for (int m = 0; m < 3; ++m)
      for (int j = 0; j < 5; ++j)
        if (H[(fid == 35 ? 0 : 3) + m][j] >= 0) add(H[(fid == 35 ? 0 : 3) + m][j], m);
  }
  return L;
}

// Does function fid have a HappyCat / HGBat job (float64 exact-order
// fallback, rb_device.cuh exact64_kernel)?
__host__ __device__ constexpr bool has_exact64(int fid) {
  const JobList L = job_list(fid);
  bool any = false;
  for (int j = 0; j < L.n; ++j) any = any || exact64_kernel(L.kernel[j]);
  return any;
}

// Kernel value of job j of function FID: a branch chain over the function's
// own job kernels only (each inlined once per job), so the register
// allocation covers these kernels and not all 21.
template <class T, int FID, int J>
__device__ __forceinline__ T spec_kernel(int j, const Pt<T>& pt) {
  constexpr JobList L = job_list(FID);
  if constexpr (J < L.n) {
    if (j == J) return kernel_value_k<T, L.kernel[J]>(pt);
    return spec_kernel<T, FID, J + 1>(j, pt);
  } else {
    return T(0);
  }
}

// Value of function FID (hybrid or composition) for the calling lane's point:
// the jobs in order, member values summed over their chunks
// (hybrid.py:105-115), composition members blended with their weights and
// skipped when no point of the tile weighs them (composition.py:157-166).
template <class T, int FID>
__device__ T spec_value(const Args<T>& a, const Smem<T>& s, TileCtx& t, bool valid, bool* ill) {
  constexpr JobList L = job_list(FID);
  constexpr bool comp = FID >= 29;
  PlanHead& P = *s.P;
  const int p = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  T om[MAX_MEMBERS];
#pragma unroll
  for (int k = 0; k < MAX_MEMBERS; ++k) om[k] = T(0);
  RB_PHASE_MARK(cw0);
  if constexpr (comp) {
    composition_weights<T, L.member[L.n - 1] + 1>(a, P, s.XS + p * a.dim, s.opt, l8, om);
    const int nm = P.fn.n_members;
    if (l8 == 0 && valid) {
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k)
        if (k < nm && om[k] != T(0)) atomicOr(&P.livek[k], 1u << p);
    }
    __syncthreads();
  }
  RB_PHASE_MARK(cw1);
  RB_PHASE_ADD(5, cw1 - cw0);
  T total = T(0);
#pragma unroll 1
  for (int j0 = 0; j0 < L.n;) {
    // member mi = jobs [j0, j1): one staging pass, then its chunk kernels
    const int mi = P.job_mem[j0];
    int j1 = j0 + 1;
    while (j1 < L.n && P.job_mem[j1] == mi) ++j1;
    if (comp) t.live = P.livek[mi];
    if (comp && t.live == 0u) {                    // composition.py:163-164
      j0 = j1;
      continue;
    }
    const rb_member& mem = P.mem[mi];
    RB_PHASE_MARK(c0);
    const T* zb = stage_member<T, false, mt2_kernel<SPEC_BASE + FID>()>(a, s, mem, t);
    if (j1 == L.n) issue_next_x(a, s, t);
    RB_PHASE_MARK(c1);
    constexpr bool kMark = sizeof(T) == 8 && has_exact64(FID);
    bool* mark = (kMark && ((P.exact_mem >> mi) & 1u)) ? ill : nullptr;
    T g = T(0);
    for (int j = j0; j < j1; ++j) {
      const rb_segment& seg = P.seg[P.job_seg[j]];
      const Pt<T> pt{zb + p * a.ldz + seg.src, seg.d, l8, a.values + seg.ctab, mark};
      const T v = spec_kernel<T, FID, 0>(j, pt);
      g = j == j0 ? v : g + v;                     // hybrid.py:105-115: 0 + K_0 + K_1 + ...
    }
    __syncthreads();                               // z is rewritten by the next member
    RB_PHASE_MARK(c2);
    RB_PHASE_ADD(1, c1 - c0);
    RB_PHASE_ADD(2, c2 - c1);
    if (comp) {
      T omk = T(0);
#pragma unroll
      for (int k = 0; k < MAX_MEMBERS; ++k)
        if (k == mi) omk = om[k];
      if (omk != T(0)) total = total + omk * ((T)mem.height * g + (T)mem.bias);
    } else {
      total = g;
    }
    j0 = j1;
  }
  return total;
}

}  // namespace rb
