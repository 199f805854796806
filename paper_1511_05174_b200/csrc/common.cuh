// Shared device helpers for the crossdict B200 engine (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CDB_FULL_MASK 0xffffffffu

namespace cdb {

// Per-signal status bits written by the engines (internal; the ABI exports
// only the reference's out_flag = "dense min-norm fallback engaged").
enum : uint32_t {
  ST_DONE = 1u,        // finished (budget, tolerance or orthogonal break)
  ST_DELEGATE = 2u,    // hand the signal to the exact engine (rank trouble /
                       // uncertifiable selection); its results are replaced
};

// Reference constants (crossdict): _kernels.py:24 RANK_TOL.
constexpr double RANK_TOL = 1e-10;
// Gram/Cholesky engines hand a signal to the exact engine when the new
// atom's distance to the span of the support falls below this (relative, in
// squared units): 1e-8 ||a||^2, i.e. d < 1e-4 ||a||, far above RANK_TOL so
// the exact MGS test of the reference decides every borderline case.
constexpr double GRAM_DELEGATE_D2 = 1e-8;

template <typename T>
__device__ __forceinline__ double ld_f64(const T *p) { return (double)(*p); }

// Programmatic dependent launch (no-ops when the grid was launched without it)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CDB_FULL_MASK, v, o);
  return v;
}

// Arg-max over (value, index) with "strictly larger wins, ties -> lower
// index" -- the reduction form of the reference's ascending scan with a
// strict '>' (_kernels.py:94-103).  Index -1 means "none".
__device__ __forceinline__ void warp_argmax(double &v, int64_t &idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(CDB_FULL_MASK, v, o);
    int64_t oi = __shfl_xor_sync(CDB_FULL_MASK, idx, o);
    bool take = (oi >= 0) && (idx < 0 || ov > v || (ov == v && oi < idx));
    if (take) {
      v = ov;
      idx = oi;
    }
  }
}

// The reference _dot4 (_kernels.py:27-42) computed by the 4 lanes of each
// lane-quad: lane m owns the i = m (mod 4) accumulator chain; the quad
// combines ((s0+s1)+s2)+s3 and adds the tail last.  Explicit _rn intrinsics
// keep every product and sum separately rounded (numba fastmath=False), so
// the value is bit-identical to the reference's.  All 32 lanes must call it
// together; every lane of a quad gets the quad's full sum.
__device__ __forceinline__ double dot4_quad(const double *a, const double *b, int64_t n,
                                            int lane) {
  const int m = lane & 3;
  const int64_t m4 = (n / 4) * 4;
  double s = 0.0;
  for (int64_t i = m; i < m4; i += 4) s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
  const int base = lane & ~3;
  const double s0 = __shfl_sync(CDB_FULL_MASK, s, base + 0);
  const double s1 = __shfl_sync(CDB_FULL_MASK, s, base + 1);
  const double s2 = __shfl_sync(CDB_FULL_MASK, s, base + 2);
  const double s3 = __shfl_sync(CDB_FULL_MASK, s, base + 3);
  double tot = __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3);
  for (int64_t i = m4; i < n; i++) tot = __dadd_rn(tot, __dmul_rn(a[i], b[i]));
  return tot;
}

// Warp maximum of values v >= 0 (negative inputs count as 0): non-negative
// IEEE doubles order like their bit patterns, so two redux.max on the high
// and low words replace a 5-round 64-bit shuffle butterfly.
__device__ __forceinline__ double warp_max_nonneg(double v) {
  const unsigned long long b = v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mhi = __reduce_max_sync(CDB_FULL_MASK, hi);
  const unsigned mlo = __reduce_max_sync(CDB_FULL_MASK, hi == mhi ? lo : 0u);
  return __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
}

// dot4_quad of a gathered vector a[idx[i]] with b[i] (same summation order
// as dot4_quad on the compacted vector): the masked exact engine's scan.
__device__ __forceinline__ double dot4_quad_g(const double *a, const int32_t *idx,
                                              const double *b, int64_t n, int lane) {
  const int m = lane & 3;
  const int64_t m4 = (n / 4) * 4;
  double s = 0.0;
  for (int64_t i = m; i < m4; i += 4) s = __dadd_rn(s, __dmul_rn(a[idx[i]], b[i]));
  const int base = lane & ~3;
  const double s0 = __shfl_sync(CDB_FULL_MASK, s, base + 0);
  const double s1 = __shfl_sync(CDB_FULL_MASK, s, base + 1);
  const double s2 = __shfl_sync(CDB_FULL_MASK, s, base + 2);
  const double s3 = __shfl_sync(CDB_FULL_MASK, s, base + 3);
  double tot = __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3);
  for (int64_t i = m4; i < n; i++) tot = __dadd_rn(tot, __dmul_rn(a[idx[i]], b[i]));
  return tot;
}

// Element i of a coded effective atom (per-patch measurement operators, SURVEY
// row f3).  ord 0: the sequential sum of atom[idx[i*fan + u]] over the listed
// sources (-1 ends the list; fan 1 = a gather: masks, mosaics, angular
// sampling), which is numpy's frame-axis sum of a temporal code applied to
// C-contiguous columns (sensing.py:89-91; the zero-coded frames add +-0).
// ord 1: numpy's pairwise_sum over exactly `fan` slots (slot -1 = 0.0), the
// order numpy takes when the frame axis is the contiguous one -- the step-2
// columns d_high.atoms_t[allowed0].T of zero_tree_omp (crossscale.py:215) or
// a single column.  fan <= 128 in that mode (one 8-accumulator block).
__device__ __forceinline__ double eff_at(const double *atom, const int32_t *idx, int fan, int ord,
                                         int64_t i) {
  if (fan == 1) return atom[idx[i]];
  const int32_t *q = idx + i * fan;
  if (ord == 0) {
    double e = atom[q[0]];
    for (int u = 1; u < fan; u++) {
      const int32_t s = q[u];
      if (s < 0) break;
      e = __dadd_rn(e, atom[s]);
    }
    return e;
  }
  auto v = [&](int u) { return q[u] >= 0 ? atom[q[u]] : 0.0; };
  if (fan < 8) {
    double res = 0.0;
    for (int u = 0; u < fan; u++) res = __dadd_rn(res, v(u));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = v(j);
  int u = 8;
  for (; u < fan - (fan % 8); u += 8)
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], v(u + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; u < fan; u++) res = __dadd_rn(res, v(u));
  return res;
}

// dot4_quad of a coded vector (eff_at) with b[i]: the masked / coded exact
// engine's scan, same summation order as dot4_quad on the compacted vector.
__device__ __forceinline__ double dot4_quad_c(const double *a, const int32_t *idx, int fan,
                                              int ord, const double *b, int64_t n, int lane) {
  const int m = lane & 3;
  const int64_t m4 = (n / 4) * 4;
  double s = 0.0;
  for (int64_t i = m; i < m4; i += 4) s = __dadd_rn(s, __dmul_rn(eff_at(a, idx, fan, ord, i), b[i]));
  const int base = lane & ~3;
  const double s0 = __shfl_sync(CDB_FULL_MASK, s, base + 0);
  const double s1 = __shfl_sync(CDB_FULL_MASK, s, base + 1);
  const double s2 = __shfl_sync(CDB_FULL_MASK, s, base + 2);
  const double s3 = __shfl_sync(CDB_FULL_MASK, s, base + 3);
  double tot = __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3);
  for (int64_t i = m4; i < n; i++) tot = __dadd_rn(tot, __dmul_rn(eff_at(a, idx, fan, ord, i), b[i]));
  return tot;
}

}  // namespace cdb
