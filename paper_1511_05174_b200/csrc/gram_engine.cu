// Gram engine: signal-stationary exact fp64 OMP driven by the dictionary's
// Gram matrix -- one warp per signal, all iterations in one launch.
//
// Same algorithm as the reference kernel (crossdict/_kernels.py:50-168):
// greedy pick of max |<d_j, r>| over the allowed, not-taken candidates with
// the lowest index winning ties, exact least squares on the support,
// residual-norm stop test -- but the least squares is an incremental
// Cholesky of the support Gram G_SS kept as its explicit inverse factor
// L^{-1}, and the residual is never materialised.  With q_i the orthonormal
// basis the reference builds by MGS (_kernels.py:111-137), z_i = q_i^T y
// (its `qty`) and h_i[j] = d_j^T q_i:
//
//     c_j   = alpha0_j - sum_i z_i h_i[j]            (correlation, fp64)
//     w     = L^{-1} G[S, new],  d^2 = G_nn - |w|^2  (MGS projection defect)
//     z_k   = (alpha0_new - w.z) / d
//     h_k   = (G[C, new] - sum_i w_i h_i) / d
//     |r|^2 = |y|^2 - |z|^2                          (stop test, exact band check)
//
// so per iteration a signal touches one Gram row and S*k fp64 values of H
// held in shared memory, instead of re-reading S atoms of length N.  All
// arithmetic is fp64; correlations agree with the reference's to ~1e-13
// relative of |r|, far inside the 1e-6 near-tie band of the parity
// contract.  Signals whose new atom is within 1e-4 |a| of the span of the
// support (the reference's rank test is d <= 1e-10 |a|, _kernels.py:126)
// are delegated to the exact engine, which reproduces the reference bit for
// bit, including the dense minimum-norm mode.
#include "candidates.cuh"
#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

// Per-warp shared memory (doubles): L^{-1} twice (row- and column-major,
// odd row stride so column walks are bank-conflict free), the k-vectors
// z, w, g, x, the support ids, then H (rows h_i over the candidates, stride
// max_cands) -- whose first n + 2 S doubles stage y, alpha0 and c while the
// signal starts.  Correlations, alpha0 and the taken bits live in registers
// (candidate j = lane + 32 u), so smem per signal is ~8 S k + 16 k^2 bytes.
__host__ __device__ inline int64_t gram_fixed_doubles(int64_t kw) {
  return 2 * kw * (kw | 1) + 5 * kw;
}
__host__ __device__ inline int64_t gram_region_doubles(int64_t s, int64_t kw, int64_t n,
                                                       bool h_in_smem) {
  const int64_t stage = n + 2 * s;
  return h_in_smem && kw * s > stage ? kw * s : stage;
}

// alpha0_j = <d_{C_j}, y> for every candidate: the warp streams 8 atom rows
// at a time with coalesced loads (lane i reads element i of each row) and
// reduces the 8 partial sums across the warp.
__device__ __forceinline__ void alpha0_rows(const double *__restrict__ d64, const Cands &cs,
                                            int64_t p, int64_t S, int64_t n, const double *y,
                                            double *alpha0, int lane) {
  for (int64_t j0 = 0; j0 < S; j0 += 8) {
    const double *rows[8];
#pragma unroll
    for (int r = 0; r < 8; r++) rows[r] = d64 + (j0 + r < S ? cs.id(p, j0 + r) : 0) * n;
    double acc[8];
#pragma unroll
    for (int r = 0; r < 8; r++) acc[r] = 0.0;
    for (int64_t i = lane; i < n; i += 32) {
      const double yi = y[i];
#pragma unroll
      for (int r = 0; r < 8; r++) acc[r] = fma(__ldg(rows[r] + i), yi, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const double v = warp_sum(acc[r]);
      if (lane == r && j0 + r < S) alpha0[j0 + r] = v;
    }
  }
}

// KWT >= k_width and U * 32 >= max_cands are compile-time bounds (register
// arrays over this lane's candidates; KWT sizes the lane-per-row loops).
template <typename YT, int KWT, int U>
__global__ void __launch_bounds__(U <= 8 ? 384 : 256)
    gram_omp_kernel(GramArgs a, const YT *__restrict__ ys, int h_in_smem, int64_t smem_per_warp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t local = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (local >= a.p) return;
  const int64_t p = a.p_offset + local;

  const int n = (int)a.n, kw = (int)a.k_width, smax = (int)a.max_cands, ldl = kw | 1;
  const int64_t T = a.t;
  const Cands cs = a.cands;
  double *lr = (double *)(smem_raw + wib * smem_per_warp);  // lr[l*ldl+i] = L^{-1}[l][i]
  double *lc = lr + kw * ldl;                                 // lc[i*ldl+l] = L^{-1}[l][i]
  double *zv = lc + kw * ldl;
  double *wv = zv + kw;
  double *gv = wv + kw;
  double *xv = gv + kw;
  int64_t *sup = (int64_t *)(xv + kw);
  double *region = (double *)(sup + kw);
  double *h = h_in_smem ? region : a.hwork + local * kw * smax;
  const YT *yg = ys + p * a.ys_stride;

  const int S = (int)cs.count(p);
  const int k_max = (int)cs.budget(p, a.k_max, n);
  int64_t *out_sel = a.out_sel + p * kw;
  double *out_coef = a.out_coef + p * kw;

  // this lane's candidates j = lane + 32u, their atom ids, unavailable bits
  int cid[U];
  unsigned tk = 0u;
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int j = lane + 32 * u;
    cid[u] = j < S ? (int)cs.id(p, j) : 0;
    if (j >= S) tk |= 1u << u;
  }
  double *y = region;  // staging until the first H row is written
  for (int i = lane; i < n; i += 32) y[i] = (double)yg[i];
  __syncwarp();
  const double ynorm = sqrt(dot4_quad(y, y, n, lane));  // reference order (_kernels.py:71)
  const double tol = a.eps[p];

  int kdone = 0;
  int64_t scans = 0;
  double rnorm = ynorm;
  double rn2_final = 0.0, yy_final = 1.0;
  bool delegate = false;

  if (!(ynorm <= tol) && k_max > 0) {
    double a0[U], cr[U];
    if (a.alpha0_in) {
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int j = lane + 32 * u;
        a0[u] = j < S ? a.alpha0_in[p * smax + j] : 0.0;
      }
    } else {
      double *al = y + n;
      alpha0_rows(a.d64, cs, p, S, n, y, al, lane);
      __syncwarp();
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int j = lane + 32 * u;
        a0[u] = j < S ? al[j] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) cr[u] = a0[u];
    double yy = 0.0;
    for (int i = lane; i < n; i += 32) yy = fma(y[i], y[i], yy);
    yy = warp_sum(yy);
    double rn2 = yy;
    yy_final = yy;
    const double tol2 = tol * tol;
    const double band = 1e-12 * yy;
    int64_t sup0 = 0, sup1 = 0;  // sup[lane], sup[lane + 32]
    __syncwarp();                // staging is dead from here (H row 0 overwrites it)

    for (int k = 0; k < k_max; k++) {
      rn2_final = rn2;
      scans += S - k;
      // ---- selection: max |c_j| over available candidates, ties -> lowest j
      double best = -1.0;
      unsigned bj = 0xffffffffu;
#pragma unroll
      for (int u = 0; u < U; u++) {
        const double v = fabs(cr[u]);
        if (!((tk >> u) & 1u) && v > best) {
          best = v;
          bj = lane + 32 * u;
        }
      }
      double m = best;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(CDB_FULL_MASK, m, o));
      if (!(m > 0.0)) break;  // nothing left, or best <= 0 (_kernels.py:104)
      const int bestj = (int)__reduce_min_sync(CDB_FULL_MASK, best == m ? bj : 0xffffffffu);
      const int ub = bestj >> 5, owner = bestj & 31;
      int my_id = 0;
      double my_a0 = 0.0;
#pragma unroll
      for (int u = 0; u < U; u++)
        if (u == ub) {
          my_id = cid[u];
          my_a0 = a0[u];
        }
      const int64_t nid = __shfl_sync(CDB_FULL_MASK, my_id, owner);
      const double a0_new = __shfl_sync(CDB_FULL_MASK, my_a0, owner);
      if (lane == owner) tk |= 1u << ub;
      // ---- gathers from Gram row `nid` (independent loads)
      const double *grow = a.gram + nid * T;
      double hacc[U];
#pragma unroll
      for (int u = 0; u < U; u++) hacc[u] = lane + 32 * u < S ? __ldg(grow + cid[u]) : 0.0;
      const double gl = lane < k ? __ldg(grow + sup0) : 0.0;
      const double gl2 = lane + 32 < k ? __ldg(grow + sup1) : 0.0;
      const double gnn = __ldg(grow + nid);
      if (lane == k) sup0 = nid;
      if (lane + 32 == k) sup1 = nid;
      if (lane == 0) sup[k] = nid;
      if (lane < k) gv[lane] = gl;
      if (lane + 32 < k) gv[lane + 32] = gl2;
      __syncwarp();
      // ---- w = L^{-1} G[S, new]   (lane l owns rows l, l + 32)
#pragma unroll
      for (int half = 0; half < (KWT + 31) / 32; half++) {
        const int l = lane + 32 * half;
        double acc = 0.0;
#pragma unroll 4
        for (int i = 0; i < k; i++)
          if (i <= l && l < k) acc = fma(lc[i * ldl + l], gv[i], acc);
        if (l < k) wv[l] = acc;
      }
      __syncwarp();
      double ww = 0.0, wz = 0.0;
      for (int l = lane; l < k; l += 32) {
        ww = fma(wv[l], wv[l], ww);
        wz = fma(wv[l], zv[l], wz);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ww += __shfl_xor_sync(CDB_FULL_MASK, ww, o);
        wz += __shfl_xor_sync(CDB_FULL_MASK, wz, o);
      }
      const double d2 = gnn - ww;
      if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine decides
        delegate = true;
        break;
      }
      const double inv_d = 1.0 / sqrt(d2);
      const double zk = (a0_new - wz) * inv_d;
      // ---- new row of L^{-1}: [-(w^T L^{-1}) / d, 1/d]
#pragma unroll
      for (int half = 0; half < (KWT + 31) / 32; half++) {
        const int i = lane + 32 * half;
        double acc = 0.0;
#pragma unroll 4
        for (int l = 0; l < k; l++)
          if (l >= i) acc = fma(wv[l], lr[l * ldl + i], acc);
        if (i <= k) {
          const double v = i == k ? inv_d : -acc * inv_d;
          lr[k * ldl + i] = v;
          lc[i * ldl + k] = v;
        }
      }
      if (lane == 0) zv[k] = zk;
      // ---- h_k over candidates, correlation update (U independent chains)
#pragma unroll 2
      for (int i = 0; i < k; i++) {
        const double wi = wv[i];
        const double *hi = h + i * smax + lane;
#pragma unroll
        for (int u = 0; u < U; u++)
          if (lane + 32 * u < S) hacc[u] = fma(-wi, hi[32 * u], hacc[u]);
      }
      double *hk = h + k * smax + lane;
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (lane + 32 * u < S) {
          const double hv = hacc[u] * inv_d;
          hk[32 * u] = hv;
          cr[u] = fma(-zk, hv, cr[u]);
        }
      }
      rn2 -= zk * zk;
      rn2_final = rn2;
      kdone = k + 1;
      __syncwarp();
      // ---- stop test (_kernels.py:156), exact residual inside the band
      const double gap = rn2 - tol2;
      if (gap > band) continue;
      if (gap < -band) break;
      for (int i = lane; i < kdone; i += 32) {
        double acc = 0.0;
        for (int l = i; l < kdone; l++) acc = fma(lr[l * ldl + i], zv[l], acc);
        xv[i] = acc;
      }
      __syncwarp();
      double rr = 0.0;
      for (int i = lane; i < n; i += 32) {
        double ri = (double)yg[i];
        for (int l = 0; l < kdone; l++) ri = fma(-xv[l], a.d64[sup[l] * n + i], ri);
        rr = fma(ri, ri, rr);
      }
      rr = warp_sum(rr);
      if (sqrt(rr) <= tol) break;
    }
  }

  if (delegate) {
    if (lane == 0) a.status[p] |= ST_DELEGATE;
    return;  // the exact engine rewrites every output of this signal
  }
  // ---- coefficients x = L^{-T} z (pick order), exact final residual norm
  __syncwarp();
  for (int i = lane; i < kdone; i += 32) {
    double acc = 0.0;
    for (int l = i; l < kdone; l++) acc = fma(lr[l * ldl + i], zv[l], acc);
    xv[i] = acc;
  }
  __syncwarp();
  if (kdone > 0) {
    // |r| = sqrt(|y|^2 - |z|^2) is accurate to ~1e-16 |y|^2 / |r|^2 relative;
    // re-materialise the residual exactly only when that is not tight
    if (rn2_final > 1e-6 * yy_final) {
      rnorm = sqrt(rn2_final);
    } else {
      double rr = 0.0;
      for (int i = lane; i < n; i += 32) {
        double ri = (double)yg[i];
        for (int l = 0; l < kdone; l++) ri = fma(-xv[l], __ldg(a.d64 + sup[l] * n + i), ri);
        rr = fma(ri, ri, rr);
      }
      rnorm = sqrt(warp_sum(rr));
    }
  }
  for (int j = lane; j < kw; j += 32) {
    out_sel[j] = j < kdone ? sup[j] : -1;
    out_coef[j] = j < kdone ? xv[j] : 0.0;
  }
  if (lane == 0) {
    a.out_count[p] = kdone;
    a.out_rnorm[p] = rnorm;
    a.out_scans[p] = scans;
    a.out_flag[p] = 0;
  }
}

template <typename YT, int KWT, int U>
cudaError_t launch_gram_tu(const GramArgs &args, const YT *ys, int h_in_smem, int64_t per_warp,
                           int wpb, int64_t blocks, cudaStream_t stream) {
  const int64_t smem = per_warp * wpb;
  cudaError_t e = cudaFuncSetAttribute(gram_omp_kernel<YT, KWT, U>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  gram_omp_kernel<YT, KWT, U><<<(unsigned)blocks, wpb * 32, smem, stream>>>(args, ys, h_in_smem,
                                                                            per_warp);
  return cudaGetLastError();
}

template <typename YT, int KWT>
cudaError_t launch_gram_t(const GramArgs &args, const YT *ys, int u, int h_in_smem,
                          int64_t per_warp, int wpb, int64_t blocks, cudaStream_t stream) {
  switch (u) {
    case 1: return launch_gram_tu<YT, KWT, 1>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 2: return launch_gram_tu<YT, KWT, 2>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 4: return launch_gram_tu<YT, KWT, 4>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 8: return launch_gram_tu<YT, KWT, 8>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 16: return launch_gram_tu<YT, KWT, 16>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
  }
  return cudaErrorInvalidValue;
}

template <typename YT>
cudaError_t launch_gram_y(const GramArgs &args, const YT *ys, int kwt, int u, int h_in_smem,
                          int64_t per_warp, int wpb, int64_t blocks, cudaStream_t stream) {
  switch (kwt) {
    case 8: return launch_gram_t<YT, 8>(args, ys, u, h_in_smem, per_warp, wpb, blocks, stream);
    case 16: return launch_gram_t<YT, 16>(args, ys, u, h_in_smem, per_warp, wpb, blocks, stream);
    case 32: return launch_gram_t<YT, 32>(args, ys, u, h_in_smem, per_warp, wpb, blocks, stream);
    case 64: return launch_gram_t<YT, 64>(args, ys, u, h_in_smem, per_warp, wpb, blocks, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int64_t gram_total_smem(int64_t s, int64_t kw, int64_t n, bool h_in_smem) {
  const int64_t b = 8 * (gram_fixed_doubles(kw) + gram_region_doubles(s, kw, n, h_in_smem));
  return (b + 15) & ~int64_t(15);
}

cudaError_t launch_gram(const GramArgs &args, const void *ys, bool ys_f32, int max_smem_per_block,
                        int num_sms, cudaStream_t stream) {
  ProfScope _ps(args.tag ? args.tag : "gram_omp", stream);
  (void)num_sms;
  if (args.p <= 0) return cudaSuccess;
  const int64_t s = args.max_cands, kw = args.k_width, n = args.n;
  const bool h_in_smem = args.hwork == nullptr;
  const int64_t per_warp = gram_total_smem(s, kw, n, h_in_smem);
  if (per_warp > max_smem_per_block) return cudaErrorInvalidValue;
  if (kw > 64 || s > 512) return cudaErrorInvalidValue;
  int u = 1;
  while (32 * u < s) u *= 2;
  int wpb = (int)(max_smem_per_block / per_warp);
  if (wpb > (u <= 8 ? 12 : 8)) wpb = u <= 8 ? 12 : 8;
  if (wpb < 1) wpb = 1;
  const int64_t blocks = (args.p + wpb - 1) / wpb;
  int kwt = 8;
  while (kwt < kw) kwt *= 2;
  note_launch();
  if (ys_f32)
    return launch_gram_y<float>(args, (const float *)ys, kwt, u, h_in_smem ? 1 : 0, per_warp, wpb,
                                blocks, stream);
  return launch_gram_y<double>(args, (const double *)ys, kwt, u, h_in_smem ? 1 : 0, per_warp, wpb,
                               blocks, stream);
}

}  // namespace cdb
