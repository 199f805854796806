// Gram engine: signal-stationary exact fp64 OMP driven by the dictionary's
// Gram matrix -- one warp per signal, all iterations in one launch.
//
// Same algorithm as the reference kernel (crossdict/_kernels.py:50-168):
// greedy pick of max |<d_j, r>| over the allowed, not-taken candidates with
// the lowest index winning ties, modified Gram-Schmidt least squares,
// residual-norm stop test, back-substitution for the coefficients -- but
// the residual and the basis vectors are never materialised.  With q_i the
// orthonormal basis the reference builds by MGS (_kernels.py:111-137),
// z_i = q_i^T y (its `qty`) and h_i[j] = q_i^T d_{C_j}:
//
//     c_j   = alpha0_j - sum_i z_i h_i[j]             (correlation, fp64)
//     w_i   = q_i^T d_new = h_i[new]                  (MGS coefficients = R[i][k])
//     d^2   = G_nn - |w|^2                            (projection defect = R[k][k]^2)
//     z_k   = c_new / d
//     h_k   = (G[C, new] - sum_i w_i h_i) / d
//     |r|^2 = |y|^2 - |z|^2                           (stop test, exact band check)
//     R x = z                                         (back-substitution, _kernels.py:159-164)
//
// so per iteration a signal touches one Gram row slice and S*k fp64 values
// of H held in shared memory, instead of re-reading S atoms of length N.
// All arithmetic is fp64; correlations agree with the reference's to
// ~1e-13 relative of |r|, far inside the 1e-6 near-tie band of the parity
// contract.  Signals whose new atom is within 1e-4 |a| of the span of the
// support (the reference's rank test is d <= 1e-10 |a|, _kernels.py:126)
// are delegated to the exact engine, which reproduces the reference bit for
// bit, including the dense minimum-norm mode.
#include "candidates.cuh"
#include <cstdlib>

#include "common.cuh"
#include "engines.h"
#include "sm100.cuh"

namespace cdb {
namespace {

// H row layout: row stride HS = 32 U doubles; candidate j = lane + 32 u sits
// at hslot(j), pairs (u = 2v, 2v + 1) of one lane adjacent so each lane moves
// its U values with U/2 conflict-free 16-byte accesses.
template <int U>
__host__ __device__ __forceinline__ int hslot(int j) {
  if (U == 1) return j;
  const int u = j >> 5;
  return (u >> 1) * 64 + (j & 31) * 2 + (u & 1);
}

// Per-warp shared memory (doubles): z, 1/d, pick slots, support ids, x
// (k_width each), then the H rows -- whose first n + S doubles stage y and
// alpha0 while the signal starts (H in global memory: staging only).
__host__ __device__ inline int64_t gram_hs(int64_t s) {
  // U = 6 and 12 (even: the paired layout) trim H for S in (128, 192] and
  // (256, 384] -- e.g. cfg 3's step 2 (S = 384): 74 instead of 98 KB per signal
  const int64_t us[7] = {1, 2, 4, 6, 8, 12, 16};
  for (int i = 0; i < 7; i++)
    if (32 * us[i] >= s) return 32 * us[i];
  return 32 * 16;
}
__host__ __device__ inline int64_t gram_region_doubles(int64_t s, int64_t kw, int64_t n,
                                                       bool h_in_smem) {
  const int64_t stage = n + s;
  const int64_t hd = kw * gram_hs(s);
  return h_in_smem && hd > stage ? hd : stage;
}
// Streamed H (see gram_omp_kernel): default warps per SM (CDB_GRAM_WPB overrides).
// cfg 4 step 2 (1M signals): 2 / 3 / 4 / 6 / 8 warps -> 1019 / 767 / 816 / 1169 /
// 1365 ms; at 3, 444 slots x (64 - 18 smem rows) x 4 KB = 84 MB stay in L2.
constexpr int kStreamWarpsPerSm = 3;
// cfg 4 step 2 per 1M signals: 2 / 3 CTAs per SM -> 729 / 1002 ms (warp kernel: 767)
constexpr int kStreamCtasPerSm = 2;
// TMEM rows for the streamed H: at most 4 warps per CTA (one TMEM lane
// quarter each).
// Measured SLOWER than reading those rows from L2 (cfg 4, 1M: 1091 / 884 ms
// at 3 / 4 warps vs 768 ms), so opt-in only: CDB_GRAM_TMEM=1.
inline bool gram_stream_tmem(int wpb) {
  const char *v = getenv("CDB_GRAM_TMEM");
  return wpb <= 4 && v && atoi(v) != 0;
}

// sum_i y_i^2 over this thread's share (i = tid, tid + nt, ...) with eight
// loads in flight: the per-signal prologue otherwise waits one HBM round trip
// per element (4096 / 128 = 32 of them per thread for cfg 4).
template <typename YT>
__device__ __forceinline__ double row_sumsq(const YT *__restrict__ y, int n, int tid, int nt) {
  double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int i = tid;
  for (; i + 7 * nt < n; i += 8 * nt) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) v[u] = (double)__ldg(y + i + u * nt);
#pragma unroll
    for (int u = 0; u < 8; u++) s[u] = fma(v[u], v[u], s[u]);
  }
  for (; i < n; i += nt) {
    const double v = (double)__ldg(y + i);
    s[0] = fma(v, v, s[0]);
  }
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
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

// Coefficients by back-substitution R x = z (_kernels.py:159-164), with the
// MGS factor read out of H: R[i][l] = q_i^T d_{s_l} = h_i[pick_l] (i < l),
// R[l][l] = d_l.  Column sweep: lane i (and i + 32) accumulates
// sum_{l > i} R[i][l] x_l.
// H rows: rows i < nr at hs + i HS (shared memory), the rest at hg + i HS.
template <int U>
__device__ __forceinline__ const double *hrow(const double *hs, const double *hg, int nr, int i) {
  return (i < nr ? hs : hg) + (int64_t)i * (32 * U);
}

// TMEM rows (TMR): rows [nr, nr + ntr) live in the warp's TMEM lane quarter,
// slot-major: candidate j = lane + 32 u, row nr + t at columns 32 u + 2 t
// (lo, hi words).  A warp-wide load of the 32 columns of slot u gives every
// lane its slot-u values of all TMEM rows; for the column R[., l] the owner
// lane of pick l publishes its 16 values through `tcol` (shared memory).
template <int U, bool TMR>
__device__ void back_substitute(const double *hs, const double *hg, int nr, int ntr,
                                uint32_t tbase, double *tcol, int kd, const double *zv,
                                const double *iv, const int *pj, double *xv, int lane) {
  const int i0 = lane, i1 = lane + 32;
  const bool t0 = TMR && i0 >= nr && i0 < nr + ntr, t1 = TMR && i1 >= nr && i1 < nr + ntr;
  const double *h0 = hrow<U>(hs, hg, nr, i0);
  const double *h1 = hrow<U>(hs, hg, nr, i1);
  double acc0 = 0.0, acc1 = 0.0;
  for (int l = kd - 1; l >= 0; l--) {
    const double accl = __shfl_sync(CDB_FULL_MASK, l < 32 ? acc0 : acc1, l & 31);
    const double xl = (zv[l] - accl) * iv[l];
    if (lane == 0) xv[l] = xl;
    const int sl = hslot<U>(pj[l]);
    double r0 = 0.0, r1 = 0.0;
    if (TMR && l > nr) {  // some row i < l lives in TMEM
      uint32_t v[32];
      sm100::tmem_ld32u(tbase + 32u * (uint32_t)(pj[l] >> 5), v);
      sm100::tmem_wait_ld();
      if (lane == (pj[l] & 31)) {
#pragma unroll
        for (int t = 0; t < 16; t++) tcol[t] = __hiloint2double((int)v[2 * t + 1], (int)v[2 * t]);
      }
      __syncwarp();
      if (t0) r0 = tcol[i0 - nr];
      if (t1) r1 = tcol[i1 - nr];
      __syncwarp();
    }
    if (lane < l) acc0 = fma(t0 ? r0 : h0[sl], xl, acc0);
    if (lane + 32 < l) acc1 = fma(t1 ? r1 : h1[sl], xl, acc1);
  }
  __syncwarp();
}

// The TMEM rows' share of the H sweep: w_t = H[j*][nr + t] from the owner
// lane's slot-ub columns, then hacc[u] -= sum_t w_t h_{nr+t}[lane + 32 u].
template <int U>
__device__ __forceinline__ void tm_sweep(uint32_t tbase, int tr, int ub, int owner,
                                         double (&hacc)[U], double &ww) {
  uint32_t v[32];
  sm100::tmem_ld32u(tbase + 32u * (uint32_t)ub, v);
  sm100::tmem_wait_ld();
  double w[16];
#pragma unroll
  for (int t = 0; t < 16; t++) {
    const double mine = __hiloint2double((int)v[2 * t + 1], (int)v[2 * t]);
    w[t] = __shfl_sync(CDB_FULL_MASK, mine, owner);
    if (t < tr) ww = fma(w[t], w[t], ww);
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    sm100::tmem_ld32u(tbase + 32u * (uint32_t)u, v);
    sm100::tmem_wait_ld();
#pragma unroll
    for (int t = 0; t < 16; t++)
      if (t < tr) hacc[u] = fma(-w[t], __hiloint2double((int)v[2 * t + 1], (int)v[2 * t]), hacc[u]);
  }
}

// hacc -= sum_{i in [i0, i1)} w_i h_i, ww += |w|^2 over those rows (w_i = h_i[bs]).
template <int U, int UNR>
__device__ __forceinline__ void h_sweep(const double *h, int i0, int i1, int bs, int lane,
                                        double (&hacc)[U], double &ww) {
  constexpr int HS = 32 * U;
#pragma unroll UNR
  for (int i = i0; i < i1; i++) {
    const double *hi = h + (int64_t)i * HS;
    const double wi = hi[bs];  // = q_i^T d_{j*}
    ww = fma(wi, wi, ww);
    if (U == 1) {
      hacc[0] = fma(-wi, hi[lane], hacc[0]);
    } else {
#pragma unroll
      for (int v = 0; v < U / 2; v++) {
        const double2 t2 = *(const double2 *)(hi + v * 64 + lane * 2);
        hacc[2 * v] = fma(-wi, t2.x, hacc[2 * v]);
        hacc[2 * v + 1] = fma(-wi, t2.y, hacc[2 * v + 1]);
      }
    }
  }
}

// U * 32 >= max_cands is a compile-time bound (register arrays over this
// lane's candidates j = lane + 32 u).
//
// Per iteration, with j* the pick: w_i = q_i^T d_{j*} = h_i[j*] (the MGS
// projection coefficients are a column of H), d^2 = G[j*,j*] - |w|^2,
// z_k = c_{j*} / d, h_k = (G[C, j*] - sum_i w_i h_i) / d, c -= z_k h_k.
// Every lane reads the w_i it needs as a broadcast out of H while it
// updates its own candidates, and accumulates |w|^2 redundantly, so an
// iteration has no triangular solve and a single cross-lane reduction
// (the argmax).
//
// HSM (H fits shared memory): one warp per signal.  Otherwise (cfg 4's step
// 2: S = 512, K = 64, 256 KB of H per signal) the warps are persistent and
// each owns one H slot: its first `nr` rows in shared memory (the oldest
// rows, read by every later iteration: rows < nr carry
// sum_{i<nr} (k_max - i) of the sum_i (k_max - i) row reads) and the rest in
// a per-warp global slot sized so that all slots stay L2-resident -- a
// streamed H is then read from L2, not HBM.
//
// HM == 2 (TMR) adds 16 TMEM rows per warp between the shared-memory and the
// global rows (each warp of the <= 4-warp CTA owns one TMEM lane quarter, 64 KB),
// so fewer rows stream from L2.
template <typename YT, int U, int HM>
__global__ void __launch_bounds__(U <= 8 ? 512 : 256)
    gram_omp_kernel(GramArgs a, const YT *__restrict__ ys, int h_rows_smem, int64_t smem_per_warp) {
  constexpr int HS = 32 * U;
  constexpr bool HSM = HM == 1, TMR = HM == 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int n = (int)a.n, kw = (int)a.k_width, smax = (int)a.max_cands;
  const int64_t T = a.t;
  const Cands cs = a.cands;
  double *zv = (double *)(smem_raw + wib * smem_per_warp);
  double *iv = zv + kw;              // 1 / d_l
  int *pj = (int *)(iv + kw);        // candidate index of pick l
  int64_t *sup = (int64_t *)(iv + 2 * kw);
  double *xv = (double *)(sup + kw);
  double *tcol = xv + kw;                     // TMR: one TMEM column, 16 doubles
  double *region = tcol + (HSM ? 0 : 16) + ((5 * kw) & 1);  // even: 16-byte H accesses
  // HSM: H in shared memory, known at compile time so its accesses are LDS/STS
  // rather than generic loads; else rows >= nr (+ TMEM rows) in this warp's global slot
  const int nr = HSM ? kw : h_rows_smem;
  const int ntr = TMR ? (kw - nr < 16 ? kw - nr : 16) : 0;
  double *hs = region;
  double *hg = HSM ? region
                   : a.hwork + gw * (int64_t)(kw - nr - ntr) * HS - (int64_t)(nr + ntr) * HS;
  __shared__ uint32_t tm_base_s;
  uint32_t tbase = 0;
  if (TMR) {
    if (wib == 0) sm100::tmem_alloc(&tm_base_s, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    tbase = tm_base_s + ((uint32_t)(32 * (wib & 3)) << 16);
#pragma unroll 1
    for (int c = 0; c < 16; c++) sm100::tmem_st32_zero(tbase + 32u * c);  // finite unused rows
    sm100::tmem_wait_st();
  }

  for (int64_t local = gw; local < a.p; local += nwarps) {
  const int64_t p = a.p_offset + local;
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
  double *y = region;  // staging until the first H row is written (in-kernel alpha0 only)
  const bool stage = a.alpha0_in == nullptr;
  double yy = 0.0;
  for (int i = lane; i < n; i += 32) {
    const double v = (double)yg[i];
    if (stage) y[i] = v;
    yy = fma(v, v, yy);
  }
  yy = warp_sum(yy);
  __syncwarp();
  const double ynorm = sqrt(yy);  // early exit |y| <= tol (_kernels.py:71-78)
  const double tol = a.eps[p];

  int kdone = 0;
  int64_t scans = 0;
  double rnorm = ynorm;
  double rn2_final = 0.0, yy_final = 1.0;
  bool delegate = false;

  if (!(ynorm <= tol) && k_max > 0) {
    double cr[U];
    if (a.alpha0_in) {
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int j = lane + 32 * u;
        cr[u] = j < S ? a.alpha0_in[p * smax + j] : 0.0;
      }
    } else {
      double *al = y + n;
      alpha0_rows(a.d64, cs, p, S, n, y, al, lane);
      __syncwarp();
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int j = lane + 32 * u;
        cr[u] = j < S ? al[j] : 0.0;
      }
    }
    double rn2 = yy;
    yy_final = yy;
    const double tol2 = tol * tol;
    const double band = 1e-12 * yy;
    __syncwarp();  // staging is dead from here (H row 0 overwrites it)

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
      const double m = warp_max_nonneg(best);
      if (!(m > 0.0)) break;  // nothing left, or best <= 0 (_kernels.py:104)
      const int bestj = (int)__reduce_min_sync(CDB_FULL_MASK, best == m ? bj : 0xffffffffu);
      const int ub = bestj >> 5, owner = bestj & 31;
      int my_id = 0;
      double my_c = 0.0;
#pragma unroll
      for (int u = 0; u < U; u++)
        if (u == ub) {
          my_id = cid[u];
          my_c = cr[u];
        }
      const int64_t nid = __shfl_sync(CDB_FULL_MASK, my_id, owner);
      const double cj = __shfl_sync(CDB_FULL_MASK, my_c, owner);
      if (lane == owner) tk |= 1u << ub;
      // ---- Gram row slice G[C, j*] (independent loads), then H update
      // 32-bit row offset when the Gram matrix has < 2^31 entries
      const double *grow = a.gram + (T * T < (int64_t(1) << 31)
                                         ? (int64_t)((uint32_t)nid * (uint32_t)T)
                                         : nid * T);
      // (loading the slice into separate registers, added after the sweep,
      // measured slower: 766 -> 802 ms per 1M on cfg 4)
      double hacc[U];
#pragma unroll
      for (int u = 0; u < U; u++) hacc[u] = lane + 32 * u < S ? __ldg(grow + cid[u]) : 0.0;
      const double gnn = __ldg(grow + nid);
      const int bs = hslot<U>(bestj);
      double ww = 0.0;
      if (HSM) {
        h_sweep<U, 2>(hs, 0, k, bs, lane, hacc, ww);
      } else {
        h_sweep<U, 2>(hs, 0, k < nr ? k : nr, bs, lane, hacc, ww);
        if (TMR && k > nr) tm_sweep<U>(tbase, k - nr < ntr ? k - nr : ntr, ub, owner, hacc, ww);
        if (k > nr + ntr) h_sweep<U, 4>(hg, nr + ntr, k, bs, lane, hacc, ww);
      }
      const double d2 = gnn - ww;
      if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine decides
        delegate = true;
        break;
      }
      const double inv_d = rsqrt(d2);
      const double zk = cj * inv_d;  // q_k^T y = q_k^T r = <d_{j*}, r> / d
      const bool in_tm = TMR && k >= nr && k < nr + ntr;
      double *hk = (HSM || k < nr ? hs : hg) + (int64_t)k * HS;
      if (in_tm) {
#pragma unroll
        for (int u = 0; u < U; u++) {
          const double hv = hacc[u] * inv_d;
          sm100::tmem_st2(tbase + 32u * u + 2u * (uint32_t)(k - nr),
                          (uint32_t)__double2loint(hv), (uint32_t)__double2hiint(hv));
          cr[u] = fma(-zk, hv, cr[u]);
        }
        sm100::tmem_wait_st();
      } else if (U == 1) {
        const double hv = hacc[0] * inv_d;
        hk[lane] = hv;
        cr[0] = fma(-zk, hv, cr[0]);
      } else {
#pragma unroll
        for (int v = 0; v < U / 2; v++) {
          const double h0 = hacc[2 * v] * inv_d, h1 = hacc[2 * v + 1] * inv_d;
          *(double2 *)(hk + v * 64 + lane * 2) = make_double2(h0, h1);
          cr[2 * v] = fma(-zk, h0, cr[2 * v]);
          cr[2 * v + 1] = fma(-zk, h1, cr[2 * v + 1]);
        }
      }
      if (lane == 0) {
        zv[k] = zk;
        iv[k] = inv_d;
        pj[k] = bestj;
        sup[k] = nid;
      }
      rn2 -= zk * zk;
      rn2_final = rn2;
      kdone = k + 1;
      __syncwarp();
      // ---- stop test (_kernels.py:156), exact residual inside the band
      const double gap = rn2 - tol2;
      if (gap > band) continue;
      if (gap < -band) break;
      back_substitute<U, TMR>(hs, hg, nr, ntr, tbase, tcol, kdone, zv, iv, pj, xv, lane);
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
    __syncwarp();
    continue;  // the exact engine rewrites every output of this signal
  }
  // ---- coefficients (pick order), exact final residual norm
  __syncwarp();
  back_substitute<U, TMR>(hs, hg, nr, ntr, tbase, tcol, kdone, zv, iv, pj, xv, lane);
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
  __syncwarp();  // the next signal re-stages the shared region
  }
  if (TMR) {
    sm100::tc_fence_before();
    __syncthreads();
    if (wib == 0) sm100::tmem_dealloc(tm_base_s, 512);
  }
}

// ---------------------------------------------------------------- CTA per signal
// Streamed H with a precomputed alpha0 (cfg 4's step 2: S = 512, K = 64): one
// 128-thread CTA per signal, thread t owning the CPT contiguous candidates
// [t CPT, t CPT + CPT).  Against the warp-per-signal kernel the per-iteration
// chain (Gram row gather, H sweep) is spread over 4 warps: each row's sweep
// is 2 x 16-byte loads per thread and 8 rows of the L2-resident part are in
// flight per thread, at the cost of one CTA barrier per iteration (the
// arg-max exchange, double-buffered by iteration parity; it also publishes
// row k-1 of H to every thread).  Same arithmetic as gram_omp_kernel.
// H rows [0, nr) in shared memory, the rest in the CTA's global slot.
template <int CPT>
__device__ void back_sub_rows(const double *hs, const double *hg, int nr, int stride, int kd,
                              const double *zv, const double *iv, const int *pj, double *xv,
                              int lane) {
  const double *h0 = (lane < nr ? hs : hg) + (int64_t)lane * stride;
  const double *h1 = (lane + 32 < nr ? hs : hg) + (int64_t)(lane + 32) * stride;
  double acc0 = 0.0, acc1 = 0.0;
  // steps in blocks of 8: the block's R entries (L2 for rows >= nr) are loaded
  // before its dependent chain, so each block waits for one round trip, not 8
  for (int l0 = kd - 1; l0 >= 0; l0 -= 8) {
    double r0[8], r1[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int l = l0 - u;
      const int sl = l >= 0 ? pj[l] : 0;
      r0[u] = l >= 0 && lane < l ? h0[sl] : 0.0;
      r1[u] = l >= 0 && lane + 32 < l ? h1[sl] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int l = l0 - u;
      if (l < 0) break;
      const double accl = __shfl_sync(CDB_FULL_MASK, l < 32 ? acc0 : acc1, l & 31);
      const double xl = (zv[l] - accl) * iv[l];
      if (lane == 0) xv[l] = xl;
      if (lane < l) acc0 = fma(r0[u], xl, acc0);
      if (lane + 32 < l) acc1 = fma(r1[u], xl, acc1);
    }
  }
  __syncwarp();
}

template <typename YT, int CPT>
__global__ void __launch_bounds__(128) gram_cta_kernel(GramArgs a, const YT *__restrict__ ys,
                                                        int nr) {
  constexpr int NT = 128, NW = NT / 32;
  constexpr int SP = NT * CPT;  // H row stride (doubles)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)a.n, kw = (int)a.k_width, smax = (int)a.max_cands;
  const int64_t T = a.t;
  const Cands cs = a.cands;
  double *zv = (double *)smem_raw;
  double *iv = zv + kw;
  int64_t *sup = (int64_t *)(iv + kw);
  double *xv = (double *)(sup + kw);
  int *pj = (int *)(xv + kw);               // kw ints in kw doubles of space
  double *xb = xv + 2 * kw;                 // exchange: [2][NW] x {|c|, c}
  int64_t *xi = (int64_t *)(xb + 4 * NW);   // exchange: [2][NW] x {j, atom}
  double *red = (double *)(xi + 4 * NW);    // NW partial sums + 2 flags
  double *hs = red + NW + 2;
  hs += ((uintptr_t)hs & 15) ? 1 : 0;       // 16-byte aligned rows
  double *hg = a.hwork + (int64_t)blockIdx.x * (kw - nr) * SP - (int64_t)nr * SP;
  const bool q8 = cs.mode == 2 && cs.q % CPT == 0;  // a thread's candidates are contiguous atoms

  for (int64_t local = blockIdx.x; local < a.p; local += gridDim.x) {
    const int64_t p = a.p_offset + local;
    const YT *yg = ys + p * a.ys_stride;
    const int S = (int)cs.count(p);
    const int k_max = (int)cs.budget(p, a.k_max, n);
    int cid[CPT];
    unsigned tk = 0u;
#pragma unroll
    for (int c = 0; c < CPT; c++) {
      const int j = tid * CPT + c;
      cid[c] = j < S ? (int)cs.id(p, j) : 0;
      if (j >= S) tk |= 1u << c;
    }
    double yy = row_sumsq(yg, n, tid, NT);
    yy = warp_sum(yy);
    if (lane == 0) red[warp] = yy;
    __syncthreads();
    yy = 0.0;
#pragma unroll
    for (int w = 0; w < NW; w++) yy += red[w];
    const double ynorm = sqrt(yy);  // early exit |y| <= tol (_kernels.py:71-78)
    const double tol = a.eps[p];
    int kdone = 0;
    int64_t scans = 0;
    double rnorm = ynorm, rn2_final = 0.0;
    bool delegate = false;
    if (!(ynorm <= tol) && k_max > 0) {
      double cr[CPT];
#pragma unroll
      for (int c = 0; c < CPT; c++) {
        const int j = tid * CPT + c;
        cr[c] = j < S ? a.alpha0_in[p * smax + j] : 0.0;
      }
      double rn2 = yy;
      const double tol2 = tol * tol, band = 1e-12 * yy;
      for (int k = 0; k < k_max; k++) {
        rn2_final = rn2;
        scans += S - k;
        // ---- arg-max: thread, warp, then the 4 warps through shared memory
        double best = -1.0;
        int bc = 0;
#pragma unroll
        for (int c = 0; c < CPT; c++) {
          const double v = fabs(cr[c]);
          if (!((tk >> c) & 1u) && v > best) {
            best = v;
            bc = c;
          }
        }
        const unsigned bj = best >= 0.0 ? (unsigned)(tid * CPT + bc) : 0xffffffffu;
        const double m = warp_max_nonneg(best);
        const unsigned wj = __reduce_min_sync(CDB_FULL_MASK, best == m ? bj : 0xffffffffu);
        const int src = __ffs(__ballot_sync(CDB_FULL_MASK, bj == wj)) - 1;
        double myc = 0.0;
        int myid = 0;
#pragma unroll
        for (int c = 0; c < CPT; c++)
          if (c == bc) {
            myc = cr[c];
            myid = cid[c];
          }
        const double wc = __shfl_sync(CDB_FULL_MASK, myc, src < 0 ? 0 : src);
        const int wid = __shfl_sync(CDB_FULL_MASK, myid, src < 0 ? 0 : src);
        const int par = k & 1;
        if (lane == 0) {
          xb[(par * NW + warp) * 2] = m;
          xb[(par * NW + warp) * 2 + 1] = wc;
          xi[(par * NW + warp) * 2] = (int64_t)wj;
          xi[(par * NW + warp) * 2 + 1] = wid;
        }
        __syncthreads();  // also publishes row k-1 of H
        double gm = -1.0, cj = 0.0;
        int64_t gj = 0xffffffffll, nid = 0;
#pragma unroll
        for (int w = 0; w < NW; w++) {
          const double mw = xb[(par * NW + w) * 2];
          const int64_t jw = xi[(par * NW + w) * 2];
          if (mw > gm || (mw == gm && jw < gj)) {
            gm = mw;
            gj = jw;
            cj = xb[(par * NW + w) * 2 + 1];
            nid = xi[(par * NW + w) * 2 + 1];
          }
        }
        if (!(gm > 0.0)) break;  // nothing left, or best <= 0 (_kernels.py:104)
        const int bestj = (int)gj;
        if (tid == bestj / CPT) tk |= 1u << (bestj % CPT);
        if (a.prefetch_runner) {
          // the best other warp's candidate often wins the next iteration: pull
          // its Gram row slice toward L2 now (the next gather then misses less)
          double g2 = -1.0;
          int64_t n2 = -1;
#pragma unroll
          for (int w = 0; w < NW; w++) {
            const double mw = xb[(par * NW + w) * 2];
            const int64_t jw = xi[(par * NW + w) * 2];
            if (jw != gj && mw > g2) {
              g2 = mw;
              n2 = xi[(par * NW + w) * 2 + 1];
            }
          }
          if (n2 >= 0 && g2 > 0.0 && tid * CPT < S)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.gram + n2 * T + cid[0]));
        }
        // ---- Gram row slice, H sweep
        // the slice (an HBM gather) lands in its own registers and is added
        // after the sweep, so its latency overlaps the sweep
        const double *grow = a.gram + nid * T;
        double gsl[CPT], hacc[CPT];
        if (q8 && tid * CPT + CPT <= S) {
          const double2 *g2 = (const double2 *)(grow + cid[0]);
#pragma unroll
          for (int c = 0; c < CPT / 2; c++) {
            const double2 t2 = __ldg(g2 + c);
            gsl[2 * c] = t2.x;
            gsl[2 * c + 1] = t2.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < CPT; c++) gsl[c] = tid * CPT + c < S ? __ldg(grow + cid[c]) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < CPT; c++) hacc[c] = 0.0;
        const double gnn = __ldg(grow + nid);
        double ww = 0.0;
        const int ks = k < nr ? k : nr;
#pragma unroll 4
        for (int i = 0; i < ks; i++) {
          const double *hi = hs + i * SP;
          const double wi = hi[bestj];
          ww = fma(wi, wi, ww);
#pragma unroll
          for (int c = 0; c < CPT / 2; c++) {
            const double2 t2 = *(const double2 *)(hi + tid * CPT + 2 * c);
            hacc[2 * c] = fma(-wi, t2.x, hacc[2 * c]);
            hacc[2 * c + 1] = fma(-wi, t2.y, hacc[2 * c + 1]);
          }
        }
        // L2-resident rows in blocks of RB, software-pipelined: block b+1's
        // 3 RB loads are issued before block b's FMAs (a plain unrolled loop
        // with a runtime bound let ptxas serialise them: one row in flight)
        constexpr int RB = 8;
        int i = nr;
        if (i + RB <= k) {
          double wc[RB];
          double2 hc[RB][CPT / 2];
#pragma unroll
          for (int q = 0; q < RB; q++) {
            const double *hi = hg + (int64_t)(i + q) * SP;
            wc[q] = hi[bestj];
#pragma unroll
            for (int c = 0; c < CPT / 2; c++) hc[q][c] = ((const double2 *)(hi + tid * CPT))[c];
          }
          for (; i + RB <= k; i += RB) {
            double wn[RB];
            double2 hn[RB][CPT / 2];
            const bool more = i + 2 * RB <= k;
            if (more) {
#pragma unroll
              for (int q = 0; q < RB; q++) {
                const double *hi = hg + (int64_t)(i + RB + q) * SP;
                wn[q] = hi[bestj];
#pragma unroll
                for (int c = 0; c < CPT / 2; c++) hn[q][c] = ((const double2 *)(hi + tid * CPT))[c];
              }
            }
#pragma unroll
            for (int q = 0; q < RB; q++) {
              ww = fma(wc[q], wc[q], ww);
#pragma unroll
              for (int c = 0; c < CPT / 2; c++) {
                hacc[2 * c] = fma(-wc[q], hc[q][c].x, hacc[2 * c]);
                hacc[2 * c + 1] = fma(-wc[q], hc[q][c].y, hacc[2 * c + 1]);
              }
            }
            if (more) {
#pragma unroll
              for (int q = 0; q < RB; q++) {
                wc[q] = wn[q];
#pragma unroll
                for (int c = 0; c < CPT / 2; c++) hc[q][c] = hn[q][c];
              }
            }
          }
        }
        for (; i < k; i++) {
          const double *hi = hg + (int64_t)i * SP;
          const double wi = hi[bestj];
          ww = fma(wi, wi, ww);
#pragma unroll
          for (int c = 0; c < CPT / 2; c++) {
            const double2 t2 = ((const double2 *)(hi + tid * CPT))[c];
            hacc[2 * c] = fma(-wi, t2.x, hacc[2 * c]);
            hacc[2 * c + 1] = fma(-wi, t2.y, hacc[2 * c + 1]);
          }
        }
#pragma unroll
        for (int c = 0; c < CPT; c++) hacc[c] += gsl[c];
        const double d2 = gnn - ww;  // identical in every thread (same w_i, same order)
        if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine decides
          delegate = true;
          break;
        }
        const double inv_d = rsqrt(d2);
        const double zk = cj * inv_d;
        double *hk = (k < nr ? hs : hg) + (int64_t)k * SP + tid * CPT;
#pragma unroll
        for (int c = 0; c < CPT / 2; c++) {
          const double h0 = hacc[2 * c] * inv_d, h1 = hacc[2 * c + 1] * inv_d;
          *(double2 *)(hk + 2 * c) = make_double2(h0, h1);
          cr[2 * c] = fma(-zk, h0, cr[2 * c]);
          cr[2 * c + 1] = fma(-zk, h1, cr[2 * c + 1]);
        }
        if (tid == 0) {
          zv[k] = zk;
          iv[k] = inv_d;
          pj[k] = bestj;
          sup[k] = nid;
        }
        rn2 -= zk * zk;
        rn2_final = rn2;
        kdone = k + 1;
        // ---- stop test (_kernels.py:156), exact residual inside the band
        const double gap = rn2 - tol2;
        if (gap > band) continue;
        if (gap < -band) break;
        __syncthreads();  // row k and the pick in place
        if (warp == 0) {
          back_sub_rows<CPT>(hs, hg, nr, SP, kdone, zv, iv, pj, xv, lane);
          double rr = 0.0;
          for (int i = lane; i < n; i += 32) {
            double ri = (double)yg[i];
            for (int l = 0; l < kdone; l++) ri = fma(-xv[l], a.d64[sup[l] * n + i], ri);
            rr = fma(ri, ri, rr);
          }
          rr = warp_sum(rr);
          if (lane == 0) red[NW] = sqrt(rr) <= tol ? 1.0 : 0.0;
        }
        __syncthreads();
        if (red[NW] != 0.0) break;
      }
    }
    __syncthreads();  // H, z, picks complete
    if (delegate) {
      if (tid == 0) a.status[p] |= ST_DELEGATE;
    } else if (warp == 0) {
      back_sub_rows<CPT>(hs, hg, nr, SP, kdone, zv, iv, pj, xv, lane);
      if (kdone > 0) {
        if (rn2_final > 1e-6 * yy) {
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
      int64_t *out_sel = a.out_sel + p * kw;
      double *out_coef = a.out_coef + p * kw;
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
    __syncthreads();  // the next signal reuses the shared state
  }
}

// ---------------------------------------------------------------- TMA-streamed rows
// gram_cta_kernel with the L2-resident rows streamed by the bulk-copy engine:
// the rows [nr, k) an iteration re-reads go through a ring of RS shared-memory
// slots (4 KB each: the whole row of the signal), issued by one thread right
// after the arg-max barrier -- before the Gram gather and the shared-memory
// rows' sweep, so their L2 latency hides behind that work -- and refilled as
// the sweep frees them (full / empty mbarriers per slot).  The row sweep order
// and arithmetic are gram_cta_kernel's, so the results are bit-identical; the
// register pipeline of 8 in-flight rows (252 registers) is gone.
constexpr int kRingSlots = 8;

template <typename YT, int CPT>
__global__ void __launch_bounds__(128) gram_tma_kernel(GramArgs a, const YT *__restrict__ ys,
                                                        int nr) {
  constexpr int NT = 128, NW = NT / 32, RS = kRingSlots;
  constexpr int SP = NT * CPT;  // H row stride (doubles)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)a.n, kw = (int)a.k_width, smax = (int)a.max_cands;
  const int64_t T = a.t;
  const Cands cs = a.cands;
  double *zv = (double *)smem_raw;
  double *iv = zv + kw;
  int64_t *sup = (int64_t *)(iv + kw);
  double *xv = (double *)(sup + kw);
  int *pj = (int *)(xv + kw);
  double *xb = xv + 2 * kw;                 // exchange: [2][NW] x {|c|, c}
  int64_t *xi = (int64_t *)(xb + 4 * NW);   // exchange: [2][NW] x {j, atom}
  double *red = (double *)(xi + 4 * NW);    // NW partial sums + 2 flags
  double *hs = red + NW + 2;
  hs += ((uintptr_t)hs & 15) ? 1 : 0;       // 16-byte aligned rows
  double *ring = hs + (int64_t)nr * SP;     // RS x SP
  uint64_t *full = (uint64_t *)(ring + (int64_t)RS * SP);
  uint64_t *empty = full + RS;
  double *hg = a.hwork + (int64_t)blockIdx.x * (kw - nr) * SP - (int64_t)nr * SP;
  const bool q8 = cs.mode == 2 && cs.q % CPT == 0;
  if (tid == 0) {
    for (int r = 0; r < RS; r++) {
      sm100::mbar_init(&full[r], 1);
      sm100::mbar_init(&empty[r], NT);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  uint32_t qbase = 0;  // ring uses so far (CTA-uniform)
  auto issue = [&](uint32_t q, int row) {  // tid 0: row -> slot q % RS once it is free
    const uint32_t sl = q % RS, ph = (q / RS) & 1;
    sm100::mbar_wait(&empty[sl], ph ^ 1);
    sm100::mbar_expect_tx(&full[sl], (uint32_t)(SP * sizeof(double)));
    sm100::bulk_load(ring + (int64_t)sl * SP, hg + (int64_t)row * SP, (uint32_t)(SP * sizeof(double)),
                     &full[sl]);
  };

  for (int64_t local = blockIdx.x; local < a.p; local += gridDim.x) {
    const int64_t p = a.p_offset + local;
    const YT *yg = ys + p * a.ys_stride;
    const int S = (int)cs.count(p);
    const int k_max = (int)cs.budget(p, a.k_max, n);
    int cid[CPT];
    unsigned tk = 0u;
#pragma unroll
    for (int c = 0; c < CPT; c++) {
      const int j = tid * CPT + c;
      cid[c] = j < S ? (int)cs.id(p, j) : 0;
      if (j >= S) tk |= 1u << c;
    }
    double yy = row_sumsq(yg, n, tid, NT);
    yy = warp_sum(yy);
    if (lane == 0) red[warp] = yy;
    __syncthreads();
    yy = 0.0;
#pragma unroll
    for (int w = 0; w < NW; w++) yy += red[w];
    const double ynorm = sqrt(yy);  // early exit |y| <= tol (_kernels.py:71-78)
    const double tol = a.eps[p];
    int kdone = 0;
    int64_t scans = 0;
    double rnorm = ynorm, rn2_final = 0.0;
    bool delegate = false;
    if (!(ynorm <= tol) && k_max > 0) {
      double cr[CPT];
#pragma unroll
      for (int c = 0; c < CPT; c++) {
        const int j = tid * CPT + c;
        cr[c] = j < S ? a.alpha0_in[p * smax + j] : 0.0;
      }
      double rn2 = yy;
      const double tol2 = tol * tol, band = 1e-12 * yy;
      for (int k = 0; k < k_max; k++) {
        rn2_final = rn2;
        scans += S - k;
        // ---- arg-max: thread, warp, then the 4 warps through shared memory
        double best = -1.0;
        int bc = 0;
#pragma unroll
        for (int c = 0; c < CPT; c++) {
          const double v = fabs(cr[c]);
          if (!((tk >> c) & 1u) && v > best) {
            best = v;
            bc = c;
          }
        }
        const unsigned bj = best >= 0.0 ? (unsigned)(tid * CPT + bc) : 0xffffffffu;
        const double m = warp_max_nonneg(best);
        const unsigned wj = __reduce_min_sync(CDB_FULL_MASK, best == m ? bj : 0xffffffffu);
        const int src = __ffs(__ballot_sync(CDB_FULL_MASK, bj == wj)) - 1;
        double myc = 0.0;
        int myid = 0;
#pragma unroll
        for (int c = 0; c < CPT; c++)
          if (c == bc) {
            myc = cr[c];
            myid = cid[c];
          }
        const double wc = __shfl_sync(CDB_FULL_MASK, myc, src < 0 ? 0 : src);
        const int wid = __shfl_sync(CDB_FULL_MASK, myid, src < 0 ? 0 : src);
        const int par = k & 1;
        if (lane == 0) {
          xb[(par * NW + warp) * 2] = m;
          xb[(par * NW + warp) * 2 + 1] = wc;
          xi[(par * NW + warp) * 2] = (int64_t)wj;
          xi[(par * NW + warp) * 2 + 1] = wid;
        }
        __syncthreads();  // also publishes row k-1 of H (shared memory or, fenced, the L2 slot)
        double gm = -1.0, cj = 0.0;
        int64_t gj = 0xffffffffll, nid = 0;
#pragma unroll
        for (int w = 0; w < NW; w++) {
          const double mw = xb[(par * NW + w) * 2];
          const int64_t jw = xi[(par * NW + w) * 2];
          if (mw > gm || (mw == gm && jw < gj)) {
            gm = mw;
            gj = jw;
            cj = xb[(par * NW + w) * 2 + 1];
            nid = xi[(par * NW + w) * 2 + 1];
          }
        }
        if (!(gm > 0.0)) break;  // nothing left, or best <= 0 (_kernels.py:104)
        const int bestj = (int)gj;
        // ---- the L2 rows of this iteration start streaming now
        const int nl = k > nr ? k - nr : 0;
        if (tid == 0)
          for (int j = 0; j < nl && j < RS; j++) issue(qbase + j, nr + j);
        if (tid == bestj / CPT) tk |= 1u << (bestj % CPT);
        // ---- Gram row slice (HBM gather, lands after the sweep), H sweep
        const double *grow = a.gram + nid * T;
        double gsl[CPT], hacc[CPT];
        if (q8 && tid * CPT + CPT <= S) {
          const double2 *g2 = (const double2 *)(grow + cid[0]);
#pragma unroll
          for (int c = 0; c < CPT / 2; c++) {
            const double2 t2 = __ldg(g2 + c);
            gsl[2 * c] = t2.x;
            gsl[2 * c + 1] = t2.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < CPT; c++) gsl[c] = tid * CPT + c < S ? __ldg(grow + cid[c]) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < CPT; c++) hacc[c] = 0.0;
        const double gnn = __ldg(grow + nid);
        double ww = 0.0;
        const int ks = k < nr ? k : nr;
#pragma unroll 4
        for (int i = 0; i < ks; i++) {
          const double *hi = hs + i * SP;
          const double wi = hi[bestj];
          ww = fma(wi, wi, ww);
#pragma unroll
          for (int c = 0; c < CPT / 2; c++) {
            const double2 t2 = *(const double2 *)(hi + tid * CPT + 2 * c);
            hacc[2 * c] = fma(-wi, t2.x, hacc[2 * c]);
            hacc[2 * c + 1] = fma(-wi, t2.y, hacc[2 * c + 1]);
          }
        }
        for (int j = 0; j < nl; j++) {  // ring rows, same order and arithmetic
          const uint32_t q = qbase + j, sl = q % RS, ph = (q / RS) & 1;
          sm100::mbar_wait(&full[sl], ph);
          const double *hi = ring + (int64_t)sl * SP;
          const double wi = hi[bestj];
          ww = fma(wi, wi, ww);
#pragma unroll
          for (int c = 0; c < CPT / 2; c++) {
            const double2 t2 = *(const double2 *)(hi + tid * CPT + 2 * c);
            hacc[2 * c] = fma(-wi, t2.x, hacc[2 * c]);
            hacc[2 * c + 1] = fma(-wi, t2.y, hacc[2 * c + 1]);
          }
          sm100::mbar_arrive(&empty[sl]);
          if (tid == 0 && j + RS < nl) issue(q + RS, nr + j + RS);
        }
        qbase += nl;
#pragma unroll
        for (int c = 0; c < CPT; c++) hacc[c] += gsl[c];
        const double d2 = gnn - ww;  // identical in every thread (same w_i, same order)
        if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine decides
          delegate = true;
          break;
        }
        const double inv_d = rsqrt(d2);
        const double zk = cj * inv_d;
        double *hk = (k < nr ? hs : hg) + (int64_t)k * SP + tid * CPT;
#pragma unroll
        for (int c = 0; c < CPT / 2; c++) {
          const double h0 = hacc[2 * c] * inv_d, h1 = hacc[2 * c + 1] * inv_d;
          *(double2 *)(hk + 2 * c) = make_double2(h0, h1);
          cr[2 * c] = fma(-zk, h0, cr[2 * c]);
          cr[2 * c + 1] = fma(-zk, h1, cr[2 * c + 1]);
        }
        if (k >= nr) sm100::fence_proxy_async_global();  // row k is read back by the bulk copies
        if (tid == 0) {
          zv[k] = zk;
          iv[k] = inv_d;
          pj[k] = bestj;
          sup[k] = nid;
        }
        rn2 -= zk * zk;
        rn2_final = rn2;
        kdone = k + 1;
        // ---- stop test (_kernels.py:156), exact residual inside the band
        const double gap = rn2 - tol2;
        if (gap > band) continue;
        if (gap < -band) break;
        __syncthreads();  // row k and the pick in place
        if (warp == 0) {
          back_sub_rows<CPT>(hs, hg, nr, SP, kdone, zv, iv, pj, xv, lane);
          double rr = 0.0;
          for (int i = lane; i < n; i += 32) {
            double ri = (double)yg[i];
            for (int l = 0; l < kdone; l++) ri = fma(-xv[l], a.d64[sup[l] * n + i], ri);
            rr = fma(ri, ri, rr);
          }
          rr = warp_sum(rr);
          if (lane == 0) red[NW] = sqrt(rr) <= tol ? 1.0 : 0.0;
        }
        __syncthreads();
        if (red[NW] != 0.0) break;
      }
    }
    __syncthreads();  // H, z, picks complete
    if (delegate) {
      if (tid == 0) a.status[p] |= ST_DELEGATE;
    } else if (warp == 0) {
      back_sub_rows<CPT>(hs, hg, nr, SP, kdone, zv, iv, pj, xv, lane);
      if (kdone > 0) {
        if (rn2_final > 1e-6 * yy) {
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
      int64_t *out_sel = a.out_sel + p * kw;
      double *out_coef = a.out_coef + p * kw;
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
    __syncthreads();  // the next signal reuses the shared state
  }
}

// ---------------------------------------------------------------- on-chip H
// cfg 4's step 2 (S = 512, K = 64: 256 KB of fp64 H per signal) with the whole
// H on chip: one 512-thread CTA per SM codes one signal at a time, thread t
// owning candidate t and its H column -- rows [0, R) in registers (the oldest
// rows, which take most of the sum_i (k_max - i) row reads), rows [R, kw) in
// shared memory, private to the thread (no bank conflicts, no barriers).  The
// streamed kernels above re-read those rows from L2 and, at 1M signals, from
// HBM (ncu: 0.5 MB of DRAM reads per signal); here the per-iteration H traffic
// is register and shared-memory bandwidth only, and the one remaining global
// access is the Gram row slice G[j*, C] (one 8-byte load per thread).
//
// Per iteration: warp arg-max (redux) -> each warp's winner publishes
// {|c|, c, d^2, G_jj, index, atom} and its H column w into a per-warp slot
// (double-buffered by iteration parity) -> one CTA barrier -> every thread
// picks the global winner from the 16 slots (strict '>' in warp order: the
// lowest index wins ties) and issues its Gram load -> sweep
// h_k = (G[j*, t] - sum_i w_i h_i[t]) / d, c_t -= z_k h_k.  d^2 = G_jj - |w|^2
// uses s_t = sum_i h_i[t]^2, kept incrementally by the owner in the order the
// other Gram kernels sum |w|^2.  The winner also files its column as column k
// of R (R[i][k] = h_i[j*]) for the back-substitution R x = z
// (_kernels.py:159-164).
// Register rows are filled 8 at a time: row k < R is written to a per-thread
// staging slot (shared memory) and, when its block of 8 is complete, the 8
// staged rows move into hr[8 b, 8 b + 8) under a warp-uniform switch -- every
// register index stays static (a dynamic hr[k] write costs R selects).
template <int R>
__device__ __forceinline__ void load_block(double (&hr)[R], int b, const double *st) {
#pragma unroll
  for (int bb = 0; bb < R / 8; bb++) {
    if (bb == b) {
#pragma unroll
      for (int u = 0; u < 8; u++) hr[8 * bb + u] = st[u * 512];
    }
  }
}

// dst[i] = src[(i - r0) * 512] for i in [r0, k): a thread's shared-memory H
// rows, four loads in flight before the stores.
__device__ __forceinline__ void copy_col(double *dst, const double *src, int r0, int k) {
  int i = r0;
  for (; i + 3 < k; i += 4) {
    const double v0 = src[(int64_t)(i - r0) * 512], v1 = src[(int64_t)(i + 1 - r0) * 512];
    const double v2 = src[(int64_t)(i + 2 - r0) * 512], v3 = src[(int64_t)(i + 3 - r0) * 512];
    dst[i] = v0;
    dst[i + 1] = v1;
    dst[i + 2] = v2;
    dst[i + 3] = v3;
  }
  for (; i < k; i++) dst[i] = src[(int64_t)(i - r0) * 512];
}

// The full register blocks of a thread's H column (rows [0, kb)) -> dst.
template <int R>
__device__ __forceinline__ void put_regs(double *dst, const double (&hr)[R], int kb) {
#pragma unroll
  for (int b = 0; b < R / 8; b++) {
    if (8 * b + 8 <= kb) {
#pragma unroll
      for (int u = 0; u < 8; u += 2)
        *(double2 *)(dst + 8 * b + u) = make_double2(hr[8 * b + u], hr[8 * b + u + 1]);
    }
  }
}

// Column l of R (R[i][l] = h_i[p_l], i < l) filed by the thread that owns
// pick l, once per signal: register rows, staged rows of the open block,
// shared-memory rows (all immutable once written).
template <int R>
__device__ __forceinline__ void file_col(double *rm, int kw, int l, const double (&hr)[R],
                                         const double *stg, const double *hsm, int kdone) {
  if (l < 0) return;
  double *col = rm + (int64_t)l * kw;
  const int kr = kdone < R ? kdone : R, kb = kr & ~7;
#pragma unroll
  for (int i = 0; i < R; i++)
    if (i < l && i < kb) col[i] = hr[i];
  for (int i = kb; i < l && i < kr; i++) col[i] = stg[(i & 7) * 512];
  if (l > R) copy_col(col, hsm, R, l);
}

// Back-substitution R x = z (_kernels.py:159-164) with column l of R at
// rm + l kw; lane i (and i + 32) accumulates sum_{l > i} R[i][l] x_l -- the
// order of back_sub_rows.
__device__ __forceinline__ void back_sub_cols(const double *rm, int kw, int kd, const double *zv,
                                              const double *iv, double *xv, int lane) {
  double acc0 = 0.0, acc1 = 0.0;
  for (int l0 = kd - 1; l0 >= 0; l0 -= 8) {  // a block's columns loaded ahead of its chain
    double r0[8], r1[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int l = l0 - u;
      const double *col = rm + (int64_t)(l >= 0 ? l : 0) * kw;
      r0[u] = l >= 0 && lane < l ? col[lane] : 0.0;
      r1[u] = l >= 0 && lane + 32 < l ? col[lane + 32] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int l = l0 - u;
      if (l < 0) break;
      const double accl = __shfl_sync(CDB_FULL_MASK, l < 32 ? acc0 : acc1, l & 31);
      const double xl = (zv[l] - accl) * iv[l];
      if (lane == 0) xv[l] = xl;
      if (lane < l) acc0 = fma(r0[u], xl, acc0);
      if (lane + 32 < l) acc1 = fma(r1[u], xl, acc1);
    }
  }
  __syncwarp();
}

template <typename YT, int R>
__global__ void __launch_bounds__(512, 1) gram_reg_kernel(GramArgs a, const YT *__restrict__ ys) {
  constexpr int NT = 512, NW = NT / 32;
  static_assert(R % 8 == 0, "register rows come in blocks of 8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n = (int)a.n, kw = (int)a.k_width, smax = (int)a.max_cands;
  const int64_t T = a.t;
  const Cands cs = a.cands;
  const int nsr = kw > R ? kw - R : 0;             // shared-memory rows
  constexpr int SL = 6 + R;                         // slot: 6 header doubles + register rows of w
  double *hsm = (double *)smem_raw;                 // nsr x NT, column t private to thread t
  // staging rows of the open register block: the first 8 shared-memory rows,
  // unused while k < R (R is a multiple of 8, the last block moves at k = R - 1)
  double *stg = hsm;
  double *slots = hsm + (int64_t)(nsr > 8 ? nsr : 8) * NT;  // [2][NW][SL]
  double *rm = a.hwork + (int64_t)blockIdx.x * kw * kw;  // kw x kw (global): column l of R at rm + l kw
  double *zv = slots + 2 * NW * SL;
  double *iv = zv + kw;
  double *xv = iv + kw;
  int64_t *sup = (int64_t *)(xv + kw);
  double *red = (double *)(sup + kw);               // NW
  auto cta_sum = [&](double v) -> double {
    v = warp_sum(v);
    __syncthreads();  // red reuse
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; w++) s += red[w];
    return s;
  };

  for (int64_t local = blockIdx.x; local < a.p; local += gridDim.x) {
    const int64_t p = a.p_offset + local;
    const YT *yg = ys + p * a.ys_stride;
    const int S = (int)cs.count(p);
    const int k_max = (int)cs.budget(p, a.k_max, n);
    const bool valid = t < S;
    const int64_t cid = valid ? cs.id(p, t) : 0;
    double yy = cta_sum(row_sumsq(yg, n, t, NT));
    const double ynorm = sqrt(yy);  // early exit |y| <= tol (_kernels.py:71-78)
    const double tol = a.eps[p];
    int kdone = 0;
    int64_t scans = 0;
    double rnorm = ynorm, rn2_final = 0.0;
    bool delegate = false;
    double hr[R];
    int mypick = -1;  // the iteration this thread's candidate was picked at
    if (!(ynorm <= tol) && k_max > 0) {
#pragma unroll
      for (int i = 0; i < R; i++) hr[i] = 0.0;
      double c = valid ? a.alpha0_in[p * smax + t] : 0.0;
      const double gjj = valid ? __ldg(a.gram + cid * T + cid) : 1.0;
      double s2 = 0.0;  // sum_i h_i[t]^2
      bool taken = !valid;
      double rn2 = yy;
      const double tol2 = tol * tol, band = 1e-12 * yy;
      int k = 0;
      for (;;) {  // iterations; leaves the inner loop only to stop or to test the band
      bool check = false;
      for (; k < k_max; k++) {
        rn2_final = rn2;
        scans += S - k;
        const int par = k & 1;
        double *sbase = slots + par * NW * SL;
        // ---- warp arg-max; the warp's winner publishes its column
        const double v = taken ? 0.0 : fabs(c);
        const double m = warp_max_nonneg(v);
        const unsigned wj = __reduce_min_sync(CDB_FULL_MASK, v == m ? (unsigned)t : 0xffffffffu);
        if ((unsigned)t == wj) {
          double *sl = sbase + warp * SL;
          sl[0] = m;
          sl[1] = c;
          sl[2] = gjj - s2;
          sl[3] = gjj;
          ((int64_t *)sl)[4] = (cid << 16) | t;
          put_regs<R>(sl + 6, hr, (k < R ? k : R) & ~7);  // other rows: read in place
        }
        __syncthreads();
        // ---- global winner: lane w reads slot w; strict '>' in warp order
        // (lowest index on ties) = the first slot holding the maximum
        const double mw = lane < NW ? sbase[lane * SL] : 0.0;
        const double gm = warp_max_nonneg(mw);
        if (!(gm > 0.0)) break;  // nothing left, or best <= 0 (_kernels.py:104)
        const int gw = __ffs(__ballot_sync(CDB_FULL_MASK, lane < NW && mw == gm)) - 1;
        const double *ws = sbase + gw * SL;
        const int64_t packed = ((const int64_t *)ws)[4];
        const int bestj = (int)(packed & 0xffff);
        const int64_t nid = packed >> 16;
        const double g = valid ? __ldg(a.gram + nid * T + cid) : 0.0;
        const double cj = ws[1], d2 = ws[2], gnn = ws[3];
        const double *w = ws + 6;
        // ---- sweep: sum_i w_i h_i[t] (register blocks, staged rows, smem rows)
        const int kr = k < R ? k : R, kb = kr & ~7;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int b = 0; b < R / 8; b++) {
          if (8 * b + 8 <= kb) {
            const double2 w0 = *(const double2 *)(w + 8 * b), w1 = *(const double2 *)(w + 8 * b + 2);
            const double2 w2 = *(const double2 *)(w + 8 * b + 4), w3 = *(const double2 *)(w + 8 * b + 6);
            a0 = fma(w0.x, hr[8 * b], a0);
            a1 = fma(w0.y, hr[8 * b + 1], a1);
            a2 = fma(w1.x, hr[8 * b + 2], a2);
            a3 = fma(w1.y, hr[8 * b + 3], a3);
            a0 = fma(w2.x, hr[8 * b + 4], a0);
            a1 = fma(w2.y, hr[8 * b + 5], a1);
            a2 = fma(w3.x, hr[8 * b + 6], a2);
            a3 = fma(w3.y, hr[8 * b + 7], a3);
          }
        }
        // staged and shared-memory rows: w_i read from the winner's own column
        for (int i = kb; i < kr; i++) a0 = fma(stg[(i & 7) * NT + bestj], stg[(i & 7) * NT + t], a0);
        {
          const double *hc = hsm + t, *wc = hsm + bestj;
          int i = R;
          for (; i + 3 < k; i += 4) {
            const int64_t o = (int64_t)(i - R) * NT;
            a0 = fma(wc[o], hc[o], a0);
            a1 = fma(wc[o + NT], hc[o + NT], a1);
            a2 = fma(wc[o + 2 * NT], hc[o + 2 * NT], a2);
            a3 = fma(wc[o + 3 * NT], hc[o + 3 * NT], a3);
          }
          for (; i < k; i++) a0 = fma(wc[(int64_t)(i - R) * NT], hc[(int64_t)(i - R) * NT], a0);
        }
        if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine decides
          delegate = true;
          break;
        }
        const double inv_d = rsqrt(d2);
        const double zk = cj * inv_d;  // q_k^T y = <d_{j*}, r> / d
        const double hk = valid ? (g - ((a0 + a1) + (a2 + a3))) * inv_d : 0.0;
        if ((unsigned)t == (unsigned)bestj) {
          taken = true;
          mypick = k;
          zv[k] = zk;
          iv[k] = inv_d;
          sup[k] = nid;
        }
        if (k < R) {
          stg[(k & 7) * NT + t] = hk;
          if ((k & 7) == 7) load_block<R>(hr, k >> 3, stg + t);
        } else {
          hsm[(int64_t)(k - R) * NT + t] = hk;
        }
        c = fma(-zk, hk, c);
        s2 = fma(hk, hk, s2);
        rn2 -= zk * zk;
        rn2_final = rn2;
        kdone = k + 1;
        // ---- stop test (_kernels.py:156), exact residual inside the band
        const double gap = rn2 - tol2;
        if (gap > band) continue;
        if (gap < -band) break;
        check = true;
        break;
      }
      if (!check) break;
      file_col<R>(rm, kw, mypick, hr, stg + t, hsm + t, kdone);
      __syncthreads();  // R and the picks in place
      if (warp == 0) back_sub_cols(rm, kw, kdone, zv, iv, xv, lane);
      __syncthreads();
      double rr = 0.0;
      for (int i = t; i < n; i += NT) {
        double ri = (double)yg[i];
        for (int l = 0; l < kdone; l++) ri = fma(-xv[l], a.d64[sup[l] * n + i], ri);
        rr = fma(ri, ri, rr);
      }
      rr = cta_sum(rr);
      if (sqrt(rr) <= tol) break;
      k++;
      }
    }
    __syncthreads();  // R, z, picks complete
    if (delegate) {
      if (t == 0) a.status[p] |= ST_DELEGATE;
      __syncthreads();
      continue;
    }
    file_col<R>(rm, kw, mypick, hr, stg + t, hsm + t, kdone);
    __syncthreads();
    if (warp == 0) back_sub_cols(rm, kw, kdone, zv, iv, xv, lane);
    __syncthreads();
    if (kdone > 0) {
      if (rn2_final > 1e-6 * yy) {
        rnorm = sqrt(rn2_final);
      } else {
        double rr = 0.0;
        for (int i = t; i < n; i += NT) {
          double ri = (double)yg[i];
          for (int l = 0; l < kdone; l++) ri = fma(-xv[l], __ldg(a.d64 + sup[l] * n + i), ri);
          rr = fma(ri, ri, rr);
        }
        rnorm = sqrt(cta_sum(rr));
      }
    }
    int64_t *out_sel = a.out_sel + p * kw;
    double *out_coef = a.out_coef + p * kw;
    for (int j = t; j < kw; j += NT) {
      out_sel[j] = j < kdone ? sup[j] : -1;
      out_coef[j] = j < kdone ? xv[j] : 0.0;
    }
    if (t == 0) {
      a.out_count[p] = kdone;
      a.out_rnorm[p] = rnorm;
      a.out_scans[p] = scans;
      a.out_flag[p] = 0;
    }
    __syncthreads();  // the next signal reuses the shared state
  }
}

// Two candidates per thread (256 threads, 8 warps: per-candidate overhead
// and the w broadcasts halve, the CTA barrier spans 8 warps): thread t owns
// candidates 2t and 2t + 1 -- one 16-byte shared-memory access per H row, one
// 16-byte Gram load per iteration for Q even.  Same arithmetic and order per
// candidate as gram_reg_kernel (row stride 512 in both).
template <int R>
__device__ __forceinline__ void load_block2(double (&h0)[R], double (&h1)[R], int b, const double *st) {
#pragma unroll
  for (int bb = 0; bb < R / 8; bb++) {
    if (bb == b) {
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const double2 v = *(const double2 *)(st + u * 512);
        h0[8 * bb + u] = v.x;
        h1[8 * bb + u] = v.y;
      }
    }
  }
}
template <int R>
__device__ __forceinline__ void put_regs_sel(double *dst, const double (&h0)[R], const double (&h1)[R],
                                             bool second, int kb) {
#pragma unroll
  for (int b = 0; b < R / 8; b++) {
    if (8 * b + 8 <= kb) {
#pragma unroll
      for (int u = 0; u < 8; u += 2)
        *(double2 *)(dst + 8 * b + u) =
            second ? make_double2(h1[8 * b + u], h1[8 * b + u + 1]) : make_double2(h0[8 * b + u], h0[8 * b + u + 1]);
    }
  }
}

template <typename YT, int R>
__global__ void __launch_bounds__(256, 1) gram_reg2_kernel(GramArgs a, const YT *__restrict__ ys) {
  constexpr int NT = 256, NW = NT / 32, NC = 512;
  static_assert(R % 8 == 0, "register rows come in blocks of 8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n = (int)a.n, kw = (int)a.k_width, smax = (int)a.max_cands;
  const int64_t T = a.t;
  const Cands cs = a.cands;
  const int nsr = kw > R ? kw - R : 0;
  constexpr int SL = 6 + R;
  double *hsm = (double *)smem_raw;                 // nsr x NC; thread t owns entries 2t, 2t + 1
  double *stg = hsm;                                // staging rows of the open register block
  double *slots = hsm + (int64_t)(nsr > 8 ? nsr : 8) * NC;  // [2][NW][SL]
  double *rm = a.hwork + (int64_t)blockIdx.x * kw * kw;
  double *zv = slots + 2 * NW * SL;
  double *iv = zv + kw;
  double *xv = iv + kw;
  int64_t *sup = (int64_t *)(xv + kw);
  double *red = (double *)(sup + kw);
  auto cta_sum = [&](double v) -> double {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; w++) s += red[w];
    return s;
  };
  const int j0 = 2 * t;
  const bool pairs = cs.mode == 2 && (cs.q & 1) == 0;  // 2t, 2t + 1 adjacent atoms

  for (int64_t local = blockIdx.x; local < a.p; local += gridDim.x) {
    const int64_t p = a.p_offset + local;
    const YT *yg = ys + p * a.ys_stride;
    const int S = (int)cs.count(p);
    const int k_max = (int)cs.budget(p, a.k_max, n);
    const bool va = j0 < S, vb = j0 + 1 < S;
    const int64_t cid0 = va ? cs.id(p, j0) : 0, cid1 = vb ? cs.id(p, j0 + 1) : 0;
    double yy = cta_sum(row_sumsq(yg, n, t, NT));
    const double ynorm = sqrt(yy);  // early exit |y| <= tol (_kernels.py:71-78)
    const double tol = a.eps[p];
    int kdone = 0;
    int64_t scans = 0;
    double rnorm = ynorm, rn2_final = 0.0;
    bool delegate = false;
    double h0[R], h1[R];
    int pick0 = -1, pick1 = -1;
    if (!(ynorm <= tol) && k_max > 0) {
#pragma unroll
      for (int i = 0; i < R; i++) h0[i] = h1[i] = 0.0;
      double c0 = va ? a.alpha0_in[p * smax + j0] : 0.0, c1 = vb ? a.alpha0_in[p * smax + j0 + 1] : 0.0;
      const double g00 = va ? __ldg(a.gram + cid0 * T + cid0) : 1.0;
      const double g11 = vb ? __ldg(a.gram + cid1 * T + cid1) : 1.0;
      double s0 = 0.0, s1 = 0.0;
      bool tk0 = !va, tk1 = !vb;
      double rn2 = yy;
      const double tol2 = tol * tol, band = 1e-12 * yy;
      int k = 0;
      for (;;) {
      bool check = false;
      for (; k < k_max; k++) {
        rn2_final = rn2;
        scans += S - k;
        const int par = k & 1;
        double *sbase = slots + par * NW * SL;
        // ---- thread best of two (lower index on ties), warp arg-max, publication
        const double a_ = tk0 ? 0.0 : fabs(c0), b_ = tk1 ? 0.0 : fabs(c1);
        const bool sec = b_ > a_;
        const double v = sec ? b_ : a_;
        const unsigned jt = (unsigned)(j0 + (sec ? 1 : 0));
        const double m = warp_max_nonneg(v);
        const unsigned wj = __reduce_min_sync(CDB_FULL_MASK, v == m ? jt : 0xffffffffu);
        if (jt == wj) {
          double *sl = sbase + warp * SL;
          sl[0] = m;
          sl[1] = sec ? c1 : c0;
          sl[2] = sec ? g11 - s1 : g00 - s0;
          sl[3] = sec ? g11 : g00;
          ((int64_t *)sl)[4] = ((sec ? cid1 : cid0) << 16) | (int64_t)jt;
          put_regs_sel<R>(sl + 6, h0, h1, sec, (k < R ? k : R) & ~7);
        }
        __syncthreads();
        const double mw = lane < NW ? sbase[lane * SL] : 0.0;
        const double gm = warp_max_nonneg(mw);
        if (!(gm > 0.0)) break;  // nothing left, or best <= 0 (_kernels.py:104)
        const int gw = __ffs(__ballot_sync(CDB_FULL_MASK, lane < NW && mw == gm)) - 1;
        const double *ws = sbase + gw * SL;
        const int64_t packed = ((const int64_t *)ws)[4];
        const int bestj = (int)(packed & 0xffff);
        const int64_t nid = packed >> 16;
        double gA = 0.0, gB = 0.0;
        if (pairs && vb) {
          const double2 g2 = __ldg((const double2 *)(a.gram + nid * T + cid0));
          gA = g2.x;
          gB = g2.y;
        } else {
          gA = va ? __ldg(a.gram + nid * T + cid0) : 0.0;
          gB = vb ? __ldg(a.gram + nid * T + cid1) : 0.0;
        }
        const double cj = ws[1], d2 = ws[2], gnn = ws[3];
        const double *w = ws + 6;
        // ---- sweep
        const int kr = k < R ? k : R, kb = kr & ~7;
        // 8 fma chains (4 per candidate): the sweep is bound by fp64 latency
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        double a2 = 0.0, a3 = 0.0, b2 = 0.0, b3 = 0.0;
#pragma unroll
        for (int b = 0; b < R / 8; b++) {
          if (8 * b + 8 <= kb) {
#pragma unroll
            for (int u = 0; u < 8; u += 4) {
              const double2 wv = *(const double2 *)(w + 8 * b + u);
              const double2 wx = *(const double2 *)(w + 8 * b + u + 2);
              a0 = fma(wv.x, h0[8 * b + u], a0);
              b0 = fma(wv.x, h1[8 * b + u], b0);
              a1 = fma(wv.y, h0[8 * b + u + 1], a1);
              b1 = fma(wv.y, h1[8 * b + u + 1], b1);
              a2 = fma(wx.x, h0[8 * b + u + 2], a2);
              b2 = fma(wx.x, h1[8 * b + u + 2], b2);
              a3 = fma(wx.y, h0[8 * b + u + 3], a3);
              b3 = fma(wx.y, h1[8 * b + u + 3], b3);
            }
          }
        }
        for (int i = kb; i < kr; i++) {
          const double wi = stg[(i & 7) * NC + bestj];
          const double2 hv = *(const double2 *)(stg + (i & 7) * NC + j0);
          a0 = fma(wi, hv.x, a0);
          b0 = fma(wi, hv.y, b0);
        }
        {
          int i = R;
          for (; i + 3 < k; i += 4) {
            const int64_t o = (int64_t)(i - R) * NC;
            const double w0 = hsm[o + bestj], w1 = hsm[o + NC + bestj];
            const double w2 = hsm[o + 2 * NC + bestj], w3 = hsm[o + 3 * NC + bestj];
            const double2 x0 = *(const double2 *)(hsm + o + j0), x1 = *(const double2 *)(hsm + o + NC + j0);
            const double2 x2 = *(const double2 *)(hsm + o + 2 * NC + j0), x3 = *(const double2 *)(hsm + o + 3 * NC + j0);
            a0 = fma(w0, x0.x, a0);
            b0 = fma(w0, x0.y, b0);
            a1 = fma(w1, x1.x, a1);
            b1 = fma(w1, x1.y, b1);
            a2 = fma(w2, x2.x, a2);
            b2 = fma(w2, x2.y, b2);
            a3 = fma(w3, x3.x, a3);
            b3 = fma(w3, x3.y, b3);
          }
          for (; i + 1 < k; i += 2) {
            const int64_t o = (int64_t)(i - R) * NC;
            const double w0 = hsm[o + bestj], w1 = hsm[o + NC + bestj];
            const double2 x0 = *(const double2 *)(hsm + o + j0), x1 = *(const double2 *)(hsm + o + NC + j0);
            a0 = fma(w0, x0.x, a0);
            b0 = fma(w0, x0.y, b0);
            a1 = fma(w1, x1.x, a1);
            b1 = fma(w1, x1.y, b1);
          }
          if (i < k) {
            const int64_t o = (int64_t)(i - R) * NC;
            const double w0 = hsm[o + bestj];
            const double2 x0 = *(const double2 *)(hsm + o + j0);
            a0 = fma(w0, x0.x, a0);
            b0 = fma(w0, x0.y, b0);
          }
        }
        if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine decides
          delegate = true;
          break;
        }
        const double inv_d = rsqrt(d2);
        const double zk = cj * inv_d;  // q_k^T y = <d_{j*}, r> / d
        const double hA = va ? (gA - ((a0 + a1) + (a2 + a3))) * inv_d : 0.0;
        const double hB = vb ? (gB - ((b0 + b1) + (b2 + b3))) * inv_d : 0.0;
        if ((bestj >> 1) == t) {
          if (bestj & 1) {
            tk1 = true;
            pick1 = k;
          } else {
            tk0 = true;
            pick0 = k;
          }
          zv[k] = zk;
          iv[k] = inv_d;
          sup[k] = nid;
        }
        if (k < R) {
          *(double2 *)(stg + (k & 7) * NC + j0) = make_double2(hA, hB);
          if ((k & 7) == 7) load_block2<R>(h0, h1, k >> 3, stg + j0);
        } else {
          *(double2 *)(hsm + (int64_t)(k - R) * NC + j0) = make_double2(hA, hB);
        }
        c0 = fma(-zk, hA, c0);
        c1 = fma(-zk, hB, c1);
        s0 = fma(hA, hA, s0);
        s1 = fma(hB, hB, s1);
        rn2 -= zk * zk;
        rn2_final = rn2;
        kdone = k + 1;
        const double gap = rn2 - tol2;  // stop test (_kernels.py:156)
        if (gap > band) continue;
        if (gap < -band) break;
        check = true;
        break;
      }
      if (!check) break;
      file_col<R>(rm, kw, pick0, h0, stg + j0, hsm + j0, kdone);
      file_col<R>(rm, kw, pick1, h1, stg + j0 + 1, hsm + j0 + 1, kdone);
      __syncthreads();
      if (warp == 0) back_sub_cols(rm, kw, kdone, zv, iv, xv, lane);
      __syncthreads();
      double rr = 0.0;
      for (int i = t; i < n; i += NT) {
        double ri = (double)yg[i];
        for (int l = 0; l < kdone; l++) ri = fma(-xv[l], a.d64[sup[l] * n + i], ri);
        rr = fma(ri, ri, rr);
      }
      rr = cta_sum(rr);
      if (sqrt(rr) <= tol) break;
      k++;
      }
    }
    __syncthreads();
    if (delegate) {
      if (t == 0) a.status[p] |= ST_DELEGATE;
      __syncthreads();
      continue;
    }
    file_col<R>(rm, kw, pick0, h0, stg + j0, hsm + j0, kdone);
    file_col<R>(rm, kw, pick1, h1, stg + j0 + 1, hsm + j0 + 1, kdone);
    __syncthreads();
    if (warp == 0) back_sub_cols(rm, kw, kdone, zv, iv, xv, lane);
    __syncthreads();
    if (kdone > 0) {
      if (rn2_final > 1e-6 * yy) {
        rnorm = sqrt(rn2_final);
      } else {
        double rr = 0.0;
        for (int i = t; i < n; i += NT) {
          double ri = (double)yg[i];
          for (int l = 0; l < kdone; l++) ri = fma(-xv[l], __ldg(a.d64 + sup[l] * n + i), ri);
          rr = fma(ri, ri, rr);
        }
        rnorm = sqrt(cta_sum(rr));
      }
    }
    int64_t *out_sel = a.out_sel + p * kw;
    double *out_coef = a.out_coef + p * kw;
    for (int j = t; j < kw; j += NT) {
      out_sel[j] = j < kdone ? sup[j] : -1;
      out_coef[j] = j < kdone ? xv[j] : 0.0;
    }
    if (t == 0) {
      a.out_count[p] = kdone;
      a.out_rnorm[p] = rnorm;
      a.out_scans[p] = scans;
      a.out_flag[p] = 0;
    }
    __syncthreads();
  }
}

template <typename YT, int R>
cudaError_t go_reg2(const GramArgs &args, const YT *ys, const GramStreamPlan &pl,
                    cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(gram_reg2_kernel<YT, R>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pl.per_warp_smem);
  if (e != cudaSuccess) return e;
  gram_reg2_kernel<YT, R><<<(unsigned)pl.warps, 256, pl.per_warp_smem, stream>>>(args, ys);
  return cudaGetLastError();
}

template <typename YT, int R>
cudaError_t go_reg(const GramArgs &args, const YT *ys, const GramStreamPlan &pl,
                   cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(gram_reg_kernel<YT, R>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pl.per_warp_smem);
  if (e != cudaSuccess) return e;
  gram_reg_kernel<YT, R><<<(unsigned)pl.warps, 512, pl.per_warp_smem, stream>>>(args, ys);
  return cudaGetLastError();
}

template <typename YT>
cudaError_t go_reg_r(const GramArgs &args, const YT *ys, const GramStreamPlan &pl,
                     cudaStream_t stream) {
  if (pl.cpt == 2) switch (pl.nr) {
      case 16: return go_reg2<YT, 16>(args, ys, pl, stream);
      case 24: return go_reg2<YT, 24>(args, ys, pl, stream);
      case 32: return go_reg2<YT, 32>(args, ys, pl, stream);
    }
  switch (pl.nr) {
    case 16: return go_reg<YT, 16>(args, ys, pl, stream);
    case 24: return go_reg<YT, 24>(args, ys, pl, stream);
    case 32: return go_reg<YT, 32>(args, ys, pl, stream);
  }
  return cudaErrorInvalidValue;
}

template <typename YT, int CPT>
cudaError_t go_tma(const GramArgs &args, const YT *ys, const GramStreamPlan &pl,
                   cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(gram_tma_kernel<YT, CPT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pl.per_warp_smem);
  if (e != cudaSuccess) return e;
  gram_tma_kernel<YT, CPT><<<(unsigned)pl.warps, 128, pl.per_warp_smem, stream>>>(args, ys, pl.nr);
  return cudaGetLastError();
}

template <typename YT, int CPT>
cudaError_t go_cta(const GramArgs &args, const YT *ys, const GramStreamPlan &pl,
                   cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(gram_cta_kernel<YT, CPT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pl.per_warp_smem);
  if (e != cudaSuccess) return e;
  gram_cta_kernel<YT, CPT><<<(unsigned)pl.warps, 128, pl.per_warp_smem, stream>>>(args, ys, pl.nr);
  return cudaGetLastError();
}

template <typename YT, int U, int HM>
cudaError_t launch_gram_tuh(const GramArgs &args, const YT *ys, int h_in_smem, int64_t per_warp,
                            int wpb, int64_t blocks, cudaStream_t stream) {
  const int64_t smem = per_warp * wpb;
  cudaError_t e = cudaFuncSetAttribute(gram_omp_kernel<YT, U, HM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  gram_omp_kernel<YT, U, HM><<<(unsigned)blocks, wpb * 32, smem, stream>>>(args, ys, h_in_smem,
                                                                           per_warp);
  return cudaGetLastError();
}

template <typename YT, int U>
cudaError_t launch_gram_tu(const GramArgs &args, const YT *ys, int h_in_smem, int64_t per_warp,
                           int wpb, int64_t blocks, cudaStream_t stream) {
  if (args.hwork == nullptr)
    return launch_gram_tuh<YT, U, 1>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
  if (gram_stream_tmem(wpb))
    return launch_gram_tuh<YT, U, 2>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
  return launch_gram_tuh<YT, U, 0>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
}

template <typename YT>
cudaError_t launch_gram_y(const GramArgs &args, const YT *ys, int u, int h_in_smem,
                          int64_t per_warp, int wpb, int64_t blocks, cudaStream_t stream) {
  switch (u) {
    case 1: return launch_gram_tu<YT, 1>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 2: return launch_gram_tu<YT, 2>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 4: return launch_gram_tu<YT, 4>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 6: return launch_gram_tu<YT, 6>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 8: return launch_gram_tu<YT, 8>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 12: return launch_gram_tu<YT, 12>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
    case 16: return launch_gram_tu<YT, 16>(args, ys, h_in_smem, per_warp, wpb, blocks, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int64_t gram_h_doubles(int64_t max_cands, int64_t kw) { return kw * gram_hs(max_cands); }

// The warp-per-signal kernel keeps 3 signals (3 warps) per SM once H passes
// ~64 KB; three 128-thread CTAs per SM with every row in shared memory hold as
// many signals with four times the threads on each chain.  cfg 2 step 2
// (S = 256, K = 32, 200 k signals): 26.7 -> 20.3 ms (2 / 4 CTAs per SM: 28.6 /
// 30.1 ms; the on-chip register kernel 55.4 ms); S = 384 (cfg 3) keeps the warp
// kernel: 12.5 ms per 100 k against 15.1 ms with rows padded to 512 candidates
// (2 CTAs per SM) and 16.3 ms with three 192-thread CTAs of exact 384-wide rows.
constexpr int kSmallCtasPerSm = 3;
bool gram_cta_preferred(int64_t s, int64_t kw, int64_t n, bool has_alpha0) {
  static const bool off = getenv("CDB_GRAM_CTA3") && atoi(getenv("CDB_GRAM_CTA3")) == 0;
  if (off || !has_alpha0 || s <= 128 || s > 256 || kw > 64) return false;
  const int64_t fixed = 8 * (5 * kw + 9 * 4 + 2 + 2);
  const int64_t per_cta = (int64_t)(228 * 1024) / kSmallCtasPerSm - 1024;
  return fixed + 8 * kw * 256 <= per_cta && gram_total_smem(s, kw, n, true) > 40 * 1024;
}

GramStreamPlan gram_stream_plan(int64_t s, int64_t kw, int64_t n, bool stage_y,
                                int max_smem_per_block, int num_sms) {
  GramStreamPlan pl{};
  const bool small_cta = gram_cta_preferred(s, kw, n, !stage_y);
  // on-chip H, one CTA per SM holding one signal's whole H: registers (R rows)
  // + shared memory.  Default: gram_reg2_kernel (256 threads, two candidates
  // per thread, R = 24): cfg 4 step 2, 131,072 signals: 87.8 ms against 93.8 ms
  // for the streamed CTA kernel below (CDB_GRAM_REG=0) and 99.8 ms for
  // gram_reg_kernel (one candidate per thread, CDB_GRAM_REG=1; R = 16 / 24 / 32:
  // CDB_GRAM_R).  One signal per SM leaves its per-iteration chain (arg-max,
  // barrier, Gram-row gather from HBM) exposed; what it saves is the L2 row
  // traffic of the streamed kernel.
  const char *rv = getenv("CDB_GRAM_REG");
  const int regmode = rv ? atoi(rv) : 2;
  if (!stage_y && s <= 512 && kw <= 64 && regmode != 0 && !small_cta) {
    int r = regmode == 2 ? 24 : 16;
    if (const char *v = getenv("CDB_GRAM_R")) r = atoi(v);
    if (r != 16 && r != 24 && r != 32) r = regmode == 2 ? 24 : 16;
    const int64_t nsr = kw > r ? kw - r : 0;
    const int64_t sl = 6 + r;
    const int64_t dbl = (nsr > 8 ? nsr : 8) * 512 + 2 * 16 * sl + 4 * kw + 16;
    pl.per_warp_smem = (8 * dbl + 15) & ~int64_t(15);  // per CTA
    pl.ok = pl.per_warp_smem <= max_smem_per_block;
    if (pl.ok) {
      pl.reg = true;
      pl.cta = true;
      pl.cpt = regmode == 2 ? 2 : 1;
      pl.wpb = pl.cpt == 2 ? 8 : 16;
      pl.nr = r;
      pl.warps = num_sms;  // CTAs
      pl.slot_doubles = kw * kw;  // the CTA's R matrix
      return pl;
    }
    pl = GramStreamPlan{};
  }
  const char *cv = getenv("CDB_GRAM_CTA");
  if (!stage_y && s <= 512 && kw <= 64 && (small_cta || !(cv && atoi(cv) == 0))) {
    // CTA per signal (gram_cta_kernel): cps CTAs per SM share its shared memory
    int cps = small_cta ? kSmallCtasPerSm : kStreamCtasPerSm;
    if (const char *v = getenv("CDB_GRAM_CPS")) cps = atoi(v) > 0 ? atoi(v) : cps;
    const int cpt = s <= 256 ? 2 : 4;
    const int64_t sp = 128 * cpt;
    const int64_t fixed = 8 * (5 * kw + 9 * 4 + 2 + 2);
    int64_t per_cta = (int64_t)(228 * 1024) / cps - 1024;
    if (per_cta > max_smem_per_block) per_cta = max_smem_per_block;
    // TMA-streamed rows (opt-in CDB_GRAM_TMA=1; a ring of kRingSlots rows + its
    // mbarriers comes out of the shared rows).  Measured on cfg 4 (65,536
    // signals, bit-identical results): 102.3 ms against 47.8 ms for the
    // register-pipelined kernel -- 8 ring slots (32 KB) keep half the bytes in
    // flight of its 16 rows x 128 threads of registers, the bulk-copy latency is
    // longer than an L2 load's, and every refill waits for the whole CTA.
    const char *tv = getenv("CDB_GRAM_TMA");
    const bool tma = tv && atoi(tv) != 0;
    const int64_t ring = tma ? kRingSlots * 8 * sp + 16 * kRingSlots + 16 : 0;
    int64_t nr = (per_cta - fixed - ring) / (8 * sp);
    if (nr > kw) nr = kw;
    if (nr < 0) nr = 0;
    pl.ok = per_cta > fixed + ring;
    pl.tma = tma && nr < kw;
    if (!pl.tma && tma) nr = (per_cta - fixed) / (8 * sp) > kw ? kw : (per_cta - fixed) / (8 * sp);
    pl.cta = true;
    pl.cpt = cpt;
    pl.wpb = 4;
    pl.nr = (int)nr;
    pl.per_warp_smem = (fixed + 8 * nr * sp + (pl.tma ? ring : 0) + 15) & ~int64_t(15);  // per CTA
    pl.warps = (int64_t)num_sms * cps;                                // CTAs
    pl.slot_doubles = (kw - nr) * sp;
    return pl;
  }
  const int64_t hs = gram_hs(s);
  int wpb = kStreamWarpsPerSm;
  if (const char *v = getenv("CDB_GRAM_WPB")) wpb = atoi(v) > 0 ? atoi(v) : wpb;
  if (wpb > 32) wpb = 32;
  const int64_t fixed = 8 * ((5 * kw + 16 + 1) & ~int64_t(1));  // + the TMEM column scratch
  int64_t per_warp = ((int64_t)max_smem_per_block / wpb) & ~int64_t(15);
  // shared memory only holds whole H rows (plus the y / alpha0 staging if needed)
  int64_t region = per_warp - fixed;
  int64_t nr = region > 0 ? region / (8 * hs) : 0;
  if (nr > kw) nr = kw;
  const int64_t need = stage_y ? n + s : 0;
  int64_t rd = nr * hs > need ? nr * hs : need;
  per_warp = (fixed + 8 * rd + 15) & ~int64_t(15);
  pl.ok = per_warp <= max_smem_per_block / wpb && per_warp > fixed;
  pl.wpb = wpb;
  pl.nr = (int)nr;
  pl.per_warp_smem = per_warp;
  pl.warps = (int64_t)num_sms * wpb;
  const int64_t ntr = gram_stream_tmem(wpb) ? (kw - nr < 16 ? kw - nr : 16) : 0;
  pl.slot_doubles = (kw - nr - ntr) * hs;
  return pl;
}

int64_t gram_total_smem(int64_t s, int64_t kw, int64_t n, bool h_in_smem) {
  const int64_t b = 8 * (((5 * kw + 1) & ~int64_t(1)) + gram_region_doubles(s, kw, n, h_in_smem));
  return (b + 15) & ~int64_t(15);
}

cudaError_t launch_gram(const GramArgs &args, const void *ys, bool ys_f32, int max_smem_per_block,
                        int num_sms, cudaStream_t stream) {
  ProfScope _ps(args.tag ? args.tag : "gram_omp", stream);
  (void)num_sms;
  if (args.p <= 0) return cudaSuccess;
  const int64_t s = args.max_cands, kw = args.k_width, n = args.n;
  const bool h_in_smem = args.hwork == nullptr;
  if (kw > 64 || s > 512) return cudaErrorInvalidValue;
  if (!h_in_smem) {  // streamed H: persistent warps, one block per SM
    const GramStreamPlan pl = gram_stream_plan(s, kw, n, args.alpha0_in == nullptr,
                                               max_smem_per_block, num_sms);
    if (!pl.ok) return cudaErrorInvalidValue;
    if (pl.reg) {  // H on chip, CTA per signal
      note_launch();
      return ys_f32 ? go_reg_r<float>(args, (const float *)ys, pl, stream)
                    : go_reg_r<double>(args, (const double *)ys, pl, stream);
    }
    if (pl.cta && pl.tma) {  // CTA per signal, L2 rows streamed by bulk copies
      note_launch();
      if (ys_f32)
        return pl.cpt == 2 ? go_tma<float, 2>(args, (const float *)ys, pl, stream)
                           : go_tma<float, 4>(args, (const float *)ys, pl, stream);
      return pl.cpt == 2 ? go_tma<double, 2>(args, (const double *)ys, pl, stream)
                         : go_tma<double, 4>(args, (const double *)ys, pl, stream);
    }
    if (pl.cta) {  // CTA per signal
      note_launch();
      if (ys_f32)
        return pl.cpt == 2 ? go_cta<float, 2>(args, (const float *)ys, pl, stream)
                           : go_cta<float, 4>(args, (const float *)ys, pl, stream);
      return pl.cpt == 2 ? go_cta<double, 2>(args, (const double *)ys, pl, stream)
                         : go_cta<double, 4>(args, (const double *)ys, pl, stream);
    }
    const int u = (int)(gram_hs(s) / 32);
    note_launch();
    if (ys_f32)
      return launch_gram_y<float>(args, (const float *)ys, u, pl.nr, pl.per_warp_smem, pl.wpb,
                                  num_sms, stream);
    return launch_gram_y<double>(args, (const double *)ys, u, pl.nr, pl.per_warp_smem, pl.wpb,
                                 num_sms, stream);
  }
  const int64_t per_warp = gram_total_smem(s, kw, n, h_in_smem);
  if (per_warp > max_smem_per_block) return cudaErrorInvalidValue;
  const int u = (int)(gram_hs(s) / 32);
  const int cap = u <= 8 ? 16 : 8;
  int max_w = (int)(max_smem_per_block / per_warp);
  if (max_w > cap) max_w = cap;
  int wpb = max_w;
  if (const char *v = getenv("CDB_GRAM_WPB")) wpb = atoi(v) < max_w ? atoi(v) : max_w;
  if (wpb < 1) wpb = 1;
  const int64_t blocks = (args.p + wpb - 1) / wpb;
  note_launch();
  if (ys_f32)
    return launch_gram_y<float>(args, (const float *)ys, u, (int)kw, per_warp, wpb, blocks,
                                stream);
  return launch_gram_y<double>(args, (const double *)ys, u, (int)kw, per_warp, wpb, blocks,
                               stream);
}

}  // namespace cdb
