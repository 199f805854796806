// Resident engine: batched OMP for dictionaries small enough to live in
// shared memory (8*N*T bytes <= ~128 KB: cfg 0 entirely, the cfg 1 coarse
// step).  One persistent CTA per SM holds the fp64 dictionary transposed
// (Dt[i][j], so a lane reading its atoms for a fixed i is bank-conflict
// free); each warp runs whole signals, all iterations, with the residual in
// fp64 shared memory -- the reference's algorithm (_kernels.py:68-168) with
// direct correlations <d_j, r> (lane per candidate), strict '>' selection,
// the least squares as an incremental Cholesky of the support Gram (computed
// from the resident atoms, kept as L^{-1}), and the residual re-materialised
// as y - D_S x every iteration.  Correlations and |r| are fp64 dots of the
// same vectors as the reference in a different summation order (~1e-16
// relative).  Near rank deficiency is delegated to the exact engine.
#include <cstdlib>

#include "candidates.cuh"
#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

// 16-byte shared-memory load (LDS.128; the compiler otherwise splits it)
__device__ __forceinline__ float4 lds128(const void *p) {
  float4 v;
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}

// packed fp32 FMA (FFMA2): two independent fma.rn in one instruction
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  const unsigned long long A = (unsigned long long)__float_as_uint(a.x) |
                               ((unsigned long long)__float_as_uint(a.y) << 32);
  const unsigned long long B = (unsigned long long)__float_as_uint(b.x) |
                               ((unsigned long long)__float_as_uint(b.y) << 32);
  const unsigned long long C = (unsigned long long)__float_as_uint(c.x) |
                               ((unsigned long long)__float_as_uint(c.y) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(A), "l"(B), "l"(C));
  return make_float2(__uint_as_float((unsigned)d), __uint_as_float((unsigned)(d >> 32)));
}

constexpr int RES_WARPS = 16;   // warps per CTA (512 threads)


// FULL: candidate jl of lane l is atom l + 32u (mode 0) -> compile-time
// shared-memory offsets in the correlation loop.  R signals per warp share
// every dictionary element loaded from shared memory (R FMAs per LDS).
//
// Per signal (shared memory, doubles): r (n), L^{-1} (k_width rows, odd
// stride), z, w, g, x (k_width each), support ids.  Taken bits, candidate
// ids and correlations live in registers.  Per iteration: argmax (fmax
// butterfly + redux.min for the lowest index among equal maxima), Cholesky
// append through the Gram row (w = L^{-1} g, d^2 = |d_new|^2 - |w|^2), the
// new L^{-1} row, and the residual update r -= z_k q_k with
// q_k = sum_l L^{-1}[k][l] d_{s_l} read from the resident atoms; the
// coefficients x = L^{-T} z are formed once at the end.
//
// F32C: the correlations are fp32 dots of an fp32 copy of the resident atoms
// with an fp32 copy of the residual (half the shared-memory bytes of the
// fp64 scan, FP32 pipe), certified against the exact fp64 values: with
// E = (N + 2) 2^-24 max|d| |r| (fp32 accumulation over N terms plus the
// rounding of both operands), any candidate whose approximate |c| is below
// max - 2E cannot be the fp64 arg-max.  When exactly one candidate is in
// the window it is the pick; otherwise the window is re-scored in fp64.  The
// winner's correlation (z_k = c / d) is always recomputed in fp64.  Layout:
// the fp32 atoms are interleaved per dimension as [U/4][lane][4] (atoms
// lane + 32 (4w + c)), one conflict-free 16-byte load per lane per 4 atoms,
// and accumulated pairwise with FFMA2; the fp32 residual is stored
// duplicated ({r_i, r_i}) so one 16-byte load feeds two dimensions.
// F32C requires FULL and U >= 4.
template <typename YT, int U, bool FULL, int R, bool F32C>
__global__ void __launch_bounds__(R >= 4 ? 384 : (R == 1 ? 1024 : 512), 1)
    resident_omp_kernel(ResidentArgs a, const YT *__restrict__ ys) {
  extern __shared__ __align__(16) double rs[];
  const int n = (int)a.n, T = (int)a.t, kw = (int)a.k_width, Tp = (int)a.t_pad;
  const int ldl = kw | 1;  // odd L^{-1} row stride: column walks hit distinct banks
  const int64_t P = a.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double *Dt = rs;                 // n x Tp  (columns T..Tp-1 are zero)
  double *nrm2 = Dt + n * Tp;      // Tp  (|d_j|^2)
  const int n2 = (n + 1) & ~1;    // F32C rows (zero row when n is odd)
  float *Df = (float *)(rs + ((n * Tp + Tp + 1) & ~1));  // F32C: n2 x 32U fp32 (16-B aligned)
  double *wbase = F32C ? (double *)(Df + n2 * 32 * U) : nrm2 + Tp;
  const int per_sig = (int)a.per_warp;  // doubles of state per signal
  __shared__ double s_dmax;

  for (int e = threadIdx.x; e < n * Tp; e += blockDim.x) {
    const int i = e / Tp, j = e % Tp;
    Dt[e] = j < T ? a.d64[(int64_t)j * n + i] : 0.0;
  }
  if (F32C)
    for (int e = threadIdx.x; e < n2 * 32 * U; e += blockDim.x) {
      const int i = e / (32 * U), rem = e % (32 * U);
      const int j = (rem % 128) / 4 + 32 * (4 * (rem / 128) + rem % 4);
      Df[e] = i < n && j < T ? (float)a.d64[(int64_t)j * n + i] : 0.0f;
    }
  __syncthreads();
  for (int j = threadIdx.x; j < Tp; j += blockDim.x) {
    double sq = 0.0;
    for (int i = 0; i < n; i++) sq = fma(Dt[i * Tp + j], Dt[i * Tp + j], sq);
    nrm2[j] = sq;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double mx = 0.0;
    for (int j = threadIdx.x; j < Tp; j += 32) mx = fmax(mx, nrm2[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(CDB_FULL_MASK, mx, o));
    if (threadIdx.x == 0) s_dmax = sqrt(mx);
  }
  __syncthreads();
  // |c~ - c| <= e_rel |r|  (F32C certification bound, 1% slack)
  const double e_rel = (double)(n + 2) * 0x1p-24 * 1.01 * s_dmax;
  const int r32_off = (n + kw * ldl + 5 * kw + 2) & ~1;  // doubles (even): fp32 residual pairs

  const Cands cs = a.cands;
  const double *eps = a.eps;
  const double *gram = a.gram;
  double *sbase = wbase + warp * R * per_sig;
  for (int64_t p0 = ((int64_t)blockIdx.x * nwarps + warp) * R; p0 < P;
       p0 += (int64_t)gridDim.x * nwarps * R) {
    // ---- per-signal setup
    int kmax[R], kdone[R], S[R];
    int64_t scans[R];
    double tol[R], rnorm[R];
    bool live[R], delegate[R];
    unsigned tk[R];  // bit u: candidate lane + 32u taken or beyond S
    int cid[R][U];
#pragma unroll
    for (int q = 0; q < R; q++) {
      const int64_t p = p0 + q;
      double *r = sbase + q * per_sig;
      const bool valid = p < P;
      S[q] = valid ? (int)cs.count(p) : 0;
      kmax[q] = valid ? (int)cs.budget(p, a.k_max, n) : 0;
      tk[q] = 0u;
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int jl = lane + 32 * u;
        cid[q][u] = FULL ? jl : (jl < S[q] ? (int)cs.id(p, jl) : Tp - 1);
        if (jl >= S[q]) tk[q] |= 1u << u;
      }
      for (int i = lane; i < n2; i += 32) {
        const double v = valid && i < n ? (double)ys[p * n + i] : 0.0;
        if (i < n) r[i] = v;
        if (F32C) ((float2 *)(r + r32_off))[i] = make_float2((float)v, (float)v);
      }
      __syncwarp();
      const double ynorm = sqrt(dot4_quad(r, r, n, lane));  // reference order (_kernels.py:71)
      tol[q] = valid ? eps[p] : 0.0;
      rnorm[q] = ynorm;
      kdone[q] = 0;
      scans[q] = 0;
      delegate[q] = false;
      live[q] = valid && !(ynorm <= tol[q]) && kmax[q] > 0;
    }
    for (int k = 0;; k++) {
      bool any = false;
#pragma unroll
      for (int q = 0; q < R; q++) {
        if (live[q] && k >= kmax[q]) live[q] = false;
        any |= live[q];
      }
      if (!any) break;
      // ---- correlations of this lane's candidates with each live residual
      double acc[R][U];
      if constexpr (F32C) {
        float2 af[R][U / 2];
#pragma unroll
        for (int q = 0; q < R; q++)
#pragma unroll
          for (int v = 0; v < U / 2; v++) af[q][v] = make_float2(0.0f, 0.0f);
        const float4 *dcol = (const float4 *)Df + lane;
#pragma unroll 2
        for (int i = 0; i < n2; i += 2) {
          float4 rq[R];
#pragma unroll
          for (int q = 0; q < R; q++)
            rq[q] = lds128((const float4 *)(sbase + q * per_sig + r32_off) + i / 2);
#pragma unroll
          for (int ii = 0; ii < 2; ii++) {
            const float4 *row = dcol + (i + ii) * 8 * U;
#pragma unroll
            for (int w = 0; w < U / 4; w++) {
              const float4 d = lds128(row + 32 * w);
#pragma unroll
              for (int q = 0; q < R; q++) {
                const float2 b = ii ? make_float2(rq[q].z, rq[q].w) : make_float2(rq[q].x, rq[q].y);
                af[q][2 * w] = ffma2(make_float2(d.x, d.y), b, af[q][2 * w]);
                af[q][2 * w + 1] = ffma2(make_float2(d.z, d.w), b, af[q][2 * w + 1]);
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < R; q++)
#pragma unroll
          for (int v = 0; v < U / 2; v++) {
            acc[q][2 * v] = (double)af[q][v].x;
            acc[q][2 * v + 1] = (double)af[q][v].y;
          }
      } else {
#pragma unroll
        for (int q = 0; q < R; q++)
#pragma unroll
          for (int u = 0; u < U; u++) acc[q][u] = 0.0;
        const double *col = FULL ? Dt + lane : Dt;
#pragma unroll 2
        for (int i = 0; i < n; i++) {
          double ri[R];
#pragma unroll
          for (int q = 0; q < R; q++) ri[q] = sbase[q * per_sig + i];
          const double *row = col + i * Tp;
#pragma unroll
          for (int u = 0; u < U; u++) {
            if (FULL) {
              const double dv = row[32 * u];
#pragma unroll
              for (int q = 0; q < R; q++) acc[q][u] = fma(dv, ri[q], acc[q][u]);
            } else {
#pragma unroll
              for (int q = 0; q < R; q++) acc[q][u] = fma(row[cid[q][u]], ri[q], acc[q][u]);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < R; q++) {
        if (!live[q]) continue;
        double *r = sbase + q * per_sig;
        double *lin = r + n;
        double *zv = lin + kw * ldl;
        double *wv = zv + kw;
        double *gv = wv + kw;
        int *sup = (int *)(gv + 2 * kw);
        scans[q] += S[q] - k;
        // ---- selection: max |c| over available candidates, ties -> lowest index
        double best = -1.0;
        unsigned bj = 0xffffffffu;
#pragma unroll
        for (int u = 0; u < U; u++) {
          const double v = fabs(acc[q][u]);
          if (!((tk[q] >> u) & 1u) && v > best) {
            best = v;
            bj = lane + 32 * u;
          }
        }
        double m = best;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(CDB_FULL_MASK, m, o));
        int bestj;
        double cbest;
        if constexpr (F32C) {
          // certification window [m - 2E, m] of the fp32 scan
          const double thr = m - 2.0 * e_rel * rnorm[q];
          int cnt = 0;
#pragma unroll
          for (int u = 0; u < U; u++)
            if (!((tk[q] >> u) & 1u) && fabs(acc[q][u]) >= thr) cnt++;
          cnt = (int)__reduce_add_sync(CDB_FULL_MASK, (unsigned)cnt);
          if (cnt == 0) {  // nothing available (_kernels.py:104)
            live[q] = false;
            continue;
          }
          if (cnt > 1) {
            // re-score the window exactly in fp64 (lane per candidate)
            best = -1.0;
            bj = 0xffffffffu;
#pragma unroll
            for (int u = 0; u < U; u++) {
              if (!((tk[q] >> u) & 1u) && fabs(acc[q][u]) >= thr) {
                const int jj = FULL ? lane + 32 * u : cid[q][u];
                double c = 0.0;
                for (int i = 0; i < n; i++) c = fma(Dt[i * Tp + jj], r[i], c);
                acc[q][u] = c;
                if (fabs(c) > best) {
                  best = fabs(c);
                  bj = lane + 32 * u;
                }
              }
            }
            m = best;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(CDB_FULL_MASK, m, o));
          }
          bestj = (int)__reduce_min_sync(CDB_FULL_MASK, best == m ? bj : 0xffffffffu);
        } else {
          if (!(m > 0.0)) {  // nothing left, or best <= 0 (_kernels.py:104)
            live[q] = false;
            continue;
          }
          bestj = (int)__reduce_min_sync(CDB_FULL_MASK, best == m ? bj : 0xffffffffu);
        }
        const int ub = bestj >> 5, owner = bestj & 31;
        double my_c = 0.0;
        int my_id = 0;
#pragma unroll
        for (int u = 0; u < U; u++)
          if (u == ub) {
            my_c = acc[q][u];
            my_id = cid[q][u];
          }
        cbest = __shfl_sync(CDB_FULL_MASK, my_c, owner);
        const int nid = FULL ? bestj : __shfl_sync(CDB_FULL_MASK, my_id, owner);
        if constexpr (F32C) {
          // the winner's exact correlation (z_k = c / d); orthogonal break on it
          double c = 0.0;
          for (int i = lane; i < n; i += 32) c = fma(Dt[i * Tp + nid], r[i], c);
          cbest = warp_sum(c);
          if (!(fabs(cbest) > 0.0)) {  // _kernels.py:104
            live[q] = false;
            continue;
          }
        }
        if (lane == owner) tk[q] |= 1u << ub;
        // ---- Cholesky append: g_l = <d_{s_l}, d_new> (Gram row gather, or a
        // dot over the resident atoms when no Gram matrix is staged)
        if (gram) {
          const double *grow = gram + (int64_t)nid * T;
          for (int l = lane; l < k; l += 32) gv[l] = __ldg(grow + sup[l]);
        } else {
          for (int l = lane; l < k; l += 32) {
            double g = 0.0;
            const int sl = sup[l];
            for (int i = 0; i < n; i++) g = fma(Dt[i * Tp + sl], Dt[i * Tp + nid], g);
            gv[l] = g;
          }
        }
        if (lane == 0) sup[k] = nid;
        __syncwarp();
        for (int l = lane; l < k; l += 32) {
          double accw = 0.0;
#pragma unroll 4
          for (int i = 0; i <= l; i++) accw = fma(lin[l * ldl + i], gv[i], accw);
          wv[l] = accw;
        }
        __syncwarp();
        double ww = 0.0;
        for (int l = lane; l < k; l += 32) ww = fma(wv[l], wv[l], ww);
        ww = warp_sum(ww);
        const double gnn = nrm2[nid];
        const double d2 = gnn - ww;
        if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {
          delegate[q] = true;
          live[q] = false;
          continue;
        }
        const double inv_d = rsqrt(d2);
        const double zk = cbest * inv_d;  // q_k^T y = q_k^T r = <d_new, r> / d
        for (int i = lane; i <= k; i += 32) {
          double v;
          if (i == k) {
            v = inv_d;
          } else {
            double accl = 0.0;
#pragma unroll 4
            for (int l = i; l < k; l++) accl = fma(wv[l], lin[l * ldl + i], accl);
            v = -accl * inv_d;
          }
          lin[k * ldl + i] = v;
        }
        if (lane == 0) zv[k] = zk;
        __syncwarp();
        kdone[q] = k + 1;
        // ---- residual r -= z_k q_k,  q_k = sum_l L^{-1}[k][l] d_{s_l}; stop test
        const double *lk = lin + k * ldl;
        double rr = 0.0;
        for (int i = lane; i < n; i += 32) {
          const double *row = Dt + i * Tp;
          double qv = 0.0;
#pragma unroll 4
          for (int l = 0; l <= k; l++) qv = fma(lk[l], row[sup[l]], qv);
          const double rv = fma(-zk, qv, r[i]);
          r[i] = rv;
          if (F32C) ((float2 *)(r + r32_off))[i] = make_float2((float)rv, (float)rv);
          rr = fma(rv, rv, rr);
        }
        rnorm[q] = sqrt(warp_sum(rr));
        __syncwarp();
        if (rnorm[q] <= tol[q]) live[q] = false;
      }
    }
    // ---- outputs: x = L^{-T} z (pick order)
#pragma unroll
    for (int q = 0; q < R; q++) {
      const int64_t p = p0 + q;
      if (p >= P) continue;
      if (delegate[q]) {
        if (lane == 0) a.status[p] |= ST_DELEGATE;
        continue;
      }
      double *lin = sbase + q * per_sig + n;
      double *zv = lin + kw * ldl;
      int *sup = (int *)(zv + 4 * kw);
      int64_t *out_sel = a.out_sel + p * kw;
      double *out_coef = a.out_coef + p * kw;
      const int kd = kdone[q];
      for (int j = lane; j < kw; j += 32) {
        double x = 0.0;
        for (int l = j; l < kd; l++) x = fma(lin[l * ldl + j], zv[l], x);
        out_sel[j] = j < kd ? sup[j] : -1;
        out_coef[j] = j < kd ? x : 0.0;
      }
      if (lane == 0) {
        a.out_count[p] = kd;
        a.out_rnorm[p] = rnorm[q];
        a.out_scans[p] = scans[q];
        a.out_flag[p] = 0;
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- lock-step tensor-core scan
// Full-dictionary OMP for N <= 32, T <= 256 (the zero-tree step 1 shape):
// the CTA's 32 warps each own one signal and advance in lock-step, so one
// iteration's correlations of all 32 signals are the GEMM C = R (32 x 32) .
// D^T (32 x 256) on the tensor cores (mma.sync m16n8k8 TF32, 3xTF32 split:
// a_lo b_hi + a_hi b_lo + a_hi b_hi, ~fp32 accuracy) -- every dictionary
// fragment is read from shared memory once per CTA-iteration instead of once
// per signal.  Each warp then certifies its pick as the F32C scan does, with
// E = 2^-15 max|d| |r| (TF32 split residuals, fp32 accumulation in the MMA,
// fp32 rounding of r: all << 2^-16 relative of sum |r_i d_i| <= |r| |d|),
// re-scores the window in fp64 when it holds more than one candidate,
// recomputes the winner's correlation in fp64, and runs the same Cholesky
// append and residual update as resident_omp_kernel, with the fp64 atoms read
// from global memory (L1-resident).  Finished signals idle (zero rows) until
// the CTA's batch of 32 completes.
constexpr int MM_W = 32;
constexpr int MM_N = 32;
constexpr int MM_T = 256;
constexpr int MM_BS = MM_T + 8;  // B row stride (floats): conflict-free fragment loads
constexpr int MM_AS = MM_N + 4;  // A row stride
constexpr int MM_CS = MM_T + 4;  // C row stride

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// W signals (warps) per CTA: 32 (one CTA per SM) or 16 (two CTAs per SM, so
// one CTA's warps issue while the other's wait at the lock-step barrier)
template <typename YT, int W>
__global__ void __launch_bounds__(W * 32, 1024 / (W * 32))
    resident_mma_kernel(ResidentArgs a, const YT *__restrict__ ys) {
  constexpr int MT = W / 16;  // m-tiles of the scan GEMM
  constexpr int U = MM_T / 32;
  extern __shared__ __align__(16) double rs[];
  __shared__ double s_dmax;
  const int n = (int)a.n, T = (int)a.t, kw = (int)a.k_width;
  const int ldl = kw | 1;
  const int64_t P = a.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float *Bs = (float *)rs;               // MM_N x MM_BS: Bs[k][j] = d_j[k]
  float *Ahi = Bs + MM_N * MM_BS;        // W x MM_AS (tf32-rounded floats)
  float *Alo = Ahi + W * MM_AS;
  float *Cs = Alo + W * MM_AS;           // W x MM_CS
  double *nrm2 = (double *)(Cs + W * MM_CS);  // MM_T
  double *st = nrm2 + MM_T + warp * a.per_warp;
  double *r = st;
  double *lin = r + n;
  double *zv = lin + kw * ldl;
  double *wv = zv + kw;
  double *gv = wv + kw;
  int *sup = (int *)(gv + 2 * kw);
  int *soff = sup + kw;  // sup[l] * n: 32-bit row offsets of the support atoms
  const double *d64 = a.d64;
  const double *gram = a.gram;

  for (int e = threadIdx.x; e < MM_N * MM_T; e += blockDim.x) {
    const int k = e / MM_T, j = e % MM_T;
    Bs[k * MM_BS + j] = k < n && j < T ? (float)d64[(int64_t)j * n + k] : 0.0f;
  }
  for (int j = threadIdx.x; j < MM_T; j += blockDim.x) {
    double sq = 0.0;
    if (j < T)
      for (int i = 0; i < n; i++) sq = fma(d64[(int64_t)j * n + i], d64[(int64_t)j * n + i], sq);
    nrm2[j] = sq;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double mx = 0.0;
    for (int j = threadIdx.x; j < MM_T; j += 32) mx = fmax(mx, nrm2[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(CDB_FULL_MASK, mx, o));
    if (threadIdx.x == 0) s_dmax = sqrt(mx);
  }
  __syncthreads();
  const double e_rel = 0x1p-15 * 1.01 * s_dmax;  // |c~ - c| <= e_rel |r|

  for (int64_t p0 = (int64_t)blockIdx.x * W; p0 < P; p0 += (int64_t)gridDim.x * W) {
    const int64_t p = p0 + warp;
    const bool valid = p < P;
    const int kmax = valid ? (int)a.cands.budget(p, a.k_max, n) : 0;
    unsigned tk = 0u;
#pragma unroll
    for (int u = 0; u < U; u++)
      if (lane + 32 * u >= T) tk |= 1u << u;
    for (int i = lane; i < n; i += 32) r[i] = valid ? (double)ys[p * n + i] : 0.0;
    __syncwarp();
    const double ynorm = sqrt(dot4_quad(r, r, n, lane));  // reference order (_kernels.py:71)
    const double tol = valid ? a.eps[p] : 0.0;
    double rnorm = ynorm;
    int kdone = 0;
    int64_t scans = 0;
    bool delegate = false;
    bool live = valid && !(ynorm <= tol) && kmax > 0;
    for (int k = 0;; k++) {
      if (live && k >= kmax) live = false;
      // this signal's row of A (zeros once finished)
      for (int i = lane; i < MM_N; i += 32) {
        const float av = live && i < n ? (float)r[i] : 0.0f;
        const uint32_t hi = to_tf32(av);
        Ahi[warp * MM_AS + i] = __uint_as_float(hi);
        Alo[warp * MM_AS + i] = av - __uint_as_float(hi);  // unrounded (see blo)
      }
      if (!__syncthreads_or(live)) break;
      {  // ---- C = A B: warp w computes m-tile (w & 1), n-tiles 2 (w >> 1) + {0, 1}
        // (k-steps outer: each A fragment is loaded once for both n-tiles)
        const int mt = warp % MT, g = lane >> 2, tq = lane & 3;
        float dd[2][4] = {{0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}};
#pragma unroll
        for (int ks = 0; ks < MM_N / 8; ks++) {
          const int k0 = ks * 8;
          const float *ah = Ahi + (mt * 16 + g) * MM_AS + k0 + tq;
          const float *al = Alo + (mt * 16 + g) * MM_AS + k0 + tq;
          const uint32_t ahi[4] = {__float_as_uint(ah[0]), __float_as_uint(ah[8 * MM_AS]),
                                   __float_as_uint(ah[4]), __float_as_uint(ah[8 * MM_AS + 4])};
          const uint32_t alo[4] = {__float_as_uint(al[0]), __float_as_uint(al[8 * MM_AS]),
                                   __float_as_uint(al[4]), __float_as_uint(al[8 * MM_AS + 4])};
#pragma unroll
          for (int nn = 0; nn < 2; nn++) {
            const int nt = (warp / MT) * 2 + nn;
            const float b0 = Bs[(k0 + tq) * MM_BS + nt * 8 + g];
            const float b1 = Bs[(k0 + tq + 4) * MM_BS + nt * 8 + g];
            const uint32_t bhi[2] = {to_tf32(b0), to_tf32(b1)};
            // the low part enters the MMA unrounded: the tensor core drops its
            // low 13 mantissa bits, <= 2^-21 |b|, far inside E (2^-15)
            const uint32_t blo[2] = {__float_as_uint(b0 - __uint_as_float(bhi[0])),
                                     __float_as_uint(b1 - __uint_as_float(bhi[1]))};
            mma_tf32(dd[nn], alo, bhi);
            mma_tf32(dd[nn], ahi, blo);
            mma_tf32(dd[nn], ahi, bhi);
          }
        }
#pragma unroll
        for (int nn = 0; nn < 2; nn++) {
          const int nt = (warp / MT) * 2 + nn;
          float *c0 = Cs + (mt * 16 + g) * MM_CS + nt * 8 + 2 * tq;
          *(float2 *)c0 = make_float2(dd[nn][0], dd[nn][1]);
          *(float2 *)(c0 + 8 * MM_CS) = make_float2(dd[nn][2], dd[nn][3]);
        }
      }
      __syncthreads();
      if (!live) continue;
      scans += T - k;
      float acc[U];
#pragma unroll
      for (int u = 0; u < U; u++) acc[u] = Cs[warp * MM_CS + lane + 32 * u];
      // ---- certified selection: max |c| over available atoms, ties -> lowest index
      // (in fp32 on the fp32 correlations: the max of non-negative floats is a
      // REDUX on their bits; the window threshold is rounded down, so the
      // window can only grow -- a larger window is re-scored exactly)
      float bestf = -1.0f;
      unsigned bj = 0xffffffffu;
#pragma unroll
      for (int u = 0; u < U; u++) {
        const float v = fabsf(acc[u]);
        if (!((tk >> u) & 1u) && v > bestf) {
          bestf = v;
          bj = lane + 32 * u;
        }
      }
      const unsigned key = bestf >= 0.0f ? __float_as_uint(bestf) : 0u;
      const unsigned mkey = __reduce_max_sync(CDB_FULL_MASK, key);
      double m = (double)__uint_as_float(mkey);
      const float thr = __double2float_rd(m - 2.0 * e_rel * rnorm);
      unsigned cand = bestf >= 0.0f && key == mkey ? bj : 0xffffffffu;
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < U; u++)
        if (!((tk >> u) & 1u) && fabsf(acc[u]) >= thr) cnt++;
      cnt = (int)__reduce_add_sync(CDB_FULL_MASK, (unsigned)cnt);
      if (cnt == 0) {  // nothing available (_kernels.py:104)
        live = false;
        continue;
      }
      if (cnt > 1) {  // re-score the window exactly in fp64 (lane per candidate)
        double best = -1.0;
        bj = 0xffffffffu;
#pragma unroll
        for (int u = 0; u < U; u++) {
          if (!((tk >> u) & 1u) && fabsf(acc[u]) >= thr) {
            const int jj = lane + 32 * u;
            const double *dj = d64 + (int64_t)jj * n;
            double c = 0.0;
            for (int i = 0; i < n; i++) c = fma(__ldg(dj + i), r[i], c);
            if (fabs(c) > best) {
              best = fabs(c);
              bj = jj;
            }
          }
        }
        m = best;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(CDB_FULL_MASK, m, o));
        cand = best == m ? bj : 0xffffffffu;
      }
      const int bestj = (int)__reduce_min_sync(CDB_FULL_MASK, cand);
      const int ub = bestj >> 5, owner = bestj & 31;
      const int nid = bestj;
      double cbest;
      {  // the winner's exact correlation (z_k = c / d); orthogonal break on it
        double c = 0.0;
        const double *drow = d64 + (uint32_t)(nid * n);  // T * n < 2^31 here (T <= 256)
        for (int i = lane; i < n; i += 32) c = fma(__ldg(drow + i), r[i], c);
        cbest = warp_sum(c);
      }
      if (!(fabs(cbest) > 0.0)) {  // _kernels.py:104
        live = false;
        continue;
      }
      if (lane == owner) tk |= 1u << ub;
      // ---- Cholesky append through the Gram row (as resident_omp_kernel)
      const double *grow = gram + (uint32_t)(nid * T);  // T <= 256: 32-bit offsets
      for (int l = lane; l < k; l += 32) gv[l] = __ldg(grow + sup[l]);
      if (lane == 0) {
        sup[k] = nid;
        soff[k] = nid * n;
      }
      __syncwarp();
      // w = L^{-1} g and the new L^{-1} row: two lanes per row, each summing
      // half of it (halves the warp's trip count of the triangular loops)
      for (int l0 = 0; l0 < k; l0 += 16) {
        const int l = l0 + (lane >> 1), h = lane & 1;
        double accw = 0.0;
        if (l < k) {
          const int mid = (l + 1) >> 1;
          const int i1 = h ? l + 1 : mid;
          for (int i = h ? mid : 0; i < i1; i++) accw = fma(lin[l * ldl + i], gv[i], accw);
        }
        accw += __shfl_xor_sync(CDB_FULL_MASK, accw, 1);
        if (l < k && h == 0) wv[l] = accw;
      }
      __syncwarp();
      double ww = 0.0;
      for (int l = lane; l < k; l += 32) ww = fma(wv[l], wv[l], ww);
      ww = warp_sum(ww);
      const double gnn = nrm2[nid];
      const double d2 = gnn - ww;
      if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {
        delegate = true;
        live = false;
        continue;
      }
      const double inv_d = rsqrt(d2);
      const double zk = cbest * inv_d;
      for (int i0 = 0; i0 <= k; i0 += 16) {
        const int i = i0 + (lane >> 1), h = lane & 1;
        double accl = 0.0;
        if (i < k) {
          const int mid = (i + k) >> 1;
          const int l1 = h ? k : mid;
          for (int l = h ? mid : i; l < l1; l++) accl = fma(wv[l], lin[l * ldl + i], accl);
        }
        accl += __shfl_xor_sync(CDB_FULL_MASK, accl, 1);
        if (i <= k && h == 0) lin[k * ldl + i] = i == k ? inv_d : -accl * inv_d;
      }
      if (lane == 0) zv[k] = zk;
      __syncwarp();
      kdone = k + 1;
      // ---- residual r -= z_k q_k,  q_k = sum_l L^{-1}[k][l] d_{s_l}; stop test
      const double *lk = lin + k * ldl;
      double rr = 0.0;
      for (int i = lane; i < n; i += 32) {
        double qv = 0.0;
        const double *dbase = d64 + i;  // + soff[l]: one address add per term
#pragma unroll 4
        for (int l = 0; l <= k; l++) qv = fma(lk[l], __ldg(dbase + soff[l]), qv);
        const double rv = fma(-zk, qv, r[i]);
        r[i] = rv;
        rr = fma(rv, rv, rr);
      }
      rnorm = sqrt(warp_sum(rr));
      __syncwarp();
      if (rnorm <= tol) live = false;
    }
    // ---- outputs: x = L^{-T} z (pick order)
    if (valid) {
      if (delegate) {
        if (lane == 0) a.status[p] |= ST_DELEGATE;
      } else {
        int64_t *out_sel = a.out_sel + p * kw;
        double *out_coef = a.out_coef + p * kw;
        for (int j = lane; j < kw; j += 32) {
          double x = 0.0;
          for (int l = j; l < kdone; l++) x = fma(lin[l * ldl + j], zv[l], x);
          out_sel[j] = j < kdone ? sup[j] : -1;
          out_coef[j] = j < kdone ? x : 0.0;
        }
        if (lane == 0) {
          a.out_count[p] = kdone;
          a.out_rnorm[p] = rnorm;
          a.out_scans[p] = scans;
          a.out_flag[p] = 0;
        }
      }
    }
    __syncwarp();
  }
}

template <int U>
// signals per warp: 1 with 32 warps/SM measured best for cfg 1 step 1
// (2.67 ms; 24 warps 2.76; R = 2 x 16 warps 2.83; R = 4 x 12 warps 3.43): the
// least-squares tail is latency-bound, so independent warps beat the
// shared-memory reuse of several signals per warp
constexpr int res_r() { return U > 0 ? 1 : 1; }
constexpr int res_max_warps(int r) { return r >= 4 ? 12 : (r == 1 ? 32 : RES_WARPS); }

template <typename YT, int U>
cudaError_t launch_u(const ResidentArgs &args, const YT *ys, int64_t base, int smem_optin,
                     int num_sms, cudaStream_t stream) {
  constexpr int R = res_r<U>();
  ResidentArgs a = args;
  const int max_w = res_max_warps(R);
  auto warps_for = [&](int64_t b) {
    int w = (int)((smem_optin - b) / (8 * a.per_warp * R));
    return w > max_w ? max_w : w;
  };
  // fp32 certified scan when the extra fp32 atom copy still leaves as many
  // warps as the fp64 scan (or a full CTA)
  const int64_t base32 = base + 16 + 4 * ((a.n + 1) & ~1LL) * 32 * U;
  const int w64 = warps_for(base), w32 = warps_for(base32);
  const bool f32c = U >= 4 && a.cands.mode == 0 && !getenv("CDB_RESIDENT_FP64") && w32 >= 8 &&
                    (w32 >= w64 || w32 >= max_w);
  const int warps = f32c ? w32 : w64;
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem = (size_t)((f32c ? base32 : base) + 8 * a.per_warp * R * warps);
  int64_t grid = (a.p + warps * R - 1) / (warps * R);
  if (grid > num_sms) grid = num_sms;
  void (*kern)(ResidentArgs, const YT *);
  if (a.cands.mode == 0)
    kern = f32c ? resident_omp_kernel<YT, U, true, R, (U >= 4)>
                : resident_omp_kernel<YT, U, true, R, false>;
  else
    kern = resident_omp_kernel<YT, U, false, R, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(int)grid, warps * 32, smem, stream>>>(a, ys);
  return cudaGetLastError();
}

template <typename YT>
cudaError_t launch_t(const ResidentArgs &a, const YT *ys, int u, int64_t base, int smem_optin,
                     int num_sms, cudaStream_t stream) {
  switch (u) {
    case 1: return launch_u<YT, 1>(a, ys, base, smem_optin, num_sms, stream);
    case 2: return launch_u<YT, 2>(a, ys, base, smem_optin, num_sms, stream);
    case 4: return launch_u<YT, 4>(a, ys, base, smem_optin, num_sms, stream);
    case 8: return launch_u<YT, 8>(a, ys, base, smem_optin, num_sms, stream);
    case 16: return launch_u<YT, 16>(a, ys, base, smem_optin, num_sms, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int64_t resident_warp_doubles(int64_t n, int64_t kw, int64_t max_cands) {
  (void)max_cands;
  // ..., fp32 residual pairs at an even offset; even total keeps 16-B alignment
  return ((n + kw * (kw | 1) + 5 * kw + 2) & ~1LL) + ((n + 1) & ~1LL);
}

// Row stride of the transposed dictionary: at least one zero column and the
// 32*U columns the lane-strided correlation loop reads, rounded to 1 mod 16
// doubles so a warp walking one column (lane = row) hits distinct banks.
static int64_t resident_tpad(int64_t t, int64_t max_cands) {
  int64_t u = 1;
  while (32 * u < max_cands) u *= 2;
  int64_t tp = t + 1 > 32 * u ? t + 1 : 32 * u;
  return (tp + 14) / 16 * 16 + 1;
}

bool resident_fits(int64_t n, int64_t t, int64_t kw, int64_t max_cands, int smem_optin) {
  if (max_cands > 512) return false;
  const int64_t tp = resident_tpad(t, max_cands);
  const int64_t base = 8 * (n * tp + tp);
  const int64_t per = 8 * resident_warp_doubles(n, kw, max_cands) * 4;
  return base + 4 * per <= smem_optin && base <= 144 * 1024;
}

cudaError_t launch_resident(const ResidentArgs &args, const void *ys, bool ys_f32, int smem_optin,
                            int num_sms, cudaStream_t stream) {
  ProfScope _ps(args.tag ? args.tag : "resident_omp", stream);
  if (args.p <= 0) return cudaSuccess;
  ResidentArgs a = args;
  a.per_warp = resident_warp_doubles(a.n, a.k_width, a.max_cands);
  a.t_pad = resident_tpad(a.t, a.max_cands);
  if (a.cands.mode == 0 && a.t_pad < 32 * ((a.max_cands + 31) / 32)) return cudaErrorInvalidValue;
  if (a.cands.mode == 0 && a.n <= MM_N && a.t <= MM_T && a.gram && !getenv("CDB_RESIDENT_NO_MMA")) {
    static const int w_env = [] {
      const char *v = getenv("CDB_MM_W");  // cfg 1 step 1: W = 16 2.23 ms, W = 32 2.29 ms
      return v ? atoi(v) : 16;
    }();
    auto smem_for = [&](int w) {
      return sizeof(float) * (MM_N * MM_BS + 2 * w * MM_AS + w * MM_CS) +
             sizeof(double) * (MM_T + w * a.per_warp);
    };
    // W = 16 only while two CTAs fit one SM
    const int W = w_env == 16 && 2 * (int64_t)smem_for(16) + 2048 <= smem_optin ? 16 : 32;
    const size_t smem = smem_for(W);
    if ((int64_t)smem <= smem_optin) {
      int64_t grid = (a.p + W - 1) / W;
      const int64_t cap = (int64_t)num_sms * (32 / W);
      if (grid > cap) grid = cap;
      const void *kern = W == 16 ? (ys_f32 ? (const void *)resident_mma_kernel<float, 16>
                                           : (const void *)resident_mma_kernel<double, 16>)
                                 : (ys_f32 ? (const void *)resident_mma_kernel<float, 32>
                                           : (const void *)resident_mma_kernel<double, 32>);
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      note_launch();
      if (W == 16) {
        if (ys_f32)
          resident_mma_kernel<float, 16><<<(int)grid, 512, smem, stream>>>(a, (const float *)ys);
        else
          resident_mma_kernel<double, 16><<<(int)grid, 512, smem, stream>>>(a, (const double *)ys);
      } else {
        if (ys_f32)
          resident_mma_kernel<float, 32><<<(int)grid, 1024, smem, stream>>>(a, (const float *)ys);
        else
          resident_mma_kernel<double, 32><<<(int)grid, 1024, smem, stream>>>(a, (const double *)ys);
      }
      return cudaGetLastError();
    }
  }
  const int64_t base = 8 * (a.n * a.t_pad + a.t_pad);
  int u = 1;
  while (32 * u < a.max_cands) u *= 2;
  note_launch();
  if (ys_f32) return launch_t<float>(a, (const float *)ys, u, base, smem_optin, num_sms, stream);
  return launch_t<double>(a, (const double *)ys, u, base, smem_optin, num_sms, stream);
}

}  // namespace cdb
