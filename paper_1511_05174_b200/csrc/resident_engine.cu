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
#include "candidates.cuh"
#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

constexpr int RES_R = 2;        // signals per warp
constexpr int RES_WARPS = 16;   // warps per CTA (512 threads)

// FULL: candidate jl of lane l is atom l + 32u (mode 0) -> compile-time
// shared-memory offsets in the correlation loop.  R signals per warp share
// every dictionary element loaded from shared memory (R FMAs per LDS).
template <typename YT, int U, bool FULL, int R>
__global__ void __launch_bounds__(512, 1)
    resident_omp_kernel(ResidentArgs a, const YT *__restrict__ ys) {
  extern __shared__ __align__(16) double rs[];
  const int n = (int)a.n, T = (int)a.t, kw = (int)a.k_width, Tp = (int)a.t_pad;
  const int ldl = kw | 1;  // odd L^{-1} row stride: column walks hit distinct banks
  const int64_t P = a.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double *Dt = rs;                 // n x Tp  (columns T..Tp-1 are zero)
  double *nrm2 = Dt + n * Tp;      // Tp  (|d_j|^2)
  double *wbase = nrm2 + Tp;
  const int per_sig = (int)a.per_warp;  // doubles of state per signal

  for (int e = threadIdx.x; e < n * Tp; e += blockDim.x) {
    const int i = e / Tp, j = e % Tp;
    Dt[e] = j < T ? a.d64[(int64_t)j * n + i] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < Tp; j += blockDim.x) {
    double sq = 0.0;
    for (int i = 0; i < n; i++) sq = fma(Dt[i * Tp + j], Dt[i * Tp + j], sq);
    nrm2[j] = sq;
  }
  __syncthreads();

  const Cands cs = a.cands;
  const double *eps = a.eps;
  const double *gram = a.gram;
  double *sbase = wbase + warp * R * per_sig;
  for (int64_t p0 = ((int64_t)blockIdx.x * nwarps + warp) * R; p0 < P;
       p0 += (int64_t)gridDim.x * nwarps * R) {
    // ---- per-signal setup
    int S[R], kmax[R], kdone[R];
    int64_t scans[R];
    double tol[R], rnorm[R];
    bool live[R], delegate[R];
    int cid[R][U];
#pragma unroll
    for (int q = 0; q < R; q++) {
      const int64_t p = p0 + q;
      double *y = sbase + q * per_sig;
      double *r = y + n;
      uint32_t *taken = (uint32_t *)(r + n + kw * ldl + 5 * kw);
      const bool valid = p < P;
      S[q] = valid ? (int)cs.count(p) : 0;
      kmax[q] = valid ? (int)cs.budget(p, a.k_max, n) : 0;
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int jl = lane + 32 * u;
        cid[q][u] = FULL ? jl : (jl < S[q] ? (int)cs.id(p, jl) : Tp - 1);
      }
      for (int i = lane; i < n; i += 32) {
        const double v = valid ? (double)ys[p * n + i] : 0.0;
        y[i] = v;
        r[i] = v;
      }
      for (int w = lane; w < (S[q] + 31) / 32; w += 32) taken[w] = 0u;
      __syncwarp();
      const double ynorm = sqrt(dot4_quad(y, y, n, lane));  // reference order (_kernels.py:71)
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
#pragma unroll
      for (int q = 0; q < R; q++)
#pragma unroll
        for (int u = 0; u < U; u++) acc[q][u] = 0.0;
      const double *col = FULL ? Dt + lane : Dt;
#pragma unroll 2
      for (int i = 0; i < n; i++) {
        double ri[R];
#pragma unroll
        for (int q = 0; q < R; q++) ri[q] = sbase[q * per_sig + n + i];
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
#pragma unroll
      for (int q = 0; q < R; q++) {
        if (!live[q]) continue;
        const int64_t p = p0 + q;
        double *y = sbase + q * per_sig;
        double *r = y + n;
        double *lin = r + n;
        double *zv = lin + kw * ldl;
        double *wv = zv + kw;
        double *xv = wv + kw;
        double *gv = xv + kw;
        int *sup = (int *)(gv + kw);
        uint32_t *taken = (uint32_t *)(gv + 2 * kw);
        scans[q] += S[q] - k;
        double best = -1.0, cbest = 0.0;
        int bestj = -1;
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int jl = lane + 32 * u;
          if (jl < S[q] && !((taken[jl >> 5] >> (jl & 31)) & 1u)) {
            const double v = fabs(acc[q][u]);
            if (v > best) {
              best = v;
              bestj = jl;
              cbest = acc[q][u];
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(CDB_FULL_MASK, best, o);
          const int oj = __shfl_xor_sync(CDB_FULL_MASK, bestj, o);
          const double oc = __shfl_xor_sync(CDB_FULL_MASK, cbest, o);
          if (oj >= 0 && (bestj < 0 || ov > best || (ov == best && oj < bestj))) {
            best = ov;
            bestj = oj;
            cbest = oc;
          }
        }
        if (bestj < 0 || best <= 0.0) {  // _kernels.py:104
          live[q] = false;
          continue;
        }
        const int nid = FULL ? bestj : (int)cs.id(p, bestj);
        if (lane == 0) {
          taken[bestj >> 5] |= 1u << (bestj & 31);
          sup[k] = nid;
        }
        __syncwarp();
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
        __syncwarp();
        for (int l = lane; l < k; l += 32) {
          double accw = 0.0;
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
        const double inv_d = 1.0 / sqrt(d2);
        const double zk = cbest * inv_d;  // q_k^T y = q_k^T r = <d_new, r> / d
        for (int i = lane; i <= k; i += 32) {
          double v;
          if (i == k) {
            v = inv_d;
          } else {
            double accl = 0.0;
            for (int l = i; l < k; l++) accl = fma(wv[l], lin[l * ldl + i], accl);
            v = -accl * inv_d;
          }
          lin[k * ldl + i] = v;
        }
        if (lane == 0) zv[k] = zk;
        __syncwarp();
        kdone[q] = k + 1;
        for (int i = lane; i <= k; i += 32) {
          double accx = 0.0;
#pragma unroll 4
          for (int l = i; l <= k; l++) accx = fma(lin[l * ldl + i], zv[l], accx);
          xv[i] = accx;
        }
        __syncwarp();
        // ---- residual r = y - D_S x (fp64) and its norm; stop test
        double rr = 0.0;
        for (int i = lane; i < n; i += 32) {
          double rv = y[i];
          const double *row = Dt + i * Tp;
#pragma unroll 4
          for (int l = 0; l <= k; l++) rv = fma(-xv[l], row[sup[l]], rv);
          r[i] = rv;
          rr = fma(rv, rv, rr);
        }
        rnorm[q] = sqrt(warp_sum(rr));
        __syncwarp();
        if (rnorm[q] <= tol[q]) live[q] = false;
      }
    }
    // ---- outputs
#pragma unroll
    for (int q = 0; q < R; q++) {
      const int64_t p = p0 + q;
      if (p >= P) continue;
      if (delegate[q]) {
        if (lane == 0) a.status[p] |= ST_DELEGATE;
        continue;
      }
      double *y = sbase + q * per_sig;
      double *xv = y + 2 * n + kw * ldl + 2 * kw;
      int *sup = (int *)(xv + 2 * kw);
      int64_t *out_sel = a.out_sel + p * kw;
      double *out_coef = a.out_coef + p * kw;
      for (int j = lane; j < kw; j += 32) {
        out_sel[j] = j < kdone[q] ? sup[j] : -1;
        out_coef[j] = j < kdone[q] ? xv[j] : 0.0;
      }
      if (lane == 0) {
        a.out_count[p] = kdone[q];
        a.out_rnorm[p] = rnorm[q];
        a.out_scans[p] = scans[q];
        a.out_flag[p] = 0;
      }
    }
    __syncwarp();
  }
}

template <typename YT, int U>
cudaError_t launch_u(const ResidentArgs &a, const YT *ys, int threads, size_t smem,
                     int grid, cudaStream_t stream) {
  auto kern = a.cands.mode == 0 ? resident_omp_kernel<YT, U, true, RES_R>
                                : resident_omp_kernel<YT, U, false, RES_R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, threads, smem, stream>>>(a, ys);
  return cudaGetLastError();
}

template <typename YT>
cudaError_t launch_t(const ResidentArgs &a, const YT *ys, int u, int threads, size_t smem,
                     int grid, cudaStream_t stream) {
  switch (u) {
    case 1: return launch_u<YT, 1>(a, ys, threads, smem, grid, stream);
    case 2: return launch_u<YT, 2>(a, ys, threads, smem, grid, stream);
    case 4: return launch_u<YT, 4>(a, ys, threads, smem, grid, stream);
    case 8: return launch_u<YT, 8>(a, ys, threads, smem, grid, stream);
    case 16: return launch_u<YT, 16>(a, ys, threads, smem, grid, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int64_t resident_warp_doubles(int64_t n, int64_t kw, int64_t max_cands) {
  return 2 * n + kw * (kw | 1) + 6 * kw + ((max_cands + 63) / 64) + 2;
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
  const int64_t per = 8 * resident_warp_doubles(n, kw, max_cands) * RES_R;
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
  const int64_t base = 8 * (a.n * a.t_pad + a.t_pad);
  int warps = (int)((smem_optin - base) / (8 * a.per_warp * RES_R));
  if (warps > RES_WARPS) warps = RES_WARPS;
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(base + 8 * a.per_warp * RES_R * warps);
  int u = 1;
  while (32 * u < a.max_cands) u *= 2;
  int64_t grid = (a.p + warps * RES_R - 1) / (warps * RES_R);
  if (grid > num_sms) grid = num_sms;
  note_launch();
  if (ys_f32) return launch_t<float>(a, (const float *)ys, u, warps * 32, smem, (int)grid, stream);
  return launch_t<double>(a, (const double *)ys, u, warps * 32, smem, (int)grid, stream);
}

}  // namespace cdb
