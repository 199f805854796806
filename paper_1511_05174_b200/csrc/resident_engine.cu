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

// FULL: candidate jl of lane l is atom l + 32u (mode 0) -> compile-time
// shared-memory offsets in the correlation loop.
template <typename YT, int U, bool FULL>
__global__ void __launch_bounds__(1024, 1)
    resident_omp_kernel(ResidentArgs a, const YT *__restrict__ ys) {
  extern __shared__ __align__(16) double rs[];
  const int n = (int)a.n, T = (int)a.t, kw = (int)a.k_width, Tp = (int)a.t_pad;
  const int64_t P = a.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double *Dt = rs;                 // n x Tp  (columns T..Tp-1 are zero)
  double *nrm2 = Dt + n * Tp;      // Tp  (|d_j|^2)
  double *wbase = nrm2 + Tp;
  const int per_warp = (int)a.per_warp;
  double *y = wbase + warp * per_warp;
  double *r = y + n;
  double *lin = r + n;             // kw x kw
  double *zv = lin + kw * kw;
  double *wv = zv + kw;
  double *xv = wv + kw;
  double *gv = xv + kw;
  int *sup = (int *)(gv + kw);     // kw ints (kw doubles reserved)
  uint32_t *taken = (uint32_t *)(gv + 2 * kw);

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
  for (int64_t p = (int64_t)blockIdx.x * nwarps + warp; p < P; p += (int64_t)gridDim.x * nwarps) {
    const int S = (int)cs.count(p);
    const int k_max = (int)cs.budget(p, a.k_max, n);
    int cid[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int jl = lane + 32 * u;
      cid[u] = FULL ? jl : (jl < S ? (int)cs.id(p, jl) : Tp - 1);  // zero column pads
    }
    for (int i = lane; i < n; i += 32) {
      const double v = (double)ys[p * n + i];
      y[i] = v;
      r[i] = v;
    }
    for (int w = lane; w < (S + 31) / 32; w += 32) taken[w] = 0u;
    __syncwarp();
    const double ynorm = sqrt(dot4_quad(y, y, n, lane));  // reference order (_kernels.py:71)
    const double tol = eps[p];
    int kdone = 0;
    int64_t scans = 0;
    double rnorm = ynorm;
    bool delegate = false;
    if (!(ynorm <= tol)) {
      for (int k = 0; k < k_max; k++) {
        scans += S - k;
        // ---- correlations of this lane's candidates with r (fp64)
        double acc[U];
#pragma unroll
        for (int u = 0; u < U; u++) acc[u] = 0.0;
        const double *col = FULL ? Dt + lane : Dt;
#pragma unroll 4
        for (int i = 0; i < n; i++) {
          const double ri = r[i];
          const double *row = col + i * Tp;
#pragma unroll
          for (int u = 0; u < U; u++) acc[u] = fma(FULL ? row[32 * u] : row[cid[u]], ri, acc[u]);
        }
        double best = -1.0, cbest = 0.0;
        int bestj = -1;
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int jl = lane + 32 * u;
          if (jl < S && !((taken[jl >> 5] >> (jl & 31)) & 1u)) {
            const double v = fabs(acc[u]);
            if (v > best) {
              best = v;
              bestj = jl;
              cbest = acc[u];
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
        if (bestj < 0 || best <= 0.0) break;  // _kernels.py:104
        const int nid = FULL ? bestj : (int)cs.id(p, bestj);
        if (lane == 0) {
          taken[bestj >> 5] |= 1u << (bestj & 31);
          sup[k] = nid;
        }
        __syncwarp();
        // ---- Cholesky append: g_l = <d_{s_l}, d_new> from the resident atoms
        if (lane < k) {
          double g = 0.0;
          const int sl = sup[lane];
          for (int i = 0; i < n; i++) g = fma(Dt[i * Tp + sl], Dt[i * Tp + nid], g);
          gv[lane] = g;
        }
        for (int l = lane + 32; l < k; l += 32) {
          double g = 0.0;
          const int sl = sup[l];
          for (int i = 0; i < n; i++) g = fma(Dt[i * Tp + sl], Dt[i * Tp + nid], g);
          gv[l] = g;
        }
        __syncwarp();
        for (int l = lane; l < k; l += 32) {
          double accw = 0.0;
          for (int i = 0; i <= l; i++) accw = fma(lin[l * kw + i], gv[i], accw);
          wv[l] = accw;
        }
        __syncwarp();
        double ww = 0.0;
        for (int l = lane; l < k; l += 32) ww = fma(wv[l], wv[l], ww);
        ww = warp_sum(ww);
        const double gnn = nrm2[nid];
        const double d2 = gnn - ww;
        if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {
          delegate = true;
          break;
        }
        const double inv_d = 1.0 / sqrt(d2);
        const double zk = cbest * inv_d;  // q_k^T y = q_k^T r = <d_new, r> / d
        for (int i = lane; i <= k; i += 32) {
          double v;
          if (i == k) {
            v = inv_d;
          } else {
            double accl = 0.0;
            for (int l = i; l < k; l++) accl = fma(wv[l], lin[l * kw + i], accl);
            v = -accl * inv_d;
          }
          lin[k * kw + i] = v;
        }
        if (lane == 0) zv[k] = zk;
        __syncwarp();
        kdone = k + 1;
        for (int i = lane; i < kdone; i += 32) {
          double accx = 0.0;
          for (int l = i; l < kdone; l++) accx = fma(lin[l * kw + i], zv[l], accx);
          xv[i] = accx;
        }
        __syncwarp();
        // ---- residual r = y - D_S x (fp64) and its norm; stop test
        double rr = 0.0;
        for (int i = lane; i < n; i += 32) {
          double ri = y[i];
          const double *row = Dt + i * Tp;
          for (int l = 0; l < kdone; l++) ri = fma(-xv[l], row[sup[l]], ri);
          r[i] = ri;
          rr = fma(ri, ri, rr);
        }
        rnorm = sqrt(warp_sum(rr));
        __syncwarp();
        if (rnorm <= tol) break;
      }
    }
    if (delegate) {
      if (lane == 0) a.status[p] |= ST_DELEGATE;
      __syncwarp();
      continue;
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
    __syncwarp();
  }
}

template <typename YT, int U>
cudaError_t launch_u(const ResidentArgs &a, const YT *ys, int threads, size_t smem,
                     int grid, cudaStream_t stream) {
  auto kern = a.cands.mode == 0 ? resident_omp_kernel<YT, U, true>
                                : resident_omp_kernel<YT, U, false>;
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
  return 2 * n + kw * kw + 6 * kw + ((max_cands + 63) / 64) + 2;
}

static int64_t resident_tpad(int64_t t, int64_t max_cands) {
  int64_t u = 1;
  while (32 * u < max_cands) u *= 2;
  int64_t tp = (t + 1 + 31) / 32 * 32;  // at least one zero column
  return tp;
}

bool resident_fits(int64_t n, int64_t t, int64_t kw, int64_t max_cands, int smem_optin) {
  if (max_cands > 512) return false;
  const int64_t tp = resident_tpad(t, max_cands);
  const int64_t base = 8 * (n * tp + tp);
  const int64_t per = 8 * resident_warp_doubles(n, kw, max_cands);
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
  int warps = (int)((smem_optin - base) / (8 * a.per_warp));
  if (warps > 32) warps = 32;
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(base + 8 * a.per_warp * warps);
  int u = 1;
  while (32 * u < a.max_cands) u *= 2;
  int64_t grid = (a.p + warps - 1) / warps;
  if (grid > num_sms) grid = num_sms;
  note_launch();
  if (ys_f32) return launch_t<float>(a, (const float *)ys, u, warps * 32, smem, (int)grid, stream);
  return launch_t<double>(a, (const double *)ys, u, warps * 32, smem, (int)grid, stream);
}

}  // namespace cdb
