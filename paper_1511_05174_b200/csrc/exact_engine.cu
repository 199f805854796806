// Exact engine: a warp-per-signal fp64 restatement of the reference kernel
// omp_batch_kernel (crossdict/_kernels.py:50-168).
//
// Every floating-point operation of the reference is reproduced in the same
// order: _dot4's four fixed accumulators (_kernels.py:27-42) are computed by
// four lanes each (lane m owns the i = m mod 4 chain), combined as
// ((s0+s1)+s2)+s3 and the tail added last; the file is compiled with
// -fmad=false so no multiply-add is contracted (numba runs with
// fastmath=False).  Selections, coefficients, residual norms, scan counts
// and flags are therefore bit-identical to the reference on the same fp64
// inputs, except coefficients in the rank-deficient dense mode, where the
// reference calls LAPACK (np.linalg.lstsq, _kernels.py:145) and this engine
// runs a one-sided Jacobi SVD minimum-norm solve (the same restatement as
// oracle/omp_oracle.c, coefficients "parity unpinned").
//
// Coded mode (rows != NULL): signal p is measured through its
// own patch operator with m_p outputs (pipelines.py:256-322, sensing.
// patch_problem): every atom access reads the effective element eff_at(atom,
// rows_p, fan, i) for i < m_p -- atom[rows[i]] for a mask / mosaic / angular
// gather, the ordered sum of the coded frames for a temporal code -- i.e. the
// reference's effective dictionary E_p = phi_p.apply_matrix(D) in its own
// arithmetic, and the signal row holds the m_p measurements.
//
// Role in the product: the engine of record for small problems and the
// fallback for signals the fast engines delegate (rank trouble or an
// uncertifiable selection).  Throughput is not its purpose.
#include "candidates.cuh"
#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

// One-sided Jacobi minimum-norm least squares, run by a single lane
// (identical to oracle/omp_oracle.c lstsq_min_norm).
__device__ void lstsq_min_norm(double *a, int64_t n, int64_t m, const double *y, double *x,
                               double *v) {
  for (int64_t i = 0; i < m * m; i++) v[i] = 0.0;
  for (int64_t i = 0; i < m; i++) v[i * m + i] = 1.0;
  const double eps = 1.1102230246251565e-16;
  for (int sweep = 0; sweep < 80; sweep++) {
    int rotated = 0;
    for (int64_t p = 0; p < m - 1; p++) {
      for (int64_t q = p + 1; q < m; q++) {
        double *ap = a + p * n, *aq = a + q * n;
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int64_t i = 0; i < n; i++) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || fabs(gamma) <= eps * sqrt(alpha * beta)) continue;
        rotated = 1;
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = c * t;
        for (int64_t i = 0; i < n; i++) {
          double xp = ap[i], xq = aq[i];
          ap[i] = c * xp - s * xq;
          aq[i] = s * xp + c * xq;
        }
        double *vp = v + p * m, *vq = v + q * m;
        for (int64_t i = 0; i < m; i++) {
          double xp = vp[i], xq = vq[i];
          vp[i] = c * xp - s * xq;
          vq[i] = s * xp + c * xq;
        }
      }
    }
    if (!rotated) break;
  }
  double smax = 0.0;
  for (int64_t j = 0; j < m; j++) {
    double s2 = 0.0;
    for (int64_t i = 0; i < n; i++) s2 += a[j * n + i] * a[j * n + i];
    double s = sqrt(s2);
    if (s > smax) smax = s;
  }
  for (int64_t i = 0; i < m; i++) x[i] = 0.0;
  for (int64_t j = 0; j < m; j++) {
    double s2 = 0.0, uy = 0.0;
    for (int64_t i = 0; i < n; i++) {
      s2 += a[j * n + i] * a[j * n + i];
      uy += a[j * n + i] * y[i];
    }
    double s = sqrt(s2);
    if (!(s > eps * smax) || s == 0.0) continue;
    double f = uy / s2;
    for (int64_t i = 0; i < m; i++) x[i] += v[j * m + i] * f;
  }
}

template <typename YT>
__global__ void __launch_bounds__(256) exact_omp_kernel(ExactArgs a, const YT *__restrict__ ys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n = a.n, kw = a.k_width;
  const Cands &cs = a.cands;

  double *work = a.work + warp_global * a.work_stride;
  double *y = work;                   // n (fp64 copy of the signal)
  double *r = y + n;                  // n
  double *u = r + n;                  // n
  double *qmat = u + n;               // kw * n
  double *rmat = qmat + kw * n;       // kw * kw
  double *qty = rmat + kw * kw;       // kw
  double *amat = qty + kw;            // n * kw
  double *coefs = amat + n * kw;      // kw
  double *vwork = coefs + kw;         // kw * kw
  uint32_t *taken = (uint32_t *)(vwork + kw * kw);  // bit mask over candidates

  const int64_t count = a.p_count_dev ? (int64_t)*a.p_count_dev : a.p_count;
  for (int64_t idx = warp_global; idx < count; idx += n_warps) {
    const int64_t p = a.sig_ids ? a.sig_ids[idx] : idx;
    const int64_t c = cs.count(p);
    const int32_t *rw = a.rows ? a.rows + p * a.rows_stride : nullptr;
    const int fan = a.fan, ord = a.sum_order;
    const int64_t ne = rw ? a.m_sig[p] : n;  // coordinates this signal is measured on
    const int64_t k_max = cs.budget(p, a.k_max, ne);
    int64_t *sel = a.out_sel + p * kw;
    double *coef = a.out_coef + p * kw;
    for (int64_t j = lane; j < kw; j += 32) {
      sel[j] = -1;
      coef[j] = 0.0;
    }
    for (int64_t i = lane; i < ne; i += 32) {
      double v = (double)ys[p * a.ys_stride + i];
      y[i] = v;
      r[i] = v;
    }
    for (int64_t w = lane; w < (c + 31) / 32; w += 32) taken[w] = 0u;
    for (int64_t i = lane; i < kw * kw; i += 32) rmat[i] = 0.0;
    __syncwarp();

    const double ynorm = sqrt(dot4_quad(y, y, ne, lane));
    const double tol = a.eps[p];
    int64_t scans = 0, kdone = 0;
    double rnorm = ynorm;
    bool dense = false, flag = false;

    if (!(ynorm <= tol)) {
      for (int64_t k = 0; k < k_max; k++) {
        scans += c - k;
        // ---- correlation scan (_kernels.py:94-103): 8 lane-quads, each a candidate
        double best = -1.0;
        int64_t bestj = -1;
        const int grp = lane >> 2;
        for (int64_t base = 0; base < c; base += 8) {
          const int64_t jl = base + grp;
          const bool live = jl < c && !((taken[jl >> 5] >> (jl & 31)) & 1u);
          const int64_t g = jl < c ? cs.id(p, jl) : 0;
          double v = rw ? dot4_quad_c(a.mat_t + g * n, rw, fan, ord, r, ne, lane)
                        : dot4_quad(a.mat_t + g * n, r, n, lane);
          if (v < 0.0) v = -v;
          if (live && v > best) {
            best = v;
            bestj = jl;
          }
        }
        warp_argmax(best, bestj);
        if (bestj < 0 || best <= 0.0) break;
        if (lane == 0) taken[bestj >> 5] |= 1u << (bestj & 31);
        const int64_t g = cs.id(p, bestj);
        if (lane == 0) sel[kdone] = g;
        kdone += 1;

        if (!dense) {
          // ---- MGS with one re-orthogonalisation (_kernels.py:111-137)
          for (int64_t i = lane; i < ne; i += 32)
            u[i] = rw ? eff_at(a.mat_t + g * n, rw, fan, ord, i) : a.mat_t[g * n + i];
          __syncwarp();
          const double anorm = sqrt(dot4_quad(u, u, ne, lane));
          for (int pass = 0; pass < 2; pass++) {
            for (int64_t j = 0; j < kdone - 1; j++) {
              const double w = dot4_quad(qmat + j * n, u, ne, lane);
              __syncwarp();
              for (int64_t i = lane; i < ne; i += 32) u[i] -= w * qmat[j * n + i];
              if (lane == 0) {
                if (pass == 0)
                  rmat[j * kw + (kdone - 1)] = w;
                else
                  rmat[j * kw + (kdone - 1)] += w;
              }
              __syncwarp();
            }
          }
          const double d = sqrt(dot4_quad(u, u, ne, lane));
          const double floor_ = anorm > 1e-300 ? anorm : 1e-300;
          if (d <= RANK_TOL * floor_) {
            dense = true;
            flag = true;
          } else {
            if (lane == 0) rmat[(kdone - 1) * kw + (kdone - 1)] = d;
            double *qk = qmat + (kdone - 1) * n;
            for (int64_t i = lane; i < ne; i += 32) qk[i] = u[i] / d;
            __syncwarp();
            const double z = dot4_quad(qk, r, ne, lane);
            if (lane == 0) qty[kdone - 1] = z;
            __syncwarp();
            for (int64_t i = lane; i < ne; i += 32) r[i] -= z * qk[i];
            __syncwarp();
            rnorm = sqrt(dot4_quad(r, r, ne, lane));
          }
        }
        if (dense) {
          // ---- dense minimum-norm fallback (_kernels.py:139-154)
          __syncwarp();
          for (int64_t j = 0; j < kdone; j++) {
            const int64_t gj = sel[j];
            for (int64_t i = lane; i < ne; i += 32)
              amat[j * ne + i] = rw ? eff_at(a.mat_t + gj * n, rw, fan, ord, i) : a.mat_t[gj * n + i];
          }
          __syncwarp();
          if (lane == 0) lstsq_min_norm(amat, ne, kdone, y, coefs, vwork);
          __syncwarp();
          for (int64_t i = lane; i < ne; i += 32) {
            double acc = 0.0;
            for (int64_t j = 0; j < kdone; j++)
              acc += (rw ? eff_at(a.mat_t + sel[j] * n, rw, fan, ord, i) : a.mat_t[sel[j] * n + i]) *
                     coefs[j];
            r[i] = y[i] - acc;
          }
          __syncwarp();
          rnorm = sqrt(dot4_quad(r, r, ne, lane));
          for (int64_t j = lane; j < kdone; j += 32) coef[j] = coefs[j];
        }
        __syncwarp();
        if (rnorm <= tol) break;
      }
      // ---- back-substitution R c = Q^T y (_kernels.py:159-164)
      if (kdone && !dense && lane == 0) {
        for (int64_t i = kdone - 1; i >= 0; i--) {
          double acc = qty[i];
          for (int64_t j = i + 1; j < kdone; j++) acc -= rmat[i * kw + j] * coef[j];
          coef[i] = acc / rmat[i * kw + i];
        }
      }
    }
    if (lane == 0) {
      a.out_count[p] = kdone;
      a.out_rnorm[p] = rnorm;
      a.out_scans[p] = scans;
      a.out_flag[p] = flag ? 1 : 0;
    }
    __syncwarp();
  }
}

}  // namespace

int64_t exact_work_stride(int64_t n, int64_t k_width, int64_t max_cands) {
  int64_t d = 3 * n + k_width * n + k_width * k_width + k_width + n * k_width + k_width +
              k_width * k_width + (max_cands + 63) / 64 + 1;
  return (d + 31) & ~int64_t(31);
}

cudaError_t launch_exact(const ExactArgs &args, const void *ys, bool ys_f32, int warps,
                         cudaStream_t stream) {
  ProfScope _ps("exact_omp", stream);
  if (args.p_count <= 0) return cudaSuccess;
  const int wpb = 4;
  const int blocks = (warps + wpb - 1) / wpb;
  if (ys_f32)
    exact_omp_kernel<float><<<blocks, wpb * 32, 0, stream>>>(args, (const float *)ys);
  else
    exact_omp_kernel<double><<<blocks, wpb * 32, 0, stream>>>(args, (const double *)ys);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cdb
