// K-SVD dictionary-update stage (SURVEY row f1 follow-on): crossdict
// learn._update_stage (learn.py:169-199) on the device.
//
// The stage is sequential over atoms (atom j's refit changes the residual
// columns the next atoms see), so one persistent CTA walks the atoms while
// the per-atom work -- gathering E_j, its Gram matrix, the leading
// eigenvector, and the rank-one update of E's columns -- is spread over the
// CTA's threads.  Per atom j with users U (the signals whose code uses j,
// ascending):
//
//   |U| < threshold:  E[:, U] += d_j x_j[U]; x_j[U] = 0; the signal with the
//                     largest residual norm not already taken replaces the
//                     atom, d_j = y_w / |y_w|   (learn.py:179-191)
//   otherwise:        E_j = E[:, U] + d_j x_j[U]; (u, s, v) = leading
//                     singular triple of E_j; d_j = u; x_j[U] = s v;
//                     E[:, U] = E_j - u (s v)^T  (learn.py:192-198)
//
// The leading triple comes from the smaller Gram matrix (E_j E_j^T when
// |U| >= N, else E_j^T E_j) by power iteration warm-started from the old atom
// (or the old code row), to |v_{i+1} - v_i| < 1e-14; the partner vector is
// E_j^T u / s (or E_j v / s).  The reference calls LAPACK's SVD
// (np.linalg.svd), whose singular vectors carry an arbitrary sign: here the
// largest-magnitude entry of u is made positive, and the results agree with
// the reference's up to that per-atom sign at ~1e-12 (parity by tolerance,
// not bits).  The elementwise updates use the reference's rounding (product
// rounded, then the sum: no contraction), and the replacement's residual
// norms are numpy's sequential sum of squares, so the replacement pick is
// the reference's.
#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

constexpr int KT = 512;  // threads of the update CTA
constexpr int CH = 32;   // summation-index chunk of the Gram matrix
constexpr int TG = 8;    // Gram tiles per warp per pass

// Block-wide sum of one double per thread (all threads get the result).
__device__ double block_sum(double v, double *red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < KT / 32; w++) s += red[w];
  return s;
}

// Two block-wide sums in one pass (red holds 2 x KT/32 doubles).
__device__ double2 block_sum2(double2 v, double *red) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    red[warp] = v.x;
    red[KT / 32 + warp] = v.y;
  }
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  for (int w = 0; w < KT / 32; w++) {
    s.x += red[w];
    s.y += red[KT / 32 + w];
  }
  return s;
}

__global__ void __launch_bounds__(KT, 1) ksvd_update_kernel(KsvdArgs a) {
  extern __shared__ double ks[];
  const int64_t n = a.n, m = a.m;
  const int tid = threadIdx.x;
  double *v = ks;                 // n: power-iteration vector
  double *w = v + n;              // n
  double *dj = w + n;             // n: the atom before its refit
  double *uv = dj + n;            // n: left singular vector
  double *red = uv + n;           // 32
  double *bs = red + 32;          // Gram matrix when it fits
  __shared__ double s_val[KT / 32];
  __shared__ int64_t s_idx[KT / 32];
  int64_t replaced = 0;
  // (user, coordinate) loops: n <= KT -> KT / n users at a time, one thread per
  // coordinate; otherwise one user at a time, coordinates strided
  const int64_t c_step = n <= KT ? KT / n : 1, c_off = n <= KT ? tid / n : 0;
  const int64_t i_step = n <= KT ? n : KT, i_off = n <= KT ? tid % n : tid;
  const bool idle = n <= KT && c_off >= c_step;  // the KT % n leftover threads
  for (int64_t j = 0; j < a.t; j++) {
    const int64_t b0 = a.ptr[j], u = a.ptr[j + 1] - b0;
    double *drow = a.d + j * n;
    for (int64_t i = tid; i < n; i += KT) dj[i] = drow[i];
    __syncthreads();
    if (u < a.threshold) {
      // ---- dead atom: drop its coefficients, re-seed from the worst-coded signal
      for (int64_t c = idle ? u : c_off; c < u; c += c_step) {
        const int64_t p = a.sig[b0 + c];
        const double xc = a.val[b0 + c];
        for (int64_t i = i_off; i < n; i += i_step)
          a.e[p * n + i] = __dadd_rn(a.e[p * n + i], __dmul_rn(dj[i], xc));
      }
      __syncthreads();
      for (int64_t c = tid; c < u; c += KT) a.val[b0 + c] = 0.0;
      double best = -2.0;
      int64_t bi = -1;
      for (int64_t p = tid; p < m; p += KT) {
        double rn = -1.0;
        if (!((a.taken[p >> 5] >> (p & 31)) & 1u)) {
          const double *ep = a.e + p * n;
          double s = __dmul_rn(ep[0], ep[0]);
          for (int64_t i = 1; i < n; i++) s = __dadd_rn(s, __dmul_rn(ep[i], ep[i]));
          rn = sqrt(s);
        }
        if (rn > best) {
          best = rn;
          bi = p;
        }
      }
      // arg-max over the CTA, lowest index among equal maxima (np.argmax)
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || ov > best || (ov == best && oi < bi))) {
          best = ov;
          bi = oi;
        }
      }
      if ((tid & 31) == 0) {
        s_val[tid >> 5] = best;
        s_idx[tid >> 5] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        for (int q = 1; q < KT / 32; q++)
          if (s_idx[q] >= 0 &&
              (bi < 0 || s_val[q] > best || (s_val[q] == best && s_idx[q] < bi))) {
            best = s_val[q];
            bi = s_idx[q];
          }
        s_idx[0] = bi;
        a.taken[bi >> 5] |= 1u << (bi & 31);
      }
      __syncthreads();
      const int64_t worst = s_idx[0];
      const double *yw = a.y + worst * n;
      double sq = 0.0;
      for (int64_t i = tid; i < n; i += KT) sq = fma(yw[i], yw[i], sq);
      const double cn = sqrt(block_sum(sq, red));
      if (cn > 0.0)
        for (int64_t i = tid; i < n; i += KT) drow[i] = yw[i] / cn;
      replaced++;
      __syncthreads();
      continue;
    }
    // ---- rank-one refit: E_j, its Gram matrix, the leading singular pair
    double *ej = a.ej;  // u x n, user-major
    {  // four users per pass: their ids, codes and E rows in flight together
      const int64_t c_lim = idle ? 0 : u;
      for (int64_t c0 = c_off; c0 < c_lim; c0 += 4 * c_step) {
        int64_t pp[4];
        double xc[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int64_t c = c0 + q * c_step;
          pp[q] = c < u ? a.sig[b0 + c] : -1;
          xc[q] = c < u ? a.val[b0 + c] : 0.0;
        }
        for (int64_t i = i_off; i < n; i += i_step) {
          double ev[4];
#pragma unroll
          for (int q = 0; q < 4; q++) ev[q] = pp[q] >= 0 ? a.e[pp[q] * n + i] : 0.0;
#pragma unroll
          for (int q = 0; q < 4; q++)
            if (pp[q] >= 0) ej[(c0 + q * c_step) * n + i] = __dadd_rn(ev[q], __dmul_rn(dj[i], xc[q]));
        }
      }
    }
    __syncthreads();
    const bool left = u >= n;
    const int64_t ms = left ? n : u;
    double *B = ms * ms <= a.smem_b ? bs : a.bglob;
    // Gram matrix on the FP64 tensor cores (mma.sync m8n8k4 f64): 8 x 8 tiles
    // on and above the diagonal, each warp accumulating up to TG tiles in
    // registers over the whole summation index (staged through shared memory
    // CH at a time), written once and mirrored
    double *chunk = bs + a.smem_b;  // CH x n (left) or u x (CH + 1) (right)
    {
      const int warp = tid >> 5, lane = tid & 31;
      const int nt = (int)((ms + 7) / 8), ntiles = nt * (nt + 1) / 2;
      const int64_t kext = left ? u : n;
      for (int g0 = 0; g0 < ntiles; g0 += (KT / 32) * TG) {
        double acc[TG][2];
        int trow[TG], tcol[TG];
#pragma unroll
        for (int q = 0; q < TG; q++) {
          acc[q][0] = acc[q][1] = 0.0;
          int id = g0 + warp + (KT / 32) * q, tr = 0;
          while (id >= 0 && tr < nt && id >= nt - tr) id -= nt - tr++;  // upper-triangle index
          trow[q] = id < ntiles && tr < nt ? tr : -1;
          tcol[q] = tr + id;
          if (g0 + warp + (KT / 32) * q >= ntiles) trow[q] = -1;
        }
        for (int64_t k0 = 0; k0 < kext; k0 += CH) {
          const int kc = (int)(kext - k0 < CH ? kext - k0 : CH);
          if (left) {
            for (int64_t idx = tid; idx < kc * n; idx += KT) chunk[idx] = ej[k0 * n + idx];
          } else {
            for (int64_t c = idle ? u : c_off; c < u; c += c_step)
              for (int64_t ii = i_off; ii < kc; ii += i_step) chunk[c * (CH + 1) + ii] = ej[c * n + k0 + ii];
          }
          __syncthreads();
          for (int ks = 0; ks < kc; ks += 4) {
            const int kk = ks + (lane & 3);
#pragma unroll
            for (int q = 0; q < TG; q++) {
              if (trow[q] < 0) continue;  // warp-uniform
              const int r = trow[q] * 8 + (lane >> 2), c = tcol[q] * 8 + (lane >> 2);
              double av = 0.0, bv = 0.0;
              if (kk < kc) {
                if (r < ms) av = left ? chunk[kk * n + r] : chunk[r * (CH + 1) + kk];
                if (c < ms) bv = left ? chunk[kk * n + c] : chunk[c * (CH + 1) + kk];
              }
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(acc[q][0]), "+d"(acc[q][1])
                           : "d"(av), "d"(bv));
            }
          }
          __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < TG; q++) {
          if (trow[q] < 0) continue;
          const int r = trow[q] * 8 + (lane >> 2);
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int c = tcol[q] * 8 + 2 * (lane & 3) + h;
            if (r < ms && c < ms) {
              B[(int64_t)r * ms + c] = acc[q][h];
              B[(int64_t)c * ms + r] = acc[q][h];
            }
          }
        }
      }
      __syncthreads();
    }
    // warm start: the old atom (left) or the old code row (right)
    double nv = 0.0;
    for (int64_t i = tid; i < ms; i += KT) {
      const double x0 = left ? dj[i] : a.val[b0 + i];
      v[i] = x0;
      nv = fma(x0, x0, nv);
    }
    nv = sqrt(block_sum(nv, red));
    if (!(nv > 0.0)) {
      for (int64_t i = tid; i < ms; i += KT) v[i] = i == 0 ? 1.0 : 0.0;
      nv = 1.0;
    }
    for (int64_t i = tid; i < ms; i += KT) v[i] /= nv;
    __syncthreads();
    double lam = 0.0, wn = 0.0;
    // matvec layout: gpr threads per row (a power of two <= 32), rows strided
    int gpr = 1;
    while (gpr < 32 && (int64_t)(KT / (2 * gpr)) >= ms) gpr *= 2;
    const int rows_per_pass = KT / gpr, part = tid % gpr;
    for (int it = 0; it < 20000; it++) {
      double vw = 0.0, ww = 0.0;
      for (int64_t r0 = 0; r0 < ms; r0 += rows_per_pass) {
        const int64_t r = r0 + tid / gpr;
        double s = 0.0;
        if (r < ms) {  // four partial sums: loads of B in flight together
          double s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int64_t c = part;
          for (; c + 3 * gpr < ms; c += 4 * gpr) {
            const double b0v = B[r * ms + c], b1v = B[r * ms + c + gpr],
                         b2v = B[r * ms + c + 2 * gpr], b3v = B[r * ms + c + 3 * gpr];
            s = fma(b0v, v[c], s);
            s1 = fma(b1v, v[c + gpr], s1);
            s2 = fma(b2v, v[c + 2 * gpr], s2);
            s3 = fma(b3v, v[c + 3 * gpr], s3);
          }
          for (; c < ms; c += gpr) s = fma(B[r * ms + c], v[c], s);
          s = (s + s1) + (s2 + s3);
        }
        for (int o = gpr / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (r < ms && part == 0) {
          w[r] = s;
          vw = fma(v[r], s, vw);
          ww = fma(s, s, ww);
        }
      }
      double2 sums = block_sum2(make_double2(vw, ww), red);
      lam = sums.x;
      wn = sqrt(sums.y);
      if (!(wn > 0.0)) break;  // E_j = 0
      double dd = 0.0;
      for (int64_t r = tid; r < ms; r += KT) {
        const double x1 = w[r] / wn;
        dd = fma(x1 - v[r], x1 - v[r], dd);
        w[r] = x1;
      }
      dd = block_sum(dd, red);
      for (int64_t r = tid; r < ms; r += KT) v[r] = w[r];
      __syncthreads();
      if (dd < 1e-28) break;
    }
    const double sigma = wn > 0.0 ? sqrt(lam > 0.0 ? lam : 0.0) : 0.0;
    if (!(sigma > 0.0)) {  // zero E_j: LAPACK's U = I, s = 0
      for (int64_t i = tid; i < n; i += KT) drow[i] = i == 0 ? 1.0 : 0.0;
      for (int64_t c = tid; c < u; c += KT) a.val[b0 + c] = 0.0;
      __syncthreads();
      continue;
    }
    // partner vector, both normalised; w holds the right vector (length u)
    if (left) {
      for (int64_t i = tid; i < n; i += KT) uv[i] = v[i];
      __syncthreads();
      double s2 = 0.0;
      {  // a warp per user row: coalesced, lanes over the coordinates
        const int lane = tid & 31, wp = tid >> 5;
        for (int64_t c = wp; c < u; c += KT / 32) {
          double s = 0.0;
          for (int64_t i = lane; i < n; i += 32) s = fma(ej[c * n + i], uv[i], s);
          s = warp_sum(s);
          if (lane == 0) {
            a.val[b0 + c] = s;  // scratch: E_j^T u
            s2 = fma(s, s, s2);
          }
        }
      }
      const double nr = sqrt(block_sum(s2, red));
      for (int64_t c = tid; c < u; c += KT) a.val[b0 + c] /= nr;
    } else {
      for (int64_t c = tid; c < u; c += KT) a.val[b0 + c] = v[c];
      __syncthreads();
      double s2 = 0.0;
      for (int64_t i = tid; i < n; i += KT) {
        double s = 0.0;
        for (int64_t c = 0; c < u; c++) s = fma(ej[c * n + i], a.val[b0 + c], s);
        uv[i] = s;
        s2 = fma(s, s, s2);
      }
      const double nr = sqrt(block_sum(s2, red));
      for (int64_t i = tid; i < n; i += KT) uv[i] /= nr;
    }
    __syncthreads();
    // sign: the largest-magnitude entry of u positive (lowest index on ties)
    if (tid == 0) {
      int64_t im = 0;
      for (int64_t i = 1; i < n; i++)
        if (fabs(uv[i]) > fabs(uv[im])) im = i;
      red[0] = uv[im] < 0.0 ? -1.0 : 1.0;
    }
    __syncthreads();
    const double sg = red[0];
    for (int64_t i = tid; i < n; i += KT) {
      uv[i] *= sg;
      drow[i] = uv[i];
    }
    for (int64_t c = tid; c < u; c += KT) a.val[b0 + c] = sigma * (sg * a.val[b0 + c]);
    __syncthreads();
    for (int64_t c = idle ? u : c_off; c < u; c += c_step) {
      const int64_t p = a.sig[b0 + c];
      const double xc = a.val[b0 + c];
      for (int64_t i = i_off; i < n; i += i_step)
        a.e[p * n + i] = __dsub_rn(ej[c * n + i], __dmul_rn(uv[i], xc));
    }
    __syncthreads();
  }
  if (tid == 0) *a.replaced = replaced;
}

}  // namespace

size_t ksvd_update_smem(int64_t n, int64_t smem_b) {
  return sizeof(double) * (4 * n + 32 + smem_b + (int64_t)(CH + 1) * n);
}

cudaError_t launch_ksvd_update(const KsvdArgs &a, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(ksvd_update_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ProfScope _ps("ksvd_update", stream);
  ksvd_update_kernel<<<1, KT, smem, stream>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cdb
