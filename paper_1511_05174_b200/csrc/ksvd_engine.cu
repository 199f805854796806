// K-SVD dictionary-update stage (SURVEY row f1 follow-on): crossdict
// learn._update_stage (learn.py:169-199) on the device.
//
// The stage is sequential over atoms (atom j's refit changes the residual
// columns the next atoms see), so one persistent cluster of 16 CTAs (N <= 64;
// ksvd_cluster_kernel below) or one CTA (larger N; ksvd_update_kernel) walks
// the atoms while the per-atom work -- gathering E_j, its Gram matrix, the
// leading eigenvector, and the rank-one update of E's columns -- is spread
// over the cluster's / CTA's threads.  Per atom j with users U (the signals whose code uses j,
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
#include <cstdlib>

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

// ---------------------------------------------------------------- cluster
// The same stage on a cluster of KC CTAs (one per SM, distributed shared
// memory): the atoms stay sequential, but each atom's work is spread over
// the cluster -- every per-user loop (E_j gather, rank-one update, partner
// vector, dead-atom code reset) and the dead-atom residual norms take a
// contiguous share of users / signals per CTA, and the Gram matrix is summed
// as KC partial Gram matrices (each over its CTA's users, mma.sync f64 tiles)
// that every CTA adds up from the others' shared memory in rank order.  The
// small power iteration then runs redundantly, bit-identically, in every CTA
// (no broadcast).  Cluster barriers (release / acquire) order the global
// writes of one atom before the reads of the next.  Left case (|U| >= N)
// only when the N x N Gram matrix fits shared memory; |U| < N (E_j^T E_j) is
// computed redundantly per CTA (|U| < N is small).

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// generic address of the same shared variable in CTA `rank` of the cluster
template <typename T>
__device__ __forceinline__ const T *cl_map(const T *p, unsigned rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"((uint64_t)p), "r"(rank));
  return (const T *)out;
}

// acc[i][j] += sum_{k in [k0, k1)} A[k][2 rb + i] A[k][cb + cs j]: one thread's
// 2 x 4 tile of A^T A (A row-major in shared memory, zero-padded columns,
// cs = np8 / 4 column groups).  Columns interleaved by cs so the 16 threads of
// a half-warp read 16 consecutive doubles (conflict-free) and the two
// half-warps the same ones (broadcast); the row pair is a broadcast too.
__device__ __forceinline__ void syrk_tile(const double *A, int ld, int cs, int k0, int k1, int rb,
                                          int cb, double (&acc)[2][4]) {
  const double *pa = A + 2 * rb, *pb = A + cb;
#pragma unroll 4
  for (int k = k0; k < k1; k++) {
    const double2 x = *(const double2 *)(pa + k * ld);
    const double y0 = pb[k * ld], y1 = pb[k * ld + cs], y2 = pb[k * ld + 2 * cs],
                 y3 = pb[k * ld + 3 * cs];
    acc[0][0] = fma(x.x, y0, acc[0][0]);
    acc[0][1] = fma(x.x, y1, acc[0][1]);
    acc[0][2] = fma(x.x, y2, acc[0][2]);
    acc[0][3] = fma(x.x, y3, acc[0][3]);
    acc[1][0] = fma(x.y, y0, acc[1][0]);
    acc[1][1] = fma(x.y, y1, acc[1][1]);
    acc[1][2] = fma(x.y, y2, acc[1][2]);
    acc[1][3] = fma(x.y, y3, acc[1][3]);
  }
}

// Partial Gram matrix B = E_U^T E_U over rows [c0, c1) of the user-major E_j
// (ld n, n <= 64): staged CH rows at a time (loads in flight, then the
// stores) into a zero-padded [CH][np8] tile; thread t owns the 2 x 4 output
// tile (t / (np8 / 4), t % (np8 / 4)).  fp64 FMAs -- the m8n8k4 DMMA chain of
// the single-CTA kernel measured ~4x slower here (a dependent DMMA per k-step).
__device__ void gram_part(const double *ej, int64_t n, int64_t c0, int64_t c1, double *chunk,
                          double *B) {
  const int tid = threadIdx.x;
  const int ms = (int)n, np8 = (ms + 7) & ~7, cbn = np8 / 4;
  const bool own = tid < (np8 / 2) * cbn;
  const int rb = own ? tid / cbn : 0, cb = own ? tid % cbn : 0;
  double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  for (int64_t k0 = c0; k0 < c1; k0 += CH) {
    const int kc = (int)(c1 - k0 < CH ? c1 - k0 : CH);
    for (int idx0 = 0; idx0 < CH * np8; idx0 += 4 * KT) {  // 4 loads in flight, then the stores
      double t4[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int idx = idx0 + q * KT + tid, k = idx / np8, i = idx - k * np8;
        t4[q] = idx < CH * np8 && k < kc && i < ms ? __ldg(ej + (k0 + k) * n + i) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; q++)
        if (idx0 + q * KT + tid < CH * np8) chunk[idx0 + q * KT + tid] = t4[q];
    }
    __syncthreads();
    if (own) syrk_tile(chunk, np8, cbn, 0, kc, rb, cb, acc);
    __syncthreads();
  }
  if (own) {
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int r = 2 * rb + i, c = cb + cbn * j;
        if (r < ms && c < ms) B[r * ms + c] = acc[i][j];
      }
  }
  __syncthreads();
}

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
// phase timer (CTA 0, thread 0; a.prof != NULL: CDB_KSVD_PROF=1)
#define KPROF(slot)                                              \
  if (a.prof && rank == 0 && tid == 0) {                         \
    const uint64_t t_ = gtime();                                 \
    a.prof[slot] += (long long)(t_ - tprev);                     \
    tprev = t_;                                                  \
  }

template <int KC>
__global__ void __launch_bounds__(KT, 1) ksvd_cluster_kernel(KsvdArgs a) {
  extern __shared__ double ks[];
  const int64_t n = a.n, m = a.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = cl_rank();
  const int np8 = (int)((n + 7) & ~7);
  double *v = ks;                  // n
  double *w = v + n;               // n
  double *dj = w + n;              // n
  double *uv = dj + n;             // n
  double *red = uv + n;            // 96 (two 48-double reduction buffers)
  double *xch = red + 96;          // 4: cluster exchange slot of this CTA
  double *bfull = xch + 4;         // n x n: the Gram matrix (or u x u, u < n)
  double *bpart = bfull + n * n;   // n x n: this CTA's partial
  double *chunk = bpart + n * n;   // CH x np8
  int64_t replaced = 0;
  const int64_t c_step = n <= KT ? KT / n : 1, c_off = n <= KT ? tid / n : 0;
  const int64_t i_step = n <= KT ? n : KT, i_off = n <= KT ? tid % n : tid;
  const bool idle = n <= KT && c_off >= c_step;
  uint64_t tprev = gtime();
  for (int64_t j = 0; j < a.t; j++) {
    KPROF(0)
    cl_sync();  // the previous atom's E / d / code writes, cluster-wide
    KPROF(1)
    const int64_t b0 = a.ptr[j], u = a.ptr[j + 1] - b0;
    const int64_t ua = u * rank / KC, ub = u * (rank + 1) / KC;  // this CTA's users
    double *drow = a.d + j * n;
    for (int64_t i = tid; i < n; i += KT) dj[i] = drow[i];
    __syncthreads();
    if (u < a.threshold) {
      // ---- dead atom (learn.py:179-191)
      for (int64_t c = ua + (idle ? ub : c_off); c < ub; c += c_step) {
        const int64_t p = a.sig[b0 + c];
        const double xc = a.val[b0 + c];
        for (int64_t i = i_off; i < n; i += i_step)
          a.e[p * n + i] = __dadd_rn(a.e[p * n + i], __dmul_rn(dj[i], xc));
      }
      for (int64_t c = ua + tid; c < ub; c += KT) a.val[b0 + c] = 0.0;
      cl_sync();  // every user's residual restored before the norms
      const int64_t pa = m * rank / KC, pb = m * (rank + 1) / KC;
      double best = -2.0;
      int64_t bi = -1;
      for (int64_t p = pa + tid; p < pb; p += KT) {
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
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || ov > best || (ov == best && oi < bi))) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        red[warp] = best;
        ((int64_t *)red)[32 + warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        for (int q = 1; q < KT / 32; q++) {
          const double vq = red[q];
          const int64_t iq = ((int64_t *)red)[32 + q];
          if (iq >= 0 && (bi < 0 || vq > best || (vq == best && iq < bi))) {
            best = vq;
            bi = iq;
          }
        }
        xch[0] = best;
        ((int64_t *)xch)[1] = bi;
      }
      cl_sync();  // every CTA's best in its slot
      if (tid == 0) {  // np.argmax over all signals: lowest index among equal maxima
        double gb = -2.0;
        int64_t gi = -1;
        for (unsigned r = 0; r < KC; r++) {
          const double *x = cl_map(xch, r);
          const double vr = x[0];
          const int64_t ir = ((const int64_t *)x)[1];
          if (ir >= 0 && (gi < 0 || vr > gb || (vr == gb && ir < gi))) {
            gb = vr;
            gi = ir;
          }
        }
        ((int64_t *)red)[0] = gi;
        if (rank == 0) a.taken[gi >> 5] |= 1u << (gi & 31);
      }
      __syncthreads();
      const int64_t worst = ((int64_t *)red)[0];
      const double *yw = a.y + worst * n;
      double sq = 0.0;
      for (int64_t i = tid; i < n; i += KT) sq = fma(yw[i], yw[i], sq);
      const double cn = sqrt(block_sum(sq, red));
      if (rank == 0 && cn > 0.0)
        for (int64_t i = tid; i < n; i += KT) drow[i] = yw[i] / cn;
      replaced++;
      KPROF(2)
      continue;
    }
    const bool left = u >= n;
    const int64_t ms = left ? n : u;
    double *ej = a.ej;  // u x n, user-major
    for (int64_t c0 = ua + (idle ? ub : c_off); c0 < ub; c0 += 4 * c_step) {
      int64_t pp[4];  // four users per pass: ids, codes and E rows in flight together
      double xc[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int64_t c = c0 + q * c_step;
        pp[q] = c < ub ? a.sig[b0 + c] : -1;
        xc[q] = c < ub ? a.val[b0 + c] : 0.0;
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
    if (left) {
      __syncthreads();
      KPROF(3)
      gram_part(ej, n, ua, ub, chunk, bpart);
      KPROF(4)
      cl_sync();  // every partial in place
      // CTA `rank` sums its 1 / KC of the entries over the KC partials (rank
      // order, all loads in flight) and stores the sum into every CTA's B
      const int64_t oa = n * n * rank / KC, ob = n * n * (rank + 1) / KC;
      for (int64_t o = oa + tid; o < ob; o += KT) {
        double pv[KC];
#pragma unroll
        for (int r = 0; r < KC; r++) pv[r] = cl_map(bpart, (unsigned)r)[o];
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < KC; r++) s += pv[r];
#pragma unroll
        for (int r = 0; r < KC; r++) ((double *)cl_map(bfull, (unsigned)r))[o] = s;
      }
      cl_sync();  // B complete in every CTA
      KPROF(5)
    } else {
      cl_sync();  // every user's E_j row in place; B = E_j E_j^T (u x u), redundant
      for (int64_t o = tid; o < u * u; o += KT) {
        const int64_t r = o / u, c = o - r * u;
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s = fma(ej[r * n + i], ej[c * n + i], s);
        bfull[o] = s;
      }
    }
    __syncthreads();
    KPROF(6)
    const double *B = bfull;
    // power iteration (as ksvd_update_kernel), warm-started
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
    // Power iteration on four warps (ms <= 64: lane owns rows lane, lane + 32;
    // warp q sums the columns c = q mod 4 -- the fp64 pipe of one SM
    // sub-partition is narrow, so the 64 x 64 matvec is spread over all four),
    // named barriers only.  Each warp adds the four partial w's itself and
    // reduces v.w, w.w and the previous step's |v - v_prev|^2 (identical in
    // all four); the step that sees |dv|^2 < 1e-28 for its input stops (one
    // matvec past the plain loop's exit: at least as converged).
    double lam = 0.0, wn = 0.0;
    if (warp < 4) {
      double *wp = chunk;  // 4 x 64 partial w's (the Gram staging tile is free here)
      const bool h0 = lane < ms, h1 = lane + 32 < ms;
      const int msi = (int)ms;
      const double *bl = B + (h0 ? lane : 0), *bh = B + (h1 ? lane + 32 : 0);
      double v0 = h0 ? v[lane] : 0.0, v1 = h1 ? v[lane + 32] : 0.0;
      double ddp = 0.0;
      int it_done = 0;
      for (int it = 0; it < 20000; it++) {
        it_done = it;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        int c = warp;
        for (; c + 4 < msi; c += 8) {
          const double vc0 = v[c], vc1 = v[c + 4];
          a0 = fma(bl[c * msi], vc0, a0);
          b0 = fma(bh[c * msi], vc0, b0);
          a1 = fma(bl[(c + 4) * msi], vc1, a1);
          b1 = fma(bh[(c + 4) * msi], vc1, b1);
        }
        if (c < msi) {
          const double vc0 = v[c];
          a0 = fma(bl[c * msi], vc0, a0);
          b0 = fma(bh[c * msi], vc0, b0);
        }
        wp[warp * 64 + lane] = a0 + a1;
        wp[warp * 64 + 32 + lane] = b0 + b1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        double w0 = 0.0, w1 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          w0 += wp[q * 64 + lane];
          w1 += wp[q * 64 + 32 + lane];
        }
        if (!h0) w0 = 0.0;
        if (!h1) w1 = 0.0;
        double vw = fma(v0, w0, v1 * w1), ww = fma(w0, w0, w1 * w1), sd = ddp;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          vw += __shfl_xor_sync(CDB_FULL_MASK, vw, o);
          ww += __shfl_xor_sync(CDB_FULL_MASK, ww, o);
          sd += __shfl_xor_sync(CDB_FULL_MASK, sd, o);
        }
        if (it > 0 && sd < 1e-28) break;  // the input v had converged: keep it
        lam = vw;
        wn = sqrt(ww);
        if (!(wn > 0.0)) break;
        const double x0 = w0 / wn, x1 = w1 / wn;
        ddp = h0 ? (x0 - v0) * (x0 - v0) : 0.0;
        if (h1) ddp = fma(x1 - v1, x1 - v1, ddp);
        v0 = h0 ? x0 : 0.0;
        v1 = h1 ? x1 : 0.0;
        if (warp == 0) {
          if (h0) v[lane] = v0;
          if (h1) v[lane + 32] = v1;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      if (warp == 0 && lane == 0) {
        red[0] = lam;
        red[1] = wn;
      }
      if (a.prof && rank == 0 && warp == 0 && lane == 0) a.prof[10] += 1000 * (it_done + 1);
    }
    __syncthreads();
    lam = red[0];
    wn = red[1];
    __syncthreads();
    KPROF(7)
    const double sigma = wn > 0.0 ? sqrt(lam > 0.0 ? lam : 0.0) : 0.0;
    if (!(sigma > 0.0)) {  // zero E_j: LAPACK's U = I, s = 0
      if (rank == 0)
        for (int64_t i = tid; i < n; i += KT) drow[i] = i == 0 ? 1.0 : 0.0;
      for (int64_t c = ua + tid; c < ub; c += KT) a.val[b0 + c] = 0.0;
      continue;
    }
    // partner vector: left -> x = E_j^T u over this CTA's users, norm cluster-wide;
    // right -> u = E_j v (all users; redundant)
    double nrx = 1.0;
    if (left) {
      for (int64_t i = tid; i < n; i += KT) uv[i] = v[i];
      __syncthreads();
      double s2 = 0.0;
      for (int64_t c0 = ua + warp; c0 < ub; c0 += 4 * (KT / 32)) {  // 4 users per warp pass
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t i = lane; i < n; i += 32) {
          double e4[4];
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const int64_t c = c0 + q * (KT / 32);
            e4[q] = c < ub ? ej[c * n + i] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 4; q++) s4[q] = fma(e4[q], uv[i], s4[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const double s = warp_sum(s4[q]);
          const int64_t c = c0 + q * (KT / 32);
          if (lane == 0 && c < ub) {
            a.val[b0 + c] = s;
            s2 = fma(s, s, s2);
          }
        }
      }
      s2 = block_sum(s2, red);
      if (tid == 0) xch[2] = s2;
      cl_sync();
      double pv[KC];
#pragma unroll
      for (int r = 0; r < KC; r++) pv[r] = cl_map(xch, (unsigned)r)[2];
      double tot = 0.0;
#pragma unroll
      for (int r = 0; r < KC; r++) tot += pv[r];
      nrx = sqrt(tot);
    } else {
      double s2 = 0.0;
      for (int64_t i = tid; i < n; i += KT) {
        double s = 0.0;
        for (int64_t c = 0; c < u; c++) s = fma(ej[c * n + i], v[c], s);
        uv[i] = s;
        s2 = fma(s, s, s2);
      }
      const double nr = sqrt(block_sum(s2, red));
      for (int64_t i = tid; i < n; i += KT) uv[i] /= nr;
    }
    __syncthreads();
    if (warp == 0) {  // sign: the largest-magnitude entry of u positive (lowest index on ties)
      double bm = -1.0;
      int64_t im = 0;
      for (int64_t i = lane; i < n; i += 32)
        if (fabs(uv[i]) > bm) {
          bm = fabs(uv[i]);
          im = i;
        }
      const double gm = warp_max_nonneg(bm);
      const unsigned gi = __reduce_min_sync(0xffffffffu, bm == gm ? (unsigned)im : 0xffffffffu);
      if (lane == 0) red[0] = uv[gi] < 0.0 ? -1.0 : 1.0;
    }
    __syncthreads();
    const double sg = red[0];
    for (int64_t i = tid; i < n; i += KT) {
      uv[i] *= sg;
      if (rank == 0) drow[i] = uv[i];
    }
    for (int64_t c = ua + tid; c < ub; c += KT)
      a.val[b0 + c] = left ? sigma * (sg * (a.val[b0 + c] / nrx)) : sigma * (sg * v[c]);
    __syncthreads();
    KPROF(8)
    for (int64_t c0 = ua + (idle ? ub : c_off); c0 < ub; c0 += 4 * c_step) {
      int64_t pp[4];
      double xc[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int64_t c = c0 + q * c_step;
        pp[q] = c < ub ? a.sig[b0 + c] : -1;
        xc[q] = c < ub ? a.val[b0 + c] : 0.0;
      }
      for (int64_t i = i_off; i < n; i += i_step) {
        double ev[4];
#pragma unroll
        for (int q = 0; q < 4; q++) ev[q] = pp[q] >= 0 ? ej[(c0 + q * c_step) * n + i] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (pp[q] >= 0) a.e[pp[q] * n + i] = __dsub_rn(ev[q], __dmul_rn(uv[i], xc[q]));
      }
    }
    KPROF(9)
  }
  cl_sync();
  if (tid == 0 && rank == 0) *a.replaced = replaced;
}

}  // namespace

size_t ksvd_update_smem(int64_t n, int64_t smem_b) {
  return sizeof(double) * (4 * n + 32 + smem_b + (int64_t)(CH + 1) * n);
}

size_t ksvd_cluster_smem(int64_t n) {
  return sizeof(double) * (4 * n + 96 + 4 + 2 * n * n + (int64_t)CH * ((n + 7) & ~7));
}

cudaError_t launch_ksvd_update(const KsvdArgs &a, size_t smem, cudaStream_t stream) {
  // cluster of 16 CTAs (non-portable size) when the device allows it, else 8;
  // CDB_KSVD_CLUSTER=0 -> the single-CTA kernel, =8|16 -> that cluster size
  const char *cv = getenv("CDB_KSVD_CLUSTER");
  const int want = cv ? atoi(cv) : 16;
  const size_t csm = ksvd_cluster_smem(a.n);
  if (want != 0 && a.n <= 64 && csm <= 200 * 1024) {
    auto k16 = ksvd_cluster_kernel<16>;
    auto k8 = ksvd_cluster_kernel<8>;
    int kc = want == 8 ? 8 : 16;
    cudaError_t e = cudaSuccess;
    if (kc == 16 &&
        (cudaFuncSetAttribute(k16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
             cudaSuccess ||
         cudaFuncSetAttribute(k16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm) !=
             cudaSuccess)) {
      (void)cudaGetLastError();
      kc = 8;
    }
    if (kc == 16) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(KT);
      cfg.dynamicSmemBytes = csm;
      cfg.stream = stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, (void *)k16, &cfg) != cudaSuccess || ncl < 1) {
        (void)cudaGetLastError();
        kc = 8;
      } else {
        ProfScope _ps("ksvd_update", stream);
        e = cudaLaunchKernelEx(&cfg, k16, a);
        note_launch();
        return e != cudaSuccess ? e : cudaGetLastError();
      }
    }
    if ((e = cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm)) !=
        cudaSuccess)
      return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8);
    cfg.blockDim = dim3(KT);
    cfg.dynamicSmemBytes = csm;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope _ps("ksvd_update", stream);
    e = cudaLaunchKernelEx(&cfg, k8, a);
    note_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  cudaError_t e = cudaFuncSetAttribute(ksvd_update_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ProfScope _ps("ksvd_update", stream);
  ksvd_update_kernel<<<1, KT, smem, stream>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cdb
