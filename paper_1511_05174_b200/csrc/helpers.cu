// Small memory-bound kernels around the OMP engines.
#include <cuda_fp16.h>

#include <cstdint>
#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

struct Shape4 {
  int64_t fine[4], fac[4], coarse[4];
  int rank;
};

// Block mean of row-major fine patches (crossdict/scaling.py:99-116,
// downsample_columns).  A CTA stages `spb` signal rows in shared memory with
// coalesced loads and builds once the fine index of every (coarse cell,
// in-block offset) -- offsets in row-major order, the summation order the
// oracle restates -- so the per-output work is `block` shared-memory reads.
template <typename YT>
__global__ void __launch_bounds__(256) downsample_kernel(const YT *__restrict__ ys, int64_t p,
                                                         int n, Shape4 sh,
                                                         double *__restrict__ out, int n_low,
                                                         int spb, double rel,
                                                         double *__restrict__ eps_low,
                                                         double *__restrict__ eps_fine) {
  extern __shared__ __align__(16) unsigned char dsm[];
  int *tab = (int *)dsm;                       // n_low * block fine indices
  YT *rows = (YT *)(dsm + ((size_t)n * 4 + 15) / 16 * 16);  // spb x n
  int block = 1;
  for (int d = 0; d < sh.rank; d++) block *= (int)sh.fac[d];
  for (int e = threadIdx.x; e < n_low * block; e += blockDim.x) {
    const int cell = e / block, bo = e % block;
    int cc[4] = {0, 0, 0, 0}, off[4] = {0, 0, 0, 0};
    int rem = cell, r = bo;
    for (int d = sh.rank - 1; d >= 0; d--) {
      cc[d] = rem % (int)sh.coarse[d];
      rem /= (int)sh.coarse[d];
      off[d] = r % (int)sh.fac[d];
      r /= (int)sh.fac[d];
    }
    int idx = 0;
    for (int d = 0; d < sh.rank; d++) idx = idx * (int)sh.fine[d] + cc[d] * (int)sh.fac[d] + off[d];
    tab[e] = idx;
  }
  // persistent CTAs: the index table is built once, then groups of spb
  // signals are staged with 16-byte loads (rows are 16-byte aligned when
  // n * sizeof(YT) is a multiple of 16)
  const bool vec = ((size_t)n * sizeof(YT)) % 16 == 0;
  constexpr int VE = 16 / sizeof(YT);
  for (int64_t s0 = (int64_t)blockIdx.x * spb; s0 < p; s0 += (int64_t)gridDim.x * spb) {
    const int ns = p - s0 < spb ? (int)(p - s0) : spb;
    __syncthreads();  // the previous group's rows are consumed
    if (vec) {
      const int4 *src = (const int4 *)(ys + s0 * n);
      int4 *dst = (int4 *)rows;
      const int64_t nv = (int64_t)ns * n / VE;
      for (int64_t e = threadIdx.x; e < nv; e += blockDim.x) dst[e] = __ldcs(src + e);
    } else {
      for (int64_t e = threadIdx.x; e < (int64_t)ns * n; e += blockDim.x) rows[e] = ys[s0 * n + e];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < ns * n_low; e += blockDim.x) {
      const int sl = e / n_low, cell = e % n_low;
      const YT *row = rows + (size_t)sl * n;
      const int *t = tab + cell * block;
      double acc = 0.0;
      for (int b = 0; b < block; b++) acc += (double)row[t[b]];
      out[(s0 + sl) * n_low + cell] = acc / (double)block;
    }
    if (!eps_low) continue;
    // fused stopping tolerances rel * |W y| (step 1) and rel * |y| (step 2)
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int sl = warp; sl < ns; sl += blockDim.x >> 5) {
      const YT *row = rows + (size_t)sl * n;
      double a = 0.0, b = 0.0;
      for (int i = lane; i < n; i += 32) a = fma((double)row[i], (double)row[i], a);
      const double *lo = out + (s0 + sl) * n_low;
      for (int i = lane; i < n_low; i += 32) b = fma(lo[i], lo[i], b);
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == 0) {
        eps_fine[s0 + sl] = rel * sqrt(a);
        eps_low[s0 + sl] = rel * sqrt(b);
      }
    }
  }
}

// Direct block means (no staging): one thread per coarse cell reads its
// `block` fine entries straight from HBM (each fine entry is read exactly once
// over the CTA, so the sectors are fully used) and the fine / coarse squared
// norms are reduced per signal in a fixed order (deterministic tolerances).
// spi = 256 / n_low signals per CTA pass when n_low < 256, else one signal
// with n_low / 256 cells per thread.
template <typename YT, int VW>
__global__ void __launch_bounds__(256) downsample_direct_kernel(
    const YT *__restrict__ ys, int64_t p, int n, int n_low, int block,
    const int *__restrict__ tab_g, double *__restrict__ out, double rel,
    double *__restrict__ eps_low, double *__restrict__ eps_fine) {
  extern __shared__ __align__(16) unsigned char dsm[];
  int *tab = (int *)dsm;  // n_low * block fine indices
  __shared__ double r_yy[2][256], r_yl[2][256];  // by pass parity: one barrier per pass
  int par = 0;
  for (int e = threadIdx.x; e < n_low * block; e += blockDim.x) tab[e] = tab_g[e];
  __syncthreads();
  const int tid = threadIdx.x;
  const int spi = n_low < 256 ? 256 / n_low : 1;
  const int tps = n_low < 256 ? n_low : 256;  // threads per signal
  const double inv_b = 1.0 / (double)block;
  for (int64_t s0 = (int64_t)blockIdx.x * spi; s0 < p; s0 += (int64_t)gridDim.x * spi) {
    double yy = 0.0, yl = 0.0;
    const int sl = tid / tps;
    const int64_t sig = s0 + sl;
    if (sl < spi && sig < p) {
      const YT *y = ys + sig * n;
      for (int cell = tid % tps; cell < n_low; cell += tps) {
        const int *t = tab + cell * block;
        double acc = 0.0;
        if constexpr (VW == 2) {  // the last axis' factor-2 pairs are adjacent: 8-byte loads
          if (block == 8) {  // 2 x 2 x 2 blocks (every 3-D BASELINE config): four loads in flight
            float2 v2[4];
#pragma unroll
            for (int b = 0; b < 4; b++) v2[b] = __ldcs((const float2 *)(y + t[2 * b]));
#pragma unroll
            for (int b = 0; b < 4; b++) {
              const double v0 = (double)v2[b].x, v1 = (double)v2[b].y;
              acc += v0;
              acc += v1;
              yy = fma(v0, v0, yy);
              yy = fma(v1, v1, yy);
            }
          } else
          for (int b = 0; b < block; b += 2) {
            const float2 v2 = __ldcs((const float2 *)(y + t[b]));
            const double v0 = (double)v2.x, v1 = (double)v2.y;
            acc += v0;
            acc += v1;
            yy = fma(v0, v0, yy);
            yy = fma(v1, v1, yy);
          }
        } else {
          for (int b = 0; b < block; b++) {
            const double v = (double)__ldcs(y + t[b]);
            acc += v;
            yy = fma(v, v, yy);
          }
        }
        const double m = acc * inv_b;
        out[sig * n_low + cell] = m;
        yl = fma(m, m, yl);
      }
    }
    if (!eps_low) continue;
    if (tps % 32 == 0) {
      // warp butterflies, then the warps of a signal in order (fixed order:
      // deterministic; a serial 256-term sum by one thread left the CTA
      // waiting at the barrier)
      yy = warp_sum(yy);
      yl = warp_sum(yl);
      const int lane = tid & 31, warp = tid >> 5, wps = tps / 32;
      if (lane == 0) {
        r_yy[par][warp] = yy;
        r_yl[par][warp] = yl;
      }
      __syncthreads();
      if (tid < spi && s0 + tid < p) {
        double a = 0.0, b = 0.0;
        for (int q = tid * wps; q < (tid + 1) * wps; q++) {
          a += r_yy[par][q];
          b += r_yl[par][q];
        }
        eps_fine[s0 + tid] = rel * sqrt(a);
        eps_low[s0 + tid] = rel * sqrt(b);
      }
      par ^= 1;  // the next pass writes the other buffer; its barrier orders the one after
      continue;
    }
    r_yy[par][tid] = yy;
    r_yl[par][tid] = yl;
    __syncthreads();
    if (tid < spi && s0 + tid < p) {
      double a = 0.0, b = 0.0;
      for (int q = tid * tps; q < (tid + 1) * tps; q++) {
        a += r_yy[par][q];
        b += r_yl[par][q];
      }
      eps_fine[s0 + tid] = rel * sqrt(a);
      eps_low[s0 + tid] = rel * sqrt(b);
    }
    par ^= 1;
  }
}

__global__ void downsample_table_kernel(Shape4 sh, int n_low, int *__restrict__ tab) {
  int block = 1;
  for (int d = 0; d < sh.rank; d++) block *= (int)sh.fac[d];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_low * block; e += gridDim.x * blockDim.x) {
    const int cell = e / block, bo = e % block;
    int cc[4] = {0, 0, 0, 0}, off[4] = {0, 0, 0, 0};
    int rem = cell, r = bo;
    for (int d = sh.rank - 1; d >= 0; d--) {
      cc[d] = rem % (int)sh.coarse[d];
      rem /= (int)sh.coarse[d];
      off[d] = r % (int)sh.fac[d];
      r /= (int)sh.fac[d];
    }
    int idx = 0;
    for (int d = 0; d < sh.rank; d++) idx = idx * (int)sh.fine[d] + cc[d] * (int)sh.fac[d] + off[d];
    tab[e] = idx;
  }
}

// eps_p = rel * ||y_p|| (pursuit.py:437), one warp per signal.
template <typename YT>
__global__ void row_tol_kernel(const YT *__restrict__ ys, int64_t p, int64_t n, double rel,
                               double *__restrict__ eps) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= p) return;
  double acc = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    const double v = (double)ys[w * n + i];
    acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) eps[w] = rel * sqrt(acc);
}

// blocks[p, :nb] = sort(low_sel[p, :nb]) (crossscale.py:268), thread per signal.
__global__ void sort_blocks_kernel(const int64_t *__restrict__ sel, const int64_t *__restrict__ cnt,
                                   int64_t p, int64_t k1, int64_t *__restrict__ blocks) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p) return;
  const int64_t nb = cnt[s];
  const int64_t *in = sel + s * k1;
  int64_t *out = blocks + s * k1;
  for (int64_t i = 0; i < nb; i++) {
    const int64_t v = in[i];
    int64_t j = i;
    while (j > 0 && out[j - 1] > v) {
      out[j] = out[j - 1];
      j--;
    }
    out[j] = v;
  }
  for (int64_t i = nb; i < k1; i++) out[i] = 0;
}

// Warp per signal (k1 <= 64): the coarse support ids are distinct, so each
// value's output slot is its rank (the count of smaller ids), found against
// all nb values broadcast by shuffles; the row is read and written coalesced
// (the thread-per-signal insertion sort above walks global memory k1^2 / 2
// times).
__global__ void __launch_bounds__(256) sort_blocks_warp_kernel(const int64_t *__restrict__ sel,
                                                               const int64_t *__restrict__ cnt,
                                                               int64_t p, int64_t k1,
                                                               int64_t *__restrict__ blocks) {
  const int lane = threadIdx.x & 31;
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= p) return;
  const int nb = (int)cnt[s];
  const int64_t *in = sel + s * k1;
  int64_t *out = blocks + s * k1;
  const int64_t v0 = lane < nb ? in[lane] : INT64_MAX, v1 = lane + 32 < nb ? in[lane + 32] : INT64_MAX;
  int r0 = 0, r1 = 0;
  for (int q = 0; q < nb && q < 32; q++) {
    const int64_t u = __shfl_sync(CDB_FULL_MASK, v0, q);
    r0 += u < v0;
    r1 += u < v1;
  }
  for (int q = 32; q < nb; q++) {
    const int64_t u = __shfl_sync(CDB_FULL_MASK, v1, q - 32);
    r0 += u < v0;
    r1 += u < v1;
  }
  if (lane < nb) out[r0] = v0;
  if (lane + 32 < nb) out[r1] = v1;
  for (int i = nb + lane; i < k1; i += 32) out[i] = 0;
}

// G = D D^T in fp64 (T x T), 64x64 tiles, 16x16 threads with 4x4 outputs.
__global__ void __launch_bounds__(256) gram_matrix_kernel(const double *__restrict__ d,
                                                          int64_t t, int64_t n,
                                                          double *__restrict__ g) {
  __shared__ double sa[16][65];
  __shared__ double sb[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < n; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int row = i / 16, kk = i % 16;
      const int64_t ra = r0 + row, rb = c0 + row, k = k0 + kk;
      sa[kk][row] = (ra < t && k < n) ? d[ra * n + k] : 0.0;
      sb[kk][row] = (rb < t && k < n) ? d[rb * n + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; kk++) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        av[i] = sa[kk][ty * 4 + i];
        bv[i] = sb[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int64_t r = r0 + ty * 4 + i, c = c0 + tx * 4 + j;
      if (r < t && c < t) g[r * t + c] = acc[i][j];
    }
}

// Tensor-core operand of the dictionary: fp16(scale * d), scale a power of
// two that puts the largest atom norm near 2^8 (fp16 carries 11 significand
// bits against bf16's 8, so the certified scan's window is ~8x narrower; the
// scale keeps every element far from both ends of the fp16 range).
__global__ void to_f16_kernel(const double *__restrict__ d, int64_t t, int64_t n, int64_t n_pad,
                              double scale, __half *__restrict__ out) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= t * n_pad) return;
  const int64_t row = gid / n_pad, col = gid % n_pad;
  out[gid] = __float2half_rn(col < n ? (float)(d[row * n + col] * scale) : 0.0f);
}

__global__ void to_f32_kernel(const double *__restrict__ d, int64_t count, float *__restrict__ out) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid < count) out[gid] = (float)d[gid];
}

__global__ void collect_delegates_kernel(const uint32_t *__restrict__ status, int64_t p,
                                         int64_t *__restrict__ ids, int *__restrict__ count) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p) return;
  if (status[s] & ST_DELEGATE) ids[atomicAdd(count, 1)] = s;
}

__global__ void row_norm_max_kernel(const double *__restrict__ d, int64_t t, int64_t n,
                                    unsigned long long *__restrict__ out) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= t) return;
  double acc = 0.0;
  for (int64_t i = lane; i < n; i += 32) acc = fma(d[w * n + i], d[w * n + i], acc);
  acc = warp_sum(acc);
  if (lane == 0) atomicMax(out, (unsigned long long)__double_as_longlong(sqrt(acc)));
}

// max over atoms of |fp16(scale d_j) / scale - d_j| (the tensor engine's
// operand rounding, measured exactly; the certification bound charges it
// instead of u |d|)
__global__ void quant_err_max_kernel(const double *__restrict__ d, const __half *__restrict__ d16,
                                     int64_t t, int64_t n, int64_t n_pad, double inv_scale,
                                     unsigned long long *__restrict__ out) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= t) return;
  double acc = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    const double e = (double)__half2float(d16[w * n_pad + i]) * inv_scale - d[w * n + i];
    acc = fma(e, e, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0)
    atomicMax(out, (unsigned long long)__double_as_longlong(sqrt(acc) * (1.0 + 1e-12)));
}

// ---- zero-tree step-2 routing: (signal, slot) pairs grouped by parent block
// Buckets are (signal block, parent): signals [sb*SB, (sb+1)*SB) x the T_low
// parents, so the alpha0 kernels sweep one L2-sized block of signal rows at a
// time (bucket = sb * t_low + parent).
__global__ void route_count_kernel(const int64_t *__restrict__ blocks, const int64_t *__restrict__ nb,
                                   int64_t p, int64_t k1, int64_t t_low, int64_t sbs,
                                   int *__restrict__ count) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p) return;
  const int64_t off = (s / sbs) * t_low;
  for (int64_t b = 0; b < nb[s]; b++) atomicAdd(&count[off + blocks[s * k1 + b]], 1);
}

// exclusive scan of count[0..m) into offs[0..m] and cursor copy (one CTA)
__global__ void route_scan_kernel(const int *__restrict__ count, int64_t m,
                                  int64_t *__restrict__ offs, int64_t *__restrict__ cursor) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (m + blockDim.x - 1) / blockDim.x;
  int64_t sum = 0;
  for (int64_t i = tid * per; i < (tid + 1) * per && i < m; i++) sum += count[i];
  part[tid] = sum;
  __syncthreads();
  if (tid == 0) {
    int64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; i++) {
      const int64_t v = part[i];
      part[i] = run;
      run += v;
    }
    offs[m] = run;
  }
  __syncthreads();
  int64_t run = part[tid];
  for (int64_t i = tid * per; i < (tid + 1) * per && i < m; i++) {
    offs[i] = run;
    cursor[i] = run;
    run += count[i];
  }
}

__global__ void route_fill_kernel(const int64_t *__restrict__ blocks, const int64_t *__restrict__ nb,
                                  int64_t p, int64_t k1, int64_t t_low, int64_t sbs,
                                  unsigned long long *__restrict__ cursor,
                                  int64_t *__restrict__ pairs) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p) return;
  const int64_t off = (s / sbs) * t_low;
  for (int64_t b = 0; b < nb[s]; b++) {
    const int64_t pos = (int64_t)atomicAdd(&cursor[off + blocks[s * k1 + b]], 1ull);
    pairs[pos] = (s << 16) | b;  // (signal, slot) pair
  }
}

// alpha0[s][b*Q + c] = <d_{parent*Q + c}, y_s> for every routed pair: one CTA
// per parent keeps its Q children in shared memory (fp64); each thread codes
// two routed signals against them (the child values are warp-broadcast
// shared-memory reads, each used for two FMAs; no cross-lane reductions).
template <typename YT, int QT>
__global__ void __launch_bounds__(256) alpha0_routed_kernel(
    const double *__restrict__ d64, int n, const YT *__restrict__ ys,
    const int64_t *__restrict__ offs, const int64_t *__restrict__ pairs, int64_t k1,
    int64_t smax, int64_t t_low, double *__restrict__ alpha0) {
  extern __shared__ double child[];  // QT x n
  const int64_t bucket = blockIdx.x, parent = bucket % t_low;
  const int64_t lo = offs[bucket], hi = offs[bucket + 1];
  if (lo == hi) return;
  for (int e = threadIdx.x; e < QT * n; e += blockDim.x) child[e] = d64[parent * QT * n + e];
  __syncthreads();
  for (int64_t e0 = lo + 2 * threadIdx.x; e0 < hi; e0 += 2 * blockDim.x) {
    const bool two = e0 + 1 < hi;
    const int64_t pr0 = pairs[e0], pr1 = two ? pairs[e0 + 1] : pr0;
    const YT *y0 = ys + (pr0 >> 16) * n;
    const YT *y1 = ys + (pr1 >> 16) * n;
    double a0[QT], a1[QT];
#pragma unroll
    for (int c = 0; c < QT; c++) {
      a0[c] = 0.0;
      a1[c] = 0.0;
    }
    int i = 0;
    if constexpr (sizeof(YT) == 4) {
      if ((n & 3) == 0) {  // 16-byte loads of both rows
        const float4 *q0 = reinterpret_cast<const float4 *>(y0);
        const float4 *q1 = reinterpret_cast<const float4 *>(y1);
#pragma unroll 2
        for (; i < n; i += 4) {
          const float4 f0 = q0[i >> 2], f1 = q1[i >> 2];
          const double u0[4] = {f0.x, f0.y, f0.z, f0.w}, u1[4] = {f1.x, f1.y, f1.z, f1.w};
#pragma unroll
          for (int t4 = 0; t4 < 4; t4++)
#pragma unroll
            for (int c = 0; c < QT; c++) {
              const double dv = child[c * n + i + t4];
              a0[c] = fma(dv, u0[t4], a0[c]);
              a1[c] = fma(dv, u1[t4], a1[c]);
            }
        }
      }
    }
#pragma unroll 4
    for (; i < n; i++) {
      const double v0 = (double)y0[i], v1 = (double)y1[i];
#pragma unroll
      for (int c = 0; c < QT; c++) {
        const double dv = child[c * n + i];
        a0[c] = fma(dv, v0, a0[c]);
        a1[c] = fma(dv, v1, a1[c]);
      }
    }
    double *o0 = alpha0 + (pr0 >> 16) * smax + (pr0 & 0xffff) * QT;
#pragma unroll
    for (int c = 0; c < QT; c++) o0[c] = a0[c];
    if (two) {
      double *o1 = alpha0 + (pr1 >> 16) * smax + (pr1 & 0xffff) * QT;
#pragma unroll
      for (int c = 0; c < QT; c++) o1[c] = a1[c];
    }
  }
}

// Shared-memory aggregated routing: a CTA histograms its chunk of signals'
// (signal, parent) pairs in shared memory and touches each global counter
// once per parent it saw (instead of once per pair).
constexpr int kRouteChunk = 1024;  // signals per CTA
}  // namespace
int64_t route_block_signals(int64_t p, int64_t n, bool ys_f32);
namespace {

__global__ void __launch_bounds__(256) route_count_smem_kernel(
    const int64_t *__restrict__ blocks, const int64_t *__restrict__ nb, int64_t p, int64_t k1,
    int t_low, int64_t sbs, int *__restrict__ count) {
  extern __shared__ int hist[];
  for (int b = threadIdx.x; b < t_low; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int64_t s0 = (int64_t)blockIdx.x * kRouteChunk;
  const int64_t s1 = s0 + kRouteChunk < p ? s0 + kRouteChunk : p;
  for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x)
    for (int64_t b = 0; b < nb[s]; b++) atomicAdd(&hist[blocks[s * k1 + b]], 1);
  __syncthreads();
  const int64_t off = (s0 / sbs) * t_low;  // the chunk lies in one signal block
  for (int b = threadIdx.x; b < t_low; b += blockDim.x)
    if (hist[b]) atomicAdd(&count[off + b], hist[b]);
}

__global__ void __launch_bounds__(256) route_fill_smem_kernel(
    const int64_t *__restrict__ blocks, const int64_t *__restrict__ nb, int64_t p, int64_t k1,
    int t_low, int64_t sbs, unsigned long long *__restrict__ cursor, int64_t *__restrict__ pairs) {
  extern __shared__ unsigned long long sh[];  // base[t_low] | hist[t_low] (as int)
  unsigned long long *base = sh;
  int *hist = (int *)(sh + t_low);
  for (int b = threadIdx.x; b < t_low; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int64_t s0 = (int64_t)blockIdx.x * kRouteChunk;
  const int64_t s1 = s0 + kRouteChunk < p ? s0 + kRouteChunk : p;
  for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x)
    for (int64_t b = 0; b < nb[s]; b++) atomicAdd(&hist[blocks[s * k1 + b]], 1);
  __syncthreads();
  const int64_t off = (s0 / sbs) * t_low;
  for (int b = threadIdx.x; b < t_low; b += blockDim.x) {
    base[b] = hist[b] ? atomicAdd(&cursor[off + b], (unsigned long long)hist[b]) : 0ull;
    hist[b] = 0;
  }
  __syncthreads();
  for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x)
    for (int64_t b = 0; b < nb[s]; b++) {
      const int64_t blk = blocks[s * k1 + b];
      pairs[base[blk] + atomicAdd(&hist[blk], 1)] = (s << 16) | b;
    }
}

// Warp per routed pair, the parent's QT children held in registers: lane
// owns the NPL = N/32 coordinates {VW*lane + 32*VW*v + e}, so each signal row
// is read with coalesced VW-wide loads; QT*NPL fp64 FMAs per lane, then a
// reduce-scatter butterfly leaves child c's sum in lanes with the matching
// bits.  A CTA covers 1/split of one parent's pairs.
template <int QT>
__device__ __forceinline__ double reduce_scatter(double (&v)[QT], int lane, int &child) {
  child = 0;
  int o = 16;
#pragma unroll
  for (int h = QT / 2; h >= 1; h >>= 1, o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; i++) {
      const double send = upper ? v[i] : v[i + h];
      const double keep = upper ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(CDB_FULL_MASK, send, o);
    }
    if (upper) child += h;
  }
  double r = v[0];
  for (; o >= 1; o >>= 1) r += __shfl_xor_sync(CDB_FULL_MASK, r, o);
  return r;
}

// HV: the parent's children are split over HV warps (QT / HV each), which
// halves the per-lane registers for QT >= 4 so more warps stay resident; a
// signal row is then read by HV warps (L1/L2 hits after the first).
template <typename YT, int QT, int NPL, int HV>
__global__ void __launch_bounds__(128) alpha0_warp_kernel(
    const double *__restrict__ d64, int n, const YT *__restrict__ ys,
    const int64_t *__restrict__ offs, const int64_t *__restrict__ pairs, int64_t k1,
    int64_t smax, int split, int t_low, double *__restrict__ alpha0) {
  constexpr int VW = NPL < 4 ? NPL : 4;  // floats per vector load
  constexpr int NV = NPL / VW;
  const int bucket = blockIdx.x / split, part = blockIdx.x % split;
  const int parent = bucket % t_low;
  const int64_t lo = offs[bucket], cnt = offs[bucket + 1] - lo;
  const int64_t a = lo + cnt * part / split, b = lo + cnt * (part + 1) / split;
  if (a >= b) return;
  constexpr int CH = QT / HV;  // children per warp
  const int lane = threadIdx.x & 31, w0 = threadIdx.x >> 5;
  const int half = w0 % HV, warp = w0 / HV, nwarps = (blockDim.x >> 5) / HV;
  double ch[CH][NPL];
#pragma unroll
  for (int c = 0; c < CH; c++)
#pragma unroll
    for (int v = 0; v < NV; v++)
#pragma unroll
      for (int e = 0; e < VW; e++)
        ch[c][v * VW + e] = __ldg(d64 + ((int64_t)parent * QT + half * CH + c) * n + VW * lane +
                                  32 * VW * v + e);
  // warp w takes the contiguous pairs [wa, wb); pair ids arrive 32 at a time
  // (one coalesced load, then shuffles) and the signal rows of the next two
  // pairs are loaded while the current two are coded
  const int64_t per = (b - a + nwarps - 1) / nwarps;
  const int64_t wa = a + warp * per, wb = wa + per < b ? wa + per : b;
  // signal values are staged in the input type: fp32 rows stay fp32 (exact),
  // fp64 rows are never rounded
  auto load_row = [&](int64_t pr, YT (&yv)[NPL]) {
    const YT *y = ys + (pr >> 16) * n;
#pragma unroll
    for (int v = 0; v < NV; v++) {
      const int i = VW * lane + 32 * VW * v;
      if constexpr (sizeof(YT) == 4 && VW == 4) {
        const float4 f = *reinterpret_cast<const float4 *>(y + i);
        yv[v * 4 + 0] = f.x;
        yv[v * 4 + 1] = f.y;
        yv[v * 4 + 2] = f.z;
        yv[v * 4 + 3] = f.w;
      } else if constexpr (sizeof(YT) == 4 && VW == 2) {
        const float2 f = *reinterpret_cast<const float2 *>(y + i);
        yv[v * 2 + 0] = f.x;
        yv[v * 2 + 1] = f.y;
      } else {
#pragma unroll
        for (int e = 0; e < VW; e++) yv[v * VW + e] = y[i + e];
      }
    }
  };
  // code two pairs at once: 2 CH independent accumulation chains
  auto code2 = [&](int64_t pra, const YT (&ya)[NPL], int64_t prb, const YT (&yb)[NPL],
                   bool second) {
    double acc[2 * CH];
#pragma unroll
    for (int c = 0; c < 2 * CH; c++) acc[c] = 0.0;
#pragma unroll
    for (int t = 0; t < NPL; t++) {
      const double va = (double)ya[t], vb = (double)yb[t];
#pragma unroll
      for (int c = 0; c < CH; c++) {
        acc[c] = fma(ch[c][t], va, acc[c]);
        acc[CH + c] = fma(ch[c][t], vb, acc[CH + c]);
      }
    }
    // reduce-scatter of both (2 CH values: pair index is the top level)
    int child;
    const double r = reduce_scatter<2 * CH>(acc, lane, child);
    const int pi = child / CH;  // 0: pair a, 1: pair b
    const int c = half * CH + child % CH;
    const int64_t pr = pi ? prb : pra;
    if ((lane & (32 / (2 * CH) - 1)) == 0 && (pi == 0 || second))
      alpha0[(pr >> 16) * smax + (pr & 0xffff) * QT + c] = r;
  };
  for (int64_t e0 = wa; e0 < wb; e0 += 32) {
    const int m = wb - e0 < 32 ? (int)(wb - e0) : 32;
    const int64_t mine = lane < m ? pairs[e0 + lane] : 0;
    YT ya[NPL], yb[NPL];
    int64_t pa = __shfl_sync(CDB_FULL_MASK, (long long)mine, 0);
    int64_t pb = __shfl_sync(CDB_FULL_MASK, (long long)mine, 1 < m ? 1 : 0);
    load_row(pa, ya);
    load_row(pb, yb);
    for (int j = 0; j < m; j += 2) {
      YT ca[NPL], cb[NPL];
#pragma unroll
      for (int t = 0; t < NPL; t++) {
        ca[t] = ya[t];
        cb[t] = yb[t];
      }
      const int64_t qa = pa, qb = pb;
      if (j + 2 < m) {
        pa = __shfl_sync(CDB_FULL_MASK, (long long)mine, j + 2);
        pb = __shfl_sync(CDB_FULL_MASK, (long long)mine, j + 3 < m ? j + 3 : j + 2);
        load_row(pa, ya);
        load_row(pb, yb);
      }
      code2(qa, ca, qb, cb, j + 1 < m);
    }
  }
}

template <typename YT, int QT, int NPL>
cudaError_t launch_alpha0_warp(const double *d64, int64_t t_low, int64_t buckets, int64_t n,
                               const YT *ys, const int64_t *offs, const int64_t *pairs,
                               int64_t k1, int64_t smax, double *alpha0, cudaStream_t stream) {
  const int split = 8;
  constexpr int HV = 1;  // splitting children over 2 warps measured slower (0.76 vs 0.63 ms, cfg 1)
  alpha0_warp_kernel<YT, QT, NPL, HV><<<(unsigned)(buckets * split), 128, 0, stream>>>(
      d64, (int)n, ys, offs, pairs, k1, smax, split, (int)t_low, alpha0);
  return cudaGetLastError();
}

// Q = 8 on the fp64 tensor cores: a warp codes 8 pairs at once as one 8x8
// tile C[child][pair] = sum_k D[child][k] y_pair[k] of m8n8k4 DMMA steps.
// Lane (r = lane>>2, j = lane&3) supplies A[r][j] = child r and B[j][r] =
// pair r at coordinate 16 t + 4 j + e of step 4 t + e -- the same k
// permutation on both sides -- so each pair row is read with one 16-B load
// per 16 coordinates and no cross-lane reduction is needed.
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Pull the next tile's pair rows into L1 while the current tile is coded
// (the rows are L2-resident; this hides the L2 latency of the next tile).
// Used by the register-children kernel (cfg 1: 0.451 -> 0.423 ms); the L1
// kernel measured slower with it (its children compete for L1).
template <typename YT>
__device__ __forceinline__ void prefetch_tile(const int64_t *__restrict__ pairs,
                                              const YT *__restrict__ ys, int n, int64_t e1,
                                              int64_t wb, int r, int j, int len) {
  if (e1 >= wb) return;
  const int mn = wb - e1 < 8 ? (int)(wb - e1) : 8;
  const int64_t pn = pairs[e1 + (r < mn ? r : mn - 1)];
  const char *row = reinterpret_cast<const char *>(ys + (pn >> 16) * n);
  const int bytes = len * (int)sizeof(YT);
  for (int o = j * 128; o < bytes; o += 4 * 128)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(row + o));
}

template <typename YT, int NT, int QT = 8>  // NT = N / 16; QT = 4: rows 4-7 of A are zero
__global__ void __launch_bounds__(128) alpha0_mma_kernel(
    const double *__restrict__ d64, int n, const YT *__restrict__ ys,
    const int64_t *__restrict__ offs, const int64_t *__restrict__ pairs, int64_t smax, int split,
    int t_low, double *__restrict__ alpha0, int pf) {
  const int bucket = blockIdx.x / split, part = blockIdx.x % split;
  const int parent = bucket % t_low;
  const int64_t lo = offs[bucket], cnt = offs[bucket + 1] - lo;
  const int64_t a = lo + cnt * part / split, b = lo + cnt * (part + 1) / split;
  if (a >= b) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int r = lane >> 2, j = lane & 3;
  double ch[4 * NT];
  {
    const double *src = d64 + ((int64_t)parent * QT + (r < QT ? r : 0)) * n + 4 * j;
#pragma unroll
    for (int t = 0; t < NT; t++) {
      const double2 u = __ldg(reinterpret_cast<const double2 *>(src + 16 * t));
      const double2 v = __ldg(reinterpret_cast<const double2 *>(src + 16 * t + 2));
      const bool live = r < QT;
      ch[4 * t + 0] = live ? u.x : 0.0;
      ch[4 * t + 1] = live ? u.y : 0.0;
      ch[4 * t + 2] = live ? v.x : 0.0;
      ch[4 * t + 3] = live ? v.y : 0.0;
    }
  }
  // warp w takes a contiguous run of whole 8-pair tiles
  const int64_t per = ((b - a + 8 * nwarps - 1) / (8 * nwarps)) * 8;
  const int64_t wa = a + warp * per, wb = wa + per < b ? wa + per : b;
  for (int64_t e0 = wa; e0 < wb; e0 += 8) {
    const int m = wb - e0 < 8 ? (int)(wb - e0) : 8;
    const int64_t pr = pairs[e0 + (r < m ? r : m - 1)];
    const YT *y = ys + (pr >> 16) * n + 4 * j;
    if (pf) prefetch_tile(pairs, ys, n, e0 + 8, wb, r, j, 16 * NT);
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int t = 0; t < NT; t++) {
      double yv[4];
      if constexpr (sizeof(YT) == 4) {
        const float4 f = *reinterpret_cast<const float4 *>(y + 16 * t);
        yv[0] = f.x;
        yv[1] = f.y;
        yv[2] = f.z;
        yv[3] = f.w;
      } else {
        const double2 u = *reinterpret_cast<const double2 *>(y + 16 * t);
        const double2 v = *reinterpret_cast<const double2 *>(y + 16 * t + 2);
        yv[0] = u.x;
        yv[1] = u.y;
        yv[2] = v.x;
        yv[3] = v.y;
      }
#pragma unroll
      for (int e = 0; e < 4; e++) dmma_8x8x4(c0, c1, ch[4 * t + e], yv[e]);
    }
    // lane holds child r of pairs 2j and 2j + 1 (pair q's id sits in lane 4q)
    const int64_t p0 = __shfl_sync(CDB_FULL_MASK, (long long)pr, 8 * j);
    const int64_t p1 = __shfl_sync(CDB_FULL_MASK, (long long)pr, 8 * j + 4);
    if (r < QT && 2 * j < m) alpha0[(p0 >> 16) * smax + (p0 & 0xffff) * QT + r] = c0;
    if (r < QT && 2 * j + 1 < m) alpha0[(p1 >> 16) * smax + (p1 & 0xffff) * QT + r] = c1;
  }
}

// The same tiles for any N (a multiple of 16) and Q = 8 CT: the children
// are read per step from L1 (a bucket's CTAs share one parent, Q N fp64),
// each 16-B pair load feeding CT child tiles.
template <typename YT, int CT>
__global__ void __launch_bounds__(128) alpha0_mma_l1_kernel(
    const double *__restrict__ d64, int n, const YT *__restrict__ ys,
    const int64_t *__restrict__ offs, const int64_t *__restrict__ pairs, int64_t smax, int split,
    int t_low, double *__restrict__ alpha0, int pf) {
  constexpr int QT = 8 * CT;
  const int bucket = blockIdx.x / split, part = blockIdx.x % split;
  const int parent = bucket % t_low;
  const int64_t lo = offs[bucket], cnt = offs[bucket + 1] - lo;
  const int64_t a = lo + cnt * part / split, b = lo + cnt * (part + 1) / split;
  if (a >= b) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int r = lane >> 2, j = lane & 3, nt = n >> 4;
  const double *dc = d64 + ((int64_t)parent * QT + r) * n + 4 * j;
  const int64_t per = ((b - a + 8 * nwarps - 1) / (8 * nwarps)) * 8;
  const int64_t wa = a + warp * per, wb = wa + per < b ? wa + per : b;
  for (int64_t e0 = wa; e0 < wb; e0 += 8) {
    const int m = wb - e0 < 8 ? (int)(wb - e0) : 8;
    const int64_t pr = pairs[e0 + (r < m ? r : m - 1)];
    const YT *y = ys + (pr >> 16) * n + 4 * j;
    if (pf) prefetch_tile(pairs, ys, n, e0 + 8, wb, r, j, n);
    double c[CT][2];
#pragma unroll
    for (int ct = 0; ct < CT; ct++) c[ct][0] = c[ct][1] = 0.0;
#pragma unroll 8
    for (int t = 0; t < nt; t++) {
      double yv[4];
      if constexpr (sizeof(YT) == 4) {
        const float4 f = *reinterpret_cast<const float4 *>(y + 16 * t);
        yv[0] = f.x;
        yv[1] = f.y;
        yv[2] = f.z;
        yv[3] = f.w;
      } else {
        const double2 u = *reinterpret_cast<const double2 *>(y + 16 * t);
        const double2 v = *reinterpret_cast<const double2 *>(y + 16 * t + 2);
        yv[0] = u.x;
        yv[1] = u.y;
        yv[2] = v.x;
        yv[3] = v.y;
      }
#pragma unroll
      for (int ct = 0; ct < CT; ct++) {
        const double2 u = __ldg(reinterpret_cast<const double2 *>(dc + (int64_t)ct * 8 * n + 16 * t));
        const double2 v =
            __ldg(reinterpret_cast<const double2 *>(dc + (int64_t)ct * 8 * n + 16 * t + 2));
        dmma_8x8x4(c[ct][0], c[ct][1], u.x, yv[0]);
        dmma_8x8x4(c[ct][0], c[ct][1], u.y, yv[1]);
        dmma_8x8x4(c[ct][0], c[ct][1], v.x, yv[2]);
        dmma_8x8x4(c[ct][0], c[ct][1], v.y, yv[3]);
      }
    }
    const int64_t p0 = __shfl_sync(CDB_FULL_MASK, (long long)pr, 8 * j);
    const int64_t p1 = __shfl_sync(CDB_FULL_MASK, (long long)pr, 8 * j + 4);
#pragma unroll
    for (int ct = 0; ct < CT; ct++) {
      if (2 * j < m) alpha0[(p0 >> 16) * smax + (p0 & 0xffff) * QT + ct * 8 + r] = c[ct][0];
      if (2 * j + 1 < m) alpha0[(p1 >> 16) * smax + (p1 & 0xffff) * QT + ct * 8 + r] = c[ct][1];
    }
  }
}

// Q = 8, any N (a multiple of 16), pairs blocked PT tiles deep: a warp codes
// 8 PT pairs of one parent per pass, so each children fragment (2 x 16 B per
// lane per 16 coordinates, an L2 read: the parent's 8 children are 8 N fp64,
// 256 KB at N = 4096, more than L1 holds) feeds PT tiles instead of one --
// the children stream per pair drops PT-fold.  A pair's DMMA sequence (and
// so its value) is the one of alpha0_mma_l1_kernel: bit-identical.  Warps of
// the CTA take the part's super-tiles round-robin.
template <typename YT, int PT>
__global__ void __launch_bounds__(128) alpha0_mma_pt_kernel(
    const double *__restrict__ d64, int n, const YT *__restrict__ ys,
    const int64_t *__restrict__ offs, const int64_t *__restrict__ pairs, int64_t smax, int split,
    int t_low, double *__restrict__ alpha0) {
  const int bucket = blockIdx.x / split, part = blockIdx.x % split;
  const int parent = bucket % t_low;
  const int64_t lo = offs[bucket], cnt = offs[bucket + 1] - lo;
  const int64_t a = lo + cnt * part / split, b = lo + cnt * (part + 1) / split;
  if (a >= b) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int r = lane >> 2, j = lane & 3, nt = n >> 4;
  const double *dc = d64 + ((int64_t)parent * 8 + r) * n + 4 * j;
  for (int64_t e0 = a + (int64_t)warp * 8 * PT; e0 < b; e0 += (int64_t)nwarps * 8 * PT) {
    int64_t pr[PT];
    const YT *y[PT];
#pragma unroll
    for (int pt = 0; pt < PT; pt++) {
      const int64_t e = e0 + pt * 8 + r;
      pr[pt] = pairs[e < b ? e : b - 1];
      y[pt] = ys + (pr[pt] >> 16) * n + 4 * j;
    }
    double c[PT][2];
#pragma unroll
    for (int pt = 0; pt < PT; pt++) c[pt][0] = c[pt][1] = 0.0;
#pragma unroll 4
    for (int t = 0; t < nt; t++) {
      const double2 u = __ldg(reinterpret_cast<const double2 *>(dc + 16 * t));
      const double2 v = __ldg(reinterpret_cast<const double2 *>(dc + 16 * t + 2));
#pragma unroll
      for (int pt = 0; pt < PT; pt++) {
        double yv[4];
        if constexpr (sizeof(YT) == 4) {
          const float4 f = *reinterpret_cast<const float4 *>(y[pt] + 16 * t);
          yv[0] = f.x;
          yv[1] = f.y;
          yv[2] = f.z;
          yv[3] = f.w;
        } else {
          const double2 p = *reinterpret_cast<const double2 *>(y[pt] + 16 * t);
          const double2 q = *reinterpret_cast<const double2 *>(y[pt] + 16 * t + 2);
          yv[0] = p.x;
          yv[1] = p.y;
          yv[2] = q.x;
          yv[3] = q.y;
        }
        dmma_8x8x4(c[pt][0], c[pt][1], u.x, yv[0]);
        dmma_8x8x4(c[pt][0], c[pt][1], u.y, yv[1]);
        dmma_8x8x4(c[pt][0], c[pt][1], v.x, yv[2]);
        dmma_8x8x4(c[pt][0], c[pt][1], v.y, yv[3]);
      }
    }
#pragma unroll
    for (int pt = 0; pt < PT; pt++) {
      const int64_t base = e0 + pt * 8;
      const int64_t p0 = __shfl_sync(CDB_FULL_MASK, (long long)pr[pt], 8 * j);
      const int64_t p1 = __shfl_sync(CDB_FULL_MASK, (long long)pr[pt], 8 * j + 4);
      if (base + 2 * j < b) alpha0[(p0 >> 16) * smax + (p0 & 0xffff) * 8 + r] = c[pt][0];
      if (base + 2 * j + 1 < b) alpha0[(p1 >> 16) * smax + (p1 & 0xffff) * 8 + r] = c[pt][1];
    }
  }
}

// configs[4] (131k signals, alpha0 per call): PT 1 / split 8 (the l1 kernel)
// 30.1 ms; PT 2 / 3 / 4 at split 1: 25.7 / 20.2 / 21.6 ms; PT 3 at split 2:
// 20.5 ms; larger routing blocks (6144 signals) no better with PT 3.
int alpha0_pt() {  // CDB_A0_PT: pair tiles per pass for Q = 8, N > 256 (1 = alpha0_mma_l1_kernel)
  const char *e = getenv("CDB_A0_PT");
  return e ? atoi(e) : 3;
}
int alpha0_split() {  // CDB_A0_SPLIT: CTAs per (signal block, parent) bucket of the PT kernel
  const char *e = getenv("CDB_A0_SPLIT");
  return e ? std::max(1, atoi(e)) : 1;
}

// CDB_A0_MMA=0 keeps the FFMA warp kernel for Q = 8
bool alpha0_mma_enabled() {
  static const int on = [] {
    const char *v = getenv("CDB_A0_MMA");
    return v ? atoi(v) : 1;
  }();
  return on != 0;
}

// The register path when the parent's children fit 64 fp64 registers per
// lane and N is 64, 128 or 256 (else the shared-memory kernel above).
template <typename YT>
bool try_alpha0_warp(const double *d64, int64_t t_low, int64_t buckets, int64_t n, int64_t q,
                     const YT *ys, const int64_t *offs, const int64_t *pairs, int64_t k1,
                     int64_t smax, double *alpha0, cudaStream_t stream, cudaError_t &err) {
  static const int pf = [] {
    const char *v = getenv("CDB_A0_PF");
    return v ? atoi(v) : 1;
  }();
  if (q == 4 && (n == 64 || n == 128) && alpha0_mma_enabled()) {
    const int split = 8;
    const unsigned grid = (unsigned)(buckets * split);
    if (n == 64)
      alpha0_mma_kernel<YT, 4, 4><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                            split, (int)t_low, alpha0, pf);
    else
      alpha0_mma_kernel<YT, 8, 4><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                            split, (int)t_low, alpha0, pf);
    err = cudaGetLastError();
    return true;
  }
  if (q == 8 && (n == 64 || n == 128 || n == 256) && alpha0_mma_enabled()) {
    const int split = 8;
    const unsigned grid = (unsigned)(buckets * split);
    if (n == 64)
      alpha0_mma_kernel<YT, 4><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                         split, (int)t_low, alpha0, pf);
    else if (n == 128)
      alpha0_mma_kernel<YT, 8><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                         split, (int)t_low, alpha0, pf);
    else
      alpha0_mma_kernel<YT, 16><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                          split, (int)t_low, alpha0, pf);
    err = cudaGetLastError();
    return true;
  }
  if (q == 8 && n % 16 == 0 && alpha0_mma_enabled() && alpha0_pt() > 1) {
    const int split = alpha0_split();
    const unsigned grid = (unsigned)(buckets * split);
    switch (alpha0_pt()) {
      case 2:
        alpha0_mma_pt_kernel<YT, 2><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                              split, (int)t_low, alpha0);
        break;
      case 3:
        alpha0_mma_pt_kernel<YT, 3><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                              split, (int)t_low, alpha0);
        break;
      default:
        alpha0_mma_pt_kernel<YT, 4><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                              split, (int)t_low, alpha0);
    }
    err = cudaGetLastError();
    return true;
  }
  if ((q == 8 || q == 16) && n % 16 == 0 && alpha0_mma_enabled()) {
    const int split = 8;
    const unsigned grid = (unsigned)(buckets * split);
    if (q == 8)
      alpha0_mma_l1_kernel<YT, 1><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                            split, (int)t_low, alpha0, 0);
    else
      alpha0_mma_l1_kernel<YT, 2><<<grid, 128, 0, stream>>>(d64, (int)n, ys, offs, pairs, smax,
                                                            split, (int)t_low, alpha0, 0);
    err = cudaGetLastError();
    return true;
  }
#define CDB_A0W(QQ, NN)                                                                      \
  if (q == QQ && n == 32 * NN) {                                                             \
    err = launch_alpha0_warp<YT, QQ, NN>(d64, t_low, buckets, n, ys, offs, pairs, k1, smax,  \
                                         alpha0, stream);                                    \
    return true;                                                                             \
  }
  CDB_A0W(1, 2) CDB_A0W(2, 2) CDB_A0W(4, 2) CDB_A0W(8, 2) CDB_A0W(16, 2)
  CDB_A0W(1, 4) CDB_A0W(2, 4) CDB_A0W(4, 4) CDB_A0W(8, 4) CDB_A0W(16, 4)
  CDB_A0W(1, 8) CDB_A0W(2, 8) CDB_A0W(4, 8) CDB_A0W(8, 8)
#undef CDB_A0W
  return false;
}

template <typename YT, int QT>
cudaError_t launch_alpha0_q(const double *d64, int64_t t_low, int64_t buckets, int64_t n,
                            const YT *ys, const int64_t *offs, const int64_t *pairs, int64_t k1,
                            int64_t smax, double *alpha0, cudaStream_t stream) {
  const size_t smem = sizeof(double) * QT * n;
  cudaError_t e = cudaFuncSetAttribute(alpha0_routed_kernel<YT, QT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  alpha0_routed_kernel<YT, QT><<<(unsigned)buckets, 256, smem, stream>>>(
      d64, (int)n, ys, offs, pairs, k1, smax, t_low, alpha0);
  return cudaGetLastError();
}

template <typename YT>
cudaError_t launch_alpha0(const double *d64, int64_t t_low, int64_t buckets, int64_t n, int64_t q,
                          const YT *ys, const int64_t *offs, const int64_t *pairs, int64_t k1,
                          int64_t smax, double *alpha0, cudaStream_t stream) {
#define CDB_A0Q(QQ)                                                                            \
  case QQ:                                                                                     \
    return launch_alpha0_q<YT, QQ>(d64, t_low, buckets, n, ys, offs, pairs, k1, smax, alpha0,  \
                                   stream);
  switch (q) { CDB_A0Q(1) CDB_A0Q(2) CDB_A0Q(4) CDB_A0Q(8) CDB_A0Q(16) }
#undef CDB_A0Q
  return cudaErrorInvalidValue;
}

inline unsigned blocks_for(int64_t work, int threads) {
  return (unsigned)((work + threads - 1) / threads);
}

}  // namespace

cudaError_t launch_downsample(const void *ys, bool ys_f32, int64_t p, int64_t n,
                              const int64_t *fine_shape, const int64_t *factors, int rank,
                              double *y_low, int64_t n_low, cudaStream_t stream, double rel,
                              double *eps_low, double *eps_fine) {
  ProfScope _ps("downsample", stream);
  if (p <= 0) return cudaSuccess;
  if (rank < 1 || rank > 4) return cudaErrorInvalidValue;
  Shape4 sh{};
  sh.rank = rank;
  for (int d = 0; d < rank; d++) {
    sh.fine[d] = fine_shape[d];
    sh.fac[d] = factors[d];
    sh.coarse[d] = fine_shape[d] / factors[d];
  }
  int block = 1;
  for (int d = 0; d < rank; d++) block *= (int)factors[d];
  static const bool direct = !(getenv("CDB_DOWNSAMPLE_STAGED") && atoi(getenv("CDB_DOWNSAMPLE_STAGED")));
  if (direct && n_low * block <= 48 * 1024 / 4) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int *tab = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&tab, sizeof(int) * n_low * block, stream);
    if (e != cudaSuccess) return e;
    downsample_table_kernel<<<(unsigned)((n_low * block + 255) / 256), 256, 0, stream>>>(sh, (int)n_low, tab);
    const int spi = n_low < 256 ? (int)(256 / n_low) : 1;
    const int64_t groups = (p + spi - 1) / spi;
    const unsigned g = (unsigned)(groups < (int64_t)sms * 8 ? groups : (int64_t)sms * 8);
    const size_t smem = sizeof(int) * n_low * block;
    // fp32 rows with a last-axis factor of 2 (every BASELINE config): pair loads
    const bool pairs = ys_f32 && factors[rank - 1] == 2 && fine_shape[rank - 1] % 2 == 0;
    if (pairs)
      downsample_direct_kernel<float, 2><<<g, 256, smem, stream>>>(
          (const float *)ys, p, (int)n, (int)n_low, block, tab, y_low, rel, eps_low, eps_fine);
    else if (ys_f32)
      downsample_direct_kernel<float, 1><<<g, 256, smem, stream>>>(
          (const float *)ys, p, (int)n, (int)n_low, block, tab, y_low, rel, eps_low, eps_fine);
    else
      downsample_direct_kernel<double, 1><<<g, 256, smem, stream>>>(
          (const double *)ys, p, (int)n, (int)n_low, block, tab, y_low, rel, eps_low, eps_fine);
    note_launch();
    note_launch();
    e = cudaGetLastError();
    cudaFreeAsync(tab, stream);
    return e;
  }
  const int64_t esz = ys_f32 ? 4 : 8;
  int spb = (int)(32768 / (n * esz));
  if (spb < 1) spb = 1;
  const size_t smem = (size_t)(n * 4 + 15) / 16 * 16 + (size_t)spb * n * esz;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = (int)((200 * 1024) / (smem + 1024)) < 8 ? (int)((200 * 1024) / (smem + 1024)) : 8;
  const int64_t groups = (p + spb - 1) / spb;
  const unsigned g = (unsigned)(groups < (int64_t)sms * per_sm ? groups : (int64_t)sms * per_sm);
  cudaError_t e;
  if (ys_f32) {
    e = cudaFuncSetAttribute(downsample_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    downsample_kernel<float><<<g, 256, smem, stream>>>((const float *)ys, p, (int)n, sh, y_low,
                                                       (int)n_low, spb, rel, eps_low, eps_fine);
  } else {
    e = cudaFuncSetAttribute(downsample_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    downsample_kernel<double><<<g, 256, smem, stream>>>((const double *)ys, p, (int)n, sh, y_low,
                                                        (int)n_low, spb, rel, eps_low, eps_fine);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_row_tol(const void *ys, bool ys_f32, int64_t p, int64_t n, double rel,
                           double *eps, cudaStream_t stream) {
  ProfScope _ps("row_tol", stream);
  if (p <= 0) return cudaSuccess;
  const unsigned g = blocks_for(p * 32, 256);
  if (ys_f32)
    row_tol_kernel<float><<<g, 256, 0, stream>>>((const float *)ys, p, n, rel, eps);
  else
    row_tol_kernel<double><<<g, 256, 0, stream>>>((const double *)ys, p, n, rel, eps);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_sort_blocks(const int64_t *low_sel, const int64_t *low_count, int64_t p,
                               int64_t k1, int64_t *blocks, cudaStream_t stream) {
  ProfScope _ps("sort_blocks", stream);
  if (p <= 0) return cudaSuccess;
  if (k1 <= 64)
    sort_blocks_warp_kernel<<<(unsigned)((p * 32 + 255) / 256), 256, 0, stream>>>(low_sel, low_count,
                                                                                 p, k1, blocks);
  else
    sort_blocks_kernel<<<blocks_for(p, 128), 128, 0, stream>>>(low_sel, low_count, p, k1, blocks);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gram_matrix(const double *d64, int64_t t, int64_t n, double *gram,
                               cudaStream_t stream) {
  ProfScope _ps("gram_matrix", stream);
  dim3 grid((unsigned)((t + 63) / 64), (unsigned)((t + 63) / 64));
  gram_matrix_kernel<<<grid, 256, 0, stream>>>(d64, t, n, gram);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_to_f16(const double *d64, int64_t t, int64_t n, int64_t n_pad, double scale,
                          void *d16, cudaStream_t stream) {
  ProfScope _ps("to_f16", stream);
  to_f16_kernel<<<blocks_for(t * n_pad, 256), 256, 0, stream>>>(d64, t, n, n_pad, scale,
                                                                 (__half *)d16);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_to_f32(const double *d64, int64_t count, float *d32, cudaStream_t stream) {
  ProfScope _ps("to_f32", stream);
  to_f32_kernel<<<blocks_for(count, 256), 256, 0, stream>>>(d64, count, d32);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_collect_delegates(const uint32_t *status, int64_t p, int64_t *ids, int *count,
                                     cudaStream_t stream) {
  ProfScope _ps("collect_delegates", stream);
  if (p <= 0) return cudaSuccess;
  collect_delegates_kernel<<<blocks_for(p, 256), 256, 0, stream>>>(status, p, ids, count);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_row_norm_max(const double *d64, int64_t t, int64_t n, double *out,
                                cudaStream_t stream) {
  ProfScope _ps("row_norm_max", stream);
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), stream);
  if (e != cudaSuccess) return e;
  row_norm_max_kernel<<<blocks_for(t * 32, 256), 256, 0, stream>>>(d64, t, n,
                                                                     (unsigned long long *)out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_quant_err_max(const double *d64, const void *d16, int64_t t, int64_t n,
                                 int64_t n_pad, double scale, double *out, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), stream);
  if (e != cudaSuccess) return e;
  quant_err_max_kernel<<<blocks_for(t * 32, 256), 256, 0, stream>>>(
      d64, (const __half *)d16, t, n, n_pad, 1.0 / scale, (unsigned long long *)out);
  note_launch();
  return cudaGetLastError();
}

// the DMMA tiles take any N (a multiple of 16) for Q in {8, 16}: above the
// L1 size the children stream from L2, still 8 pairs per read
bool route_alpha0_dmma(int64_t q, int64_t n) {
  return (q == 8 || q == 16) && n % 16 == 0 && alpha0_mma_enabled();
}

cudaError_t launch_route_alpha0(const double *d64, int64_t t_low, int64_t n, int64_t q,
                               const void *ys, bool ys_f32, const int64_t *blocks,
                               const int64_t *nb, int64_t p, int64_t k1, int64_t smax,
                               double *alpha0, void *work, cudaStream_t stream) {
  ProfScope _ps("route_alpha0", stream);
  // buckets = (signal block, parent); work: count int[m] | offs int64[m+1] |
  // cursor u64[m] | pairs int64[p*k1], m = blocks * t_low
  const int64_t sbs = route_block_signals(p, n, ys_f32);
  const int64_t m = ((p + sbs - 1) / sbs) * t_low;
  uint8_t *w = (uint8_t *)work;
  int *count = (int *)w;
  w += ((m * 4 + 255) / 256) * 256;
  int64_t *offs = (int64_t *)w;
  w += (((m + 1) * 8 + 255) / 256) * 256;
  int64_t *cursor = (int64_t *)w;
  w += ((m * 8 + 255) / 256) * 256;
  int64_t *pairs = (int64_t *)w;
  cudaError_t e = cudaMemsetAsync(count, 0, m * 4, stream);
  if (e != cudaSuccess) return e;
  const bool smem_route = t_low * 12 <= 48 * 1024;
  const unsigned rgrid = (unsigned)((p + kRouteChunk - 1) / kRouteChunk);
  if (smem_route)
    route_count_smem_kernel<<<rgrid, 256, t_low * 4, stream>>>(blocks, nb, p, k1, (int)t_low, sbs,
                                                               count);
  else
    route_count_kernel<<<blocks_for(p, 256), 256, 0, stream>>>(blocks, nb, p, k1, t_low, sbs,
                                                               count);
  route_scan_kernel<<<1, 1024, 0, stream>>>(count, m, offs, cursor);
  if (smem_route)
    route_fill_smem_kernel<<<rgrid, 256, t_low * 12, stream>>>(
        blocks, nb, p, k1, (int)t_low, sbs, (unsigned long long *)cursor, pairs);
  else
    route_fill_kernel<<<blocks_for(p, 256), 256, 0, stream>>>(
        blocks, nb, p, k1, t_low, sbs, (unsigned long long *)cursor, pairs);
  bool done = ys_f32 ? try_alpha0_warp<float>(d64, t_low, m, n, q, (const float *)ys, offs, pairs,
                                              k1, smax, alpha0, stream, e)
                     : try_alpha0_warp<double>(d64, t_low, m, n, q, (const double *)ys, offs,
                                               pairs, k1, smax, alpha0, stream, e);
  if (!done)
    e = ys_f32 ? launch_alpha0<float>(d64, t_low, m, n, q, (const float *)ys, offs, pairs, k1,
                                      smax, alpha0, stream)
               : launch_alpha0<double>(d64, t_low, m, n, q, (const double *)ys, offs, pairs, k1,
                                       smax, alpha0, stream);
  if (e != cudaSuccess) return e;
  note_launch(4);
  return cudaGetLastError();
}

// Signals per routing block: ~48 MB of signal rows stay L2-resident while
// every parent of the block is coded (measured on cfg 1, 100k signals:
// 8 MB 0.79 ms, 16 MB 0.685, 32 MB 0.637, 40-64 MB 0.627-0.629, one block
// 0.68); a multiple of the 1024-signal routing chunk; CDB_ROUTE_SB overrides
// (0 = one block).
int64_t route_block_signals(int64_t p, int64_t n, bool ys_f32) {
  int64_t sbs = (int64_t(48) << 20) / ((ys_f32 ? 4 : 8) * (n > 0 ? n : 1));
  if (const char *v = getenv("CDB_ROUTE_SB")) sbs = atoll(v);
  if (sbs <= 0) return p > 0 ? ((p + kRouteChunk - 1) / kRouteChunk) * kRouteChunk : kRouteChunk;
  sbs = (sbs / kRouteChunk) * kRouteChunk;
  return sbs < kRouteChunk ? kRouteChunk : sbs;
}

int64_t route_work_bytes(int64_t t_low, int64_t p, int64_t k1, int64_t n, bool ys_f32) {
  const int64_t sbs = route_block_signals(p, n, ys_f32);
  const int64_t m = ((p + sbs - 1) / sbs) * t_low;
  return ((m * 4 + 255) / 256) * 256 + (((m + 1) * 8 + 255) / 256) * 256 +
         ((m * 8 + 255) / 256) * 256 + p * k1 * 8 + 256;
}

// ---------------------------------------------------------------- column batches
// rows[j][i] = cols[i][j]: an n x len column block (the reference's N x P
// batch layout, pursuit.py:433 transposes it on the host) into len x n rows.
// 32 x 32 tiles through shared memory (row stride 33: conflict-free column
// reads), 8 rows per thread; both sides touch whole 128-byte lines for fp32.
template <typename T>
__global__ void __launch_bounds__(256) cols_to_rows_kernel(const T *__restrict__ cols, int64_t n,
                                                           int64_t len, T *__restrict__ rows) {
  __shared__ T tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int64_t i = i0 + ty + r, j = j0 + tx;
    if (i < n && j < len) tile[ty + r][tx] = cols[i * len + j];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int64_t j = j0 + ty + r, i = i0 + tx;
    if (j < len && i < n) rows[j * n + i] = tile[tx][ty + r];
  }
}

cudaError_t launch_cols_to_rows(const void *cols, bool f32, int64_t n, int64_t len, void *rows,
                                cudaStream_t stream) {
  ProfScope _ps("cols_to_rows", stream);
  if (n <= 0 || len <= 0) return cudaSuccess;
  if ((n + 31) / 32 > 65535) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)((len + 31) / 32), (unsigned)((n + 31) / 32));
  if (f32)
    cols_to_rows_kernel<float><<<grid, 256, 0, stream>>>((const float *)cols, n, len, (float *)rows);
  else
    cols_to_rows_kernel<double><<<grid, 256, 0, stream>>>((const double *)cols, n, len,
                                                           (double *)rows);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cdb
