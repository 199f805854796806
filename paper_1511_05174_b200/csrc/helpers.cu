// Small memory-bound kernels around the OMP engines.
#include <cuda_bf16.h>

#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

struct Shape4 {
  int64_t fine[4], fac[4], coarse[4];
  int rank;
};

// Block mean of row-major fine patches (crossdict/scaling.py:99-116,
// downsample_columns), one thread per (signal, coarse cell).
template <typename YT>
__global__ void downsample_kernel(const YT *__restrict__ ys, int64_t p, int64_t n, Shape4 sh,
                                  double *__restrict__ out, int64_t n_low) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= p * n_low) return;
  const int64_t sig = gid / n_low, cell = gid % n_low;
  int64_t cc[4] = {0, 0, 0, 0};
  int64_t rem = cell;
  for (int d = sh.rank - 1; d >= 0; d--) {
    cc[d] = rem % sh.coarse[d];
    rem /= sh.coarse[d];
  }
  int64_t block = 1;
  for (int d = 0; d < sh.rank; d++) block *= sh.fac[d];
  double acc = 0.0;
  for (int64_t b = 0; b < block; b++) {
    int64_t off[4] = {0, 0, 0, 0};
    int64_t r = b;
    for (int d = sh.rank - 1; d >= 0; d--) {
      off[d] = r % sh.fac[d];
      r /= sh.fac[d];
    }
    int64_t idx = 0;
    for (int d = 0; d < sh.rank; d++) idx = idx * sh.fine[d] + cc[d] * sh.fac[d] + off[d];
    acc += (double)ys[sig * n + idx];
  }
  out[sig * n_low + cell] = acc / (double)block;
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

__global__ void to_bf16_kernel(const double *__restrict__ d, int64_t t, int64_t n, int64_t n_pad,
                               __nv_bfloat16 *__restrict__ out) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= t * n_pad) return;
  const int64_t row = gid / n_pad, col = gid % n_pad;
  out[gid] = __float2bfloat16_rn(col < n ? (float)d[row * n + col] : 0.0f);
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

inline unsigned blocks_for(int64_t work, int threads) {
  return (unsigned)((work + threads - 1) / threads);
}

}  // namespace

cudaError_t launch_downsample(const void *ys, bool ys_f32, int64_t p, int64_t n,
                              const int64_t *fine_shape, const int64_t *factors, int rank,
                              double *y_low, int64_t n_low, cudaStream_t stream) {
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
  const unsigned g = blocks_for(p * n_low, 256);
  if (ys_f32)
    downsample_kernel<float><<<g, 256, 0, stream>>>((const float *)ys, p, n, sh, y_low, n_low);
  else
    downsample_kernel<double><<<g, 256, 0, stream>>>((const double *)ys, p, n, sh, y_low, n_low);
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

cudaError_t launch_to_bf16(const double *d64, int64_t t, int64_t n, int64_t n_pad, void *d16,
                           cudaStream_t stream) {
  ProfScope _ps("to_bf16", stream);
  to_bf16_kernel<<<blocks_for(t * n_pad, 256), 256, 0, stream>>>(d64, t, n, n_pad,
                                                                  (__nv_bfloat16 *)d16);
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

}  // namespace cdb
