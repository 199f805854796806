// Patch pipeline ends around the pursuit: the denoise /
// recovery flow extract_patches -> OMP -> atoms @ coef -> aggregate_patches
// (crossdict patchwork.py:58-122, pipelines.py:200-253), on the device so the
// patch rows never leave HBM between the steps.
//
//  * extract_rows_kernel: every stride position of a rank <= 4 row-major
//    signal becomes one row of the P x N patch matrix (the OMP row layout:
//    the reference's columns transposed), in fp64.  With remove_dc the
//    per-patch mean is subtracted: summed by one lane in element order and
//    divided by N -- the order numpy's cols.mean(axis=0) reduces in.
//  * reconstruct_kernel: est_p = D_S x (+ dc_p) straight from the solve's
//    (sel, coef) rows -- no dense T x P coefficient matrix.
//  * aggregate_kernel: overlap-add as a gather, one thread per output cell,
//    adding the covering patches in ascending patch order (the reference's
//    accumulation order) and dividing by the coverage count; uncovered cells
//    are 0 and counted.
#include <cstdlib>

#include "common.cuh"
#include "engines.h"

namespace cdb {
namespace {

struct Geom {
  int rank;
  int64_t sig[4];   // signal extents
  int64_t pat[4];   // patch extents
  int64_t str[4];   // strides
  int64_t grid[4];  // patch positions per axis
  int64_t n;        // patch size
  int64_t p;        // patch count
  int64_t cells;    // signal size
};

// linear signal offset of patch element e relative to the patch origin
__device__ __forceinline__ int64_t elem_offset(const Geom &g, int64_t e) {
  int64_t off = 0, mul = 1;
  for (int d = g.rank - 1; d >= 0; d--) {
    const int64_t u = e % g.pat[d];
    e /= g.pat[d];
    off += u * mul;
    mul *= g.sig[d];
  }
  return off;
}

__device__ __forceinline__ int64_t origin_offset(const Geom &g, int64_t p) {
  int64_t off = 0, mul = 1;
  for (int d = g.rank - 1; d >= 0; d--) {
    const int64_t gi = p % g.grid[d];
    p /= g.grid[d];
    off += gi * g.str[d] * mul;
    mul *= g.sig[d];
  }
  return off;
}

// warp per patch; the patch is staged in shared memory (n doubles per warp),
// the cell offsets of a patch relative to its origin are a per-block table
template <typename ST>
__global__ void __launch_bounds__(256) extract_rows_kernel(const ST *__restrict__ sig, Geom g,
                                                           int remove_dc, double *__restrict__ rows,
                                                           double *__restrict__ dc) {
  extern __shared__ double xs[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = (int)g.n;
  const int nwarps = blockDim.x >> 5;
  int *offs = (int *)(xs + (size_t)nwarps * (remove_dc ? 33 : 1) * n);  // n cell offsets
  for (int e = threadIdx.x; e < n; e += blockDim.x) offs[e] = (int)elem_offset(g, e);
  __syncthreads();
  double *buf = xs + (size_t)wib * (remove_dc ? 33 : 1) * n;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  if (!remove_dc) {
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; p < g.p; p += nw) {
      const ST *src = sig + origin_offset(g, p);
      double *dst = rows + p * n;
      for (int e = lane; e < n; e += 32) dst[e] = (double)src[offs[e]];
    }
    return;
  }
  // remove_dc: the mean of each patch is numpy's sequential axis-0 sum, so
  // a warp takes 32 patches at a time, stages them as buf[e][q] (row stride
  // 33: few bank conflicts), and lane q sums patch q in element order -- 32
  // sequential sums in parallel -- before the rows go out coalesced.
  const int64_t nw32 = nw * 32;
  for (int64_t p0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * 32; p0 < g.p; p0 += nw32) {
    const int np = g.p - p0 < 32 ? (int)(g.p - p0) : 32;
    for (int q = 0; q < np; q++) {
      const ST *src = sig + origin_offset(g, p0 + q);
      for (int e = lane; e < n; e += 32) buf[e * 33 + q] = (double)src[offs[e]];
    }
    __syncwarp();
    double s = 0.0;
    if (lane < np)
      for (int e = 0; e < n; e++) s += buf[e * 33 + lane];  // numpy's axis-0 order
    const double mean = s / (double)n;
    if (lane < np) dc[p0 + lane] = mean;
    for (int q = 0; q < np; q++) {
      const double mq = __shfl_sync(CDB_FULL_MASK, mean, q);
      double *dst = rows + (p0 + q) * n;
      for (int e = lane; e < n; e += 32) dst[e] = buf[e * 33 + q] - mq;
    }
    __syncwarp();
  }
}

// Segment extraction: a warp takes up to 32 consecutive patches of one
// patch row (same grid index on every axis but the last).  Their union is
// (n / pl) signal rows of W = (np - 1) s + pl contiguous cells -- read once
// into shared memory (coalesced), instead of n cells per patch.  Lane q sums
// patch q in element order (numpy's axis-0 order, as extract_rows_kernel),
// and the np x n output rows, contiguous in HBM, go out as 16-byte stores.
// toff[e] = tile offset of element e for patch 0 (patch q adds q s).
template <typename ST>
__global__ void __launch_bounds__(512) extract_seg_kernel(const ST *__restrict__ sig, Geom g,
                                                          int remove_dc, int wmax,
                                                          double *__restrict__ rows,
                                                          double *__restrict__ dc) {
  extern __shared__ double xs[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const int n = (int)g.n, rank = g.rank;
  const int pl = (int)g.pat[rank - 1], nrow = n / pl, st = (int)g.str[rank - 1];
  const int64_t gl = g.grid[rank - 1], segs = (gl + 31) / 32, tasks = (g.p / gl) * segs;
  int *toff = (int *)xs;                           // n
  int *roff = toff + n;                            // nrow signal offsets of the tile rows
  double *tile = xs + ((2 * n + 1) / 2 + 1) / 2 * 2 + (size_t)wib * (nrow * wmax + 32);
  double *mean = tile + nrow * wmax;
  for (int e = threadIdx.x; e < n; e += blockDim.x) toff[e] = (e / pl) * wmax + e % pl;
  for (int r = threadIdx.x; r < nrow; r += blockDim.x) roff[r] = (int)elem_offset(g, (int64_t)r * pl);
  __syncthreads();
  for (int64_t task = (int64_t)blockIdx.x * nwb + wib; task < tasks; task += (int64_t)gridDim.x * nwb) {
    const int64_t rowp = task / segs, si = task % segs;
    const int64_t p0 = rowp * gl + si * 32;
    const int np = (int)(gl - si * 32 < 32 ? gl - si * 32 : 32);
    const int w = (np - 1) * st + pl;
    const ST *src = sig + origin_offset(g, p0);
    for (int idx = lane; idx < nrow * w; idx += 32) {
      const int r = idx / w, x = idx - r * w;
      tile[r * wmax + x] = (double)src[roff[r] + x];
    }
    __syncwarp();
    double mq = 0.0;
    if (remove_dc) {
      double s = 0.0;
      if (lane < np)
        for (int e = 0; e < n; e++) s += tile[toff[e] + lane * st];  // numpy's axis-0 order
      mq = s / (double)n;
      if (lane < np) dc[p0 + lane] = mq;
      mean[lane] = mq;
      __syncwarp();
    }
    double *dst = rows + p0 * n;
    const int tot = np * n;
    if ((n & 1) == 0) {  // pairs of elements of one patch: 16-byte stores
      for (int idx = 2 * lane; idx < tot; idx += 64) {
        const int q = idx / n, e = idx - q * n;
        const double t0 = tile[toff[e] + q * st], t1 = tile[toff[e + 1] + q * st];
        *(double2 *)(dst + idx) =
            remove_dc ? make_double2(t0 - mean[q], t1 - mean[q]) : make_double2(t0, t1);
      }
    } else {
      for (int idx = lane; idx < tot; idx += 32) {
        const int q = idx / n, e = idx - q * n;
        const double v = tile[toff[e] + q * st];
        dst[idx] = remove_dc ? v - mean[q] : v;
      }
    }
    __syncwarp();
  }
}

// est[p][e] = sum_l coef[p][l] * d[sel[p][l]][e]  (+ dc[p]); warp per patch.
// The patch's codes are loaded once (lane l holds pick l) and broadcast by
// shuffles; each lane then runs the reference-order fma chain for its
// elements with coalesced atom-row loads.
__global__ void __launch_bounds__(256) reconstruct_kernel(const double *__restrict__ d64,
                                                          int64_t n, const int64_t *__restrict__ sel,
                                                          const double *__restrict__ coef,
                                                          int64_t kw, int64_t p,
                                                          const double *__restrict__ dc,
                                                          double *__restrict__ est) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < p; q += nw) {
    const int64_t *sq = sel + q * kw;
    const double *cq = coef + q * kw;
    const double dq = dc ? dc[q] : 0.0;
    if (kw <= 32 && n <= 64 && (int64_t)n * 65536 < ((int64_t)1 << 31)) {
      const int64_t jl = lane < kw ? sq[lane] : -1;
      const int js = (int)jl * (int)n;  // row offset (T n < 2^31)
      const double cs = lane < kw ? cq[lane] : 0.0;
      // picks before the first -1 (the reference breaks there)
      const unsigned neg = __ballot_sync(CDB_FULL_MASK, lane < kw && jl < 0);
      const int kv = neg ? __ffs(neg) - 1 : (int)kw;
      const int e0 = lane, e1 = lane + 32;
      const int c0 = e0 < n ? e0 : (int)n - 1, c1 = e1 < n ? e1 : (int)n - 1;
      double a0 = 0.0, a1 = 0.0;
      for (int l = 0; l < kv; l++) {
        const double cl = __shfl_sync(CDB_FULL_MASK, cs, l);
        const double *row = d64 + __shfl_sync(CDB_FULL_MASK, js, l);
        a0 = fma(cl, __ldg(row + c0), a0);
        a1 = fma(cl, __ldg(row + c1), a1);
      }
      if (e0 < n) est[q * n + e0] = dc ? a0 + dq : a0;
      if (e1 < n) est[q * n + e1] = dc ? a1 + dq : a1;
      continue;
    }
    for (int64_t e = lane; e < n; e += 32) {
      double acc = 0.0;
      for (int64_t l = 0; l < kw; l++) {
        const int64_t j = sq[l];
        if (j < 0) break;  // -1 padding after the last pick
        acc = fma(cq[l], __ldg(d64 + j * n + e), acc);
      }
      est[q * n + e] = dc ? acc + dq : acc;
    }
  }
}

// thread per output cell: covering patches in ascending patch index
// (dc != NULL: the patch values are est + dc_p, added before accumulation as
// the reference's cols + dc[None, :]).  32-bit index math (cells < 2^31).
__global__ void __launch_bounds__(256) aggregate_kernel(const double *__restrict__ est,
                                                        const double *__restrict__ dc, Geom g,
                                                        double *__restrict__ out,
                                                        unsigned long long *__restrict__ uncovered) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= g.cells) return;
  const int rank = g.rank, n = (int)g.n;
  int xc[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
  {
    int r = x;
    for (int d = rank - 1; d >= 0; d--) {
      xc[d] = r % (int)g.sig[d];
      r /= (int)g.sig[d];
    }
  }
  bool any = true;
  for (int d = 0; d < rank; d++) {  // grid indices gi with gi*str <= xc < gi*str + pat
    const int st = (int)g.str[d];
    const int a = xc[d] - (int)g.pat[d] + 1;
    const int l = a <= 0 ? 0 : (a + st - 1) / st;
    int h = xc[d] / st;
    if (h > (int)g.grid[d] - 1) h = (int)g.grid[d] - 1;
    lo[d] = l;
    hi[d] = h;
    if (l > h) any = false;
  }
  double acc = 0.0, w = 0.0;
  if (any) {
    int gi[4] = {lo[0], lo[1], lo[2], lo[3]};
    bool more = true;
    while (more) {
      // up to 8 covering patches in ascending p: their loads in flight
      // together, accumulated in order
      int off[8], pp[8];  // cells < 2^31 and P n < 2^31 (checked at launch)
      int m = 0;
      while (more && m < 8) {
        int p = 0, e = 0;
        for (int d = 0; d < rank; d++) {
          p = p * (int)g.grid[d] + gi[d];
          e = e * (int)g.pat[d] + (xc[d] - gi[d] * (int)g.str[d]);
        }
        off[m] = p * n + e;
        pp[m] = p;
        m++;
        int d = rank - 1;  // odometer, last axis fastest = ascending p
        while (d >= 0 && ++gi[d] > hi[d]) {
          gi[d] = lo[d];
          d--;
        }
        more = d >= 0;
      }
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u < m) v[u] = __ldg(est + off[u]) + (dc ? __ldg(dc + pp[u]) : 0.0);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u < m) {
          acc += v[u];
          w += 1.0;
        }
    }
  }
  if (w == 0.0) {
    atomicAdd(uncovered, 1ull);
    w = 1.0;
  }
  out[x] = acc / w;
}

cudaError_t make_geom(Geom &g, int rank, const int64_t *sig, const int64_t *pat,
                      const int64_t *str) {
  if (rank < 1 || rank > 4) return cudaErrorInvalidValue;
  g.rank = rank;
  g.n = 1;
  g.p = 1;
  g.cells = 1;
  for (int d = 0; d < 4; d++) g.sig[d] = g.pat[d] = g.str[d] = g.grid[d] = 1;
  for (int d = 0; d < rank; d++) {
    if (pat[d] < 1 || str[d] < 1 || pat[d] > sig[d]) return cudaErrorInvalidValue;
    g.sig[d] = sig[d];
    g.pat[d] = pat[d];
    g.str[d] = str[d];
    g.grid[d] = (sig[d] - pat[d]) / str[d] + 1;
    g.n *= pat[d];
    g.p *= g.grid[d];
    g.cells *= sig[d];
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_extract_patches(const void *signal, bool f32, int rank, const int64_t *sig,
                                   const int64_t *pat, const int64_t *str, int remove_dc,
                                   double *rows, double *dc, int num_sms, cudaStream_t stream) {
  ProfScope _ps("extract_patches", stream);
  Geom g;
  cudaError_t e = make_geom(g, rank, sig, pat, str);
  if (e != cudaSuccess) return e;
  if (g.cells >= (int64_t)1 << 31) return cudaErrorInvalidValue;
  {  // segment path: 32 patches of a patch row share one tile (CDB_EXTRACT_SEG=0: off)
    const int pl = (int)g.pat[rank - 1], st = (int)g.str[rank - 1];
    const int64_t wmax = 31 * (int64_t)st + pl, nrow = g.n / pl;
    const size_t head = (size_t)(((2 * g.n + 1) / 2 + 1) / 2 * 2) * sizeof(double);
    const size_t per_w = (size_t)(nrow * wmax + 32) * sizeof(double);
    const char *sv = getenv("CDB_EXTRACT_SEG");
    if (!(sv && atoi(sv) == 0) && nrow * wmax <= 2048 && wmax < (1 << 20)) {
      int warps = 16;
      while (warps > 1 && head + warps * per_w > 160 * 1024) warps /= 2;
      const size_t smem = head + warps * per_w;
      const int64_t gl = g.grid[rank - 1];
      const int64_t tasks = (g.p / gl) * ((gl + 31) / 32);
      int64_t blocks = (tasks + warps - 1) / warps;
      const int per_sm = (int)((200 * 1024) / smem) < 1 ? 1 : (int)((200 * 1024) / smem);
      if (blocks > (int64_t)num_sms * per_sm) blocks = (int64_t)num_sms * per_sm;
      auto sf = extract_seg_kernel<float>;
      auto sd = extract_seg_kernel<double>;
      if ((e = cudaFuncSetAttribute(f32 ? (const void *)sf : (const void *)sd,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
          cudaSuccess)
        return e;
      if (f32)
        sf<<<(unsigned)blocks, 32 * warps, smem, stream>>>((const float *)signal, g, remove_dc,
                                                            (int)wmax, rows, dc);
      else
        sd<<<(unsigned)blocks, 32 * warps, smem, stream>>>((const double *)signal, g, remove_dc,
                                                            (int)wmax, rows, dc);
      note_launch();
      return cudaGetLastError();
    }
  }
  // 8 warps; remove_dc stages 32 patches per warp
  const size_t per_warp = (remove_dc ? 33 : 1) * sizeof(double) * (size_t)g.n;
  int warps = 8;
  while (warps > 1 && warps * per_warp + sizeof(int) * (size_t)g.n > 200 * 1024) warps /= 2;
  const size_t smem = warps * per_warp + sizeof(int) * (size_t)g.n;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  const int64_t per_block = (int64_t)warps * (remove_dc ? 32 : 1);
  int64_t blocks = (g.p + per_block - 1) / per_block;
  if (blocks > (int64_t)num_sms * 32) blocks = (int64_t)num_sms * 32;
  if (g.cells >= (int64_t)1 << 31) return cudaErrorInvalidValue;
  auto kf = extract_rows_kernel<float>;
  auto kd = extract_rows_kernel<double>;
  if ((e = cudaFuncSetAttribute(f32 ? (const void *)kf : (const void *)kd,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  if (f32)
    kf<<<(unsigned)blocks, 32 * warps, smem, stream>>>((const float *)signal, g, remove_dc, rows, dc);
  else
    kd<<<(unsigned)blocks, 32 * warps, smem, stream>>>((const double *)signal, g, remove_dc, rows, dc);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_reconstruct_aggregate(const double *d64, int64_t n, const int64_t *sel,
                                         const double *coef, int64_t kw, int64_t p,
                                         const double *dc, int rank, const int64_t *sig,
                                         const int64_t *pat, const int64_t *str, double *est,
                                         double *out, unsigned long long *uncovered, int num_sms,
                                         cudaStream_t stream) {
  ProfScope _ps("reconstruct_aggregate", stream);
  Geom g;
  cudaError_t e = make_geom(g, rank, sig, pat, str);
  if (e != cudaSuccess) return e;
  if (g.n != n || g.p != p) return cudaErrorInvalidValue;
  if (g.cells >= (int64_t)1 << 31) return cudaErrorInvalidValue;
  if (p * n >= (int64_t)1 << 31) return cudaErrorInvalidValue;
  int64_t blocks = (p + 7) / 8;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  reconstruct_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d64, n, sel, coef, kw, p, dc, est);
  aggregate_kernel<<<(unsigned)((g.cells + 255) / 256), 256, 0, stream>>>(est, nullptr, g, out,
                                                                           uncovered);
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_aggregate(const double *rows, const double *dc, int rank, const int64_t *sig,
                             const int64_t *pat, const int64_t *str, double *out,
                             unsigned long long *uncovered, cudaStream_t stream) {
  ProfScope _ps("aggregate", stream);
  Geom g;
  cudaError_t e = make_geom(g, rank, sig, pat, str);
  if (e != cudaSuccess) return e;
  if (g.cells >= (int64_t)1 << 31 || g.p * g.n >= (int64_t)1 << 31) return cudaErrorInvalidValue;
  aggregate_kernel<<<(unsigned)((g.cells + 255) / 256), 256, 0, stream>>>(rows, dc, g, out,
                                                                           uncovered);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cdb
