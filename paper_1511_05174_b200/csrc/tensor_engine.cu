// Tensor engine: batched OMP over large dictionaries with the correlation
// scan on the 5th-generation tensor cores and a certified fp64 selection.
//
// Per OMP iteration (all signals of the batch in lock-step):
//
//  1. corr_topk_kernel  C = R16 . D16^T on tcgen05 (bf16 x bf16 -> fp32 in
//     TMEM), operands staged by TMA with 128-byte swizzle, two 256-column
//     accumulator buffers so the epilogue of atom tile t overlaps the MMAs
//     of tile t+1.  The epilogue never writes C: each thread keeps, for its
//     signal row, the 8 largest |c| seen and the largest value it dropped.
//     Replaces the reference's scan, _kernels.py:94-103.
//  2. ls_step_kernel (one warp per signal, fp64)  re-scores the approximate
//     winners exactly (c_j = <d_j, r> in fp64) and CERTIFIES the pick: with
//     E the rigorous bf16/fp32 error bound of step 1, every atom outside
//     the re-scored set has |c| <= (its approximate value) + E < best exact.
//     Certified picks are therefore the exact fp64 argmax (ties -> lowest
//     index, as the reference's strict '>' scan).  An uncertifiable pick, or
//     a new atom within 1e-4 |a| of the span of the support, hands the
//     signal to the exact engine.  Then: Cholesky append of the support Gram
//     (G row gather, explicit L^{-1}), z_k = c_new / d (the reference's
//     q_k^T y), coefficients x = L^{-T} z, and the residual r = y - D_S x
//     rematerialised in fp64 from y (no drift), its exact norm for the stop
//     test (_kernels.py:156) and its bf16 copy as the next GEMM operand.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "engines.h"
#include "sm100.cuh"

namespace cdb {
namespace {

constexpr int BM = 128;          // signals per tile (MMA M)
constexpr int BN = 256;          // atoms per tile (MMA N)
constexpr int BK = 64;           // bf16 elements per 128-byte swizzled row chunk
constexpr int STAGES = 4;
constexpr int NCAND = 8;         // approximate candidates kept per signal
constexpr int EPI_WARPS = 8;     // 2 per TMEM lane quarter (column halves)
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr uint32_t A_BYTES = BM * BK * 2;
constexpr uint32_t B_BYTES = BN * BK * 2;
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t TMEM_COLS = 2 * BN;

struct __align__(16) EpiList {
  float val[NCAND];
  int idx[NCAND];
  float dropped;
};

struct CorrSmem {
  uint8_t stage[STAGES][STAGE_BYTES];  // 1024-aligned (base is)
  EpiList part[BM];                    // half-1 partial lists for the merge
  uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void list_insert(float (&val)[NCAND], int (&idx)[NCAND], float &dropped,
                                            float v, int j) {
  if (v > val[NCAND - 1]) {
    float cv = v;
    int ci = j;
#pragma unroll
    for (int i = 0; i < NCAND; i++) {
      const bool sw = cv > val[i];
      const float tv = val[i];
      const int ti = idx[i];
      val[i] = sw ? cv : tv;
      idx[i] = sw ? ci : ti;
      cv = sw ? tv : cv;
      ci = sw ? ti : ci;
    }
    dropped = fmaxf(dropped, cv);
  } else {
    dropped = fmaxf(dropped, v);
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    corr_topk_kernel(const __grid_constant__ CUtensorMap tm_a,
                     const __grid_constant__ CUtensorMap tm_b, int64_t p, int64_t t,
                     int n_kchunks, int64_t m_tiles, const int *__restrict__ active,
                     int *__restrict__ cand_idx, float *__restrict__ cand_val,
                     float *__restrict__ cand_drop) {
  if (active && *active == 0) return;  // every signal already finished
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  CorrSmem &sm = *reinterpret_cast<CorrSmem *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t_tiles = (int)((t + BN - 1) / BN);

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_a);
    sm100::tma_prefetch(&tm_b);
    for (int s = 0; s < STAGES; s++) {
      sm100::mbar_init(&sm.full[s], 1);
      sm100::mbar_init(&sm.empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      sm100::mbar_init(&sm.tfull[a], 1);
      sm100::mbar_init(&sm.tempty[a], EPI_WARPS * 32);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc(&sm.tmem_base, TMEM_COLS);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (int64_t mt = blockIdx.x; mt < m_tiles; mt += gridDim.x) {
        for (int tt = 0; tt < t_tiles; tt++) {
          for (int kc = 0; kc < n_kchunks; kc++) {
            sm100::mbar_wait(&sm.empty[s], ph ^ 1);
            sm100::mbar_expect_tx(&sm.full[s], STAGE_BYTES);
            sm100::tma_load_2d(sm.stage[s], &tm_a, &sm.full[s], kc * BK, (int)(mt * BM));
            sm100::tma_load_2d(sm.stage[s] + A_BYTES, &tm_b, &sm.full[s], kc * BK, tt * BN);
            if (++s == STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_bf16_f32(BM, BN);
      uint32_t s = 0, ph = 0, acc = 0, acc_ph = 0;
      for (int64_t mt = blockIdx.x; mt < m_tiles; mt += gridDim.x) {
        for (int tt = 0; tt < t_tiles; tt++) {
          sm100::mbar_wait(&sm.tempty[acc], acc_ph ^ 1);
          sm100::tc_fence_after();
          const uint32_t d_tmem = tmem + acc * BN;
          for (int kc = 0; kc < n_kchunks; kc++) {
            sm100::mbar_wait(&sm.full[s], ph);
            sm100::tc_fence_after();
            const uint32_t a_addr = sm100::smem_u32(sm.stage[s]);
            const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; k++) {
              sm100::mma_bf16(d_tmem, sm100::desc_kmajor_sw128(a_addr + k * 32),
                              sm100::desc_kmajor_sw128(b_addr + k * 32), idesc,
                              (kc | k) != 0 ? 1u : 0u);
            }
            sm100::mma_commit(&sm.empty[s]);
            if (++s == STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
          sm100::mma_commit(&sm.tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_ph ^= 1;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue: top-k |c| per row
    const int ew = warp - 2;            // 0..7
    const int quarter = warp & 3;       // TMEM lane quarter this warp may access
    const int half = ew >> 2;           // column half of each 256-atom tile
    const int row = quarter * 32 + lane;
    uint32_t acc = 0, acc_ph = 0;
    for (int64_t mt = blockIdx.x; mt < m_tiles; mt += gridDim.x) {
      float val[NCAND];
      int idx[NCAND];
      float dropped = -1.0f;
#pragma unroll
      for (int i = 0; i < NCAND; i++) {
        val[i] = -1.0f;
        idx[i] = -1;
      }
      for (int tt = 0; tt < t_tiles; tt++) {
        sm100::mbar_wait(&sm.tfull[acc], acc_ph);
        sm100::tc_fence_after();
        const int col0 = tt * BN + half * (BN / 2);
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          float v[32];
          sm100::tmem_ld32(tmem + acc * BN + half * (BN / 2) + c + ((uint32_t)(quarter * 32) << 16),
                           v);
#pragma unroll
          for (int i = 0; i < 32; i++) {
            const int j = col0 + c + i;
            if (j < t) list_insert(val, idx, dropped, fabsf(v[i]), j);
          }
        }
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_ph ^= 1;
        }
      }
      // merge the two column halves of each row, write the row's list
      if (half == 1) {
#pragma unroll
        for (int i = 0; i < NCAND; i++) {
          sm.part[row].val[i] = val[i];
          sm.part[row].idx[i] = idx[i];
        }
        sm.part[row].dropped = dropped;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
      if (half == 0) {
#pragma unroll
        for (int i = 0; i < NCAND; i++) {
          const int oi = sm.part[row].idx[i];
          if (oi >= 0) list_insert(val, idx, dropped, sm.part[row].val[i], oi);
        }
        dropped = fmaxf(dropped, sm.part[row].dropped);
        const int64_t grow = mt * BM + row;
        if (grow < p) {
#pragma unroll
          for (int i = 0; i < NCAND; i++) {
            cand_idx[grow * NCAND + i] = idx[i];
            cand_val[grow * NCAND + i] = val[i];
          }
          cand_drop[grow] = dropped;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, TMEM_COLS);
  }
}

// ---------------------------------------------------------------- LS side
struct TensorState {
  double *r64;          // P x n    residual (fp64, exact)
  __nv_bfloat16 *r16;   // Ppad x n_pad   GEMM operand
  double *linv;         // P x kw x kw    L^{-1} row-major
  double *z;            // P x kw
  double *rnorm;        // P   ||r||
  double *tol;          // P
  uint32_t *status;     // P   ST_DONE | ST_DELEGATE
  const int *cand_idx;
  const float *cand_val;
  const float *cand_drop;
  int *active;          // per iteration: signals still running after it
};

template <typename YT>
__global__ void __launch_bounds__(256) ls_init_kernel(const YT *__restrict__ ys, int64_t p,
                                                      int64_t n, int64_t n_pad, int64_t kw,
                                                      const double *__restrict__ eps,
                                                      TensorState st, int64_t *out_sel,
                                                      double *out_coef, int64_t *out_count,
                                                      double *out_rnorm, int64_t *out_scans,
                                                      uint8_t *out_flag) {
  const int64_t sig = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sig >= p) return;
  double *r = st.r64 + sig * n;
  double ss = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    const double v = (double)ys[sig * n + i];
    r[i] = v;
    st.r16[sig * n_pad + i] = __float2bfloat16_rn((float)v);
    ss = fma(v, v, ss);
  }
  __syncwarp();
  const double ynorm = sqrt(dot4_quad(r, r, n, lane));  // reference order (_kernels.py:71)
  (void)ss;
  for (int64_t j = lane; j < kw; j += 32) {
    out_sel[sig * kw + j] = -1;
    out_coef[sig * kw + j] = 0.0;
  }
  if (lane == 0) {
    const double tol = eps[sig];
    st.tol[sig] = tol;
    st.rnorm[sig] = ynorm;
    st.status[sig] = ynorm <= tol ? ST_DONE : 0u;
    out_count[sig] = 0;
    out_rnorm[sig] = ynorm;
    out_scans[sig] = 0;
    out_flag[sig] = 0;
  }
}

// One OMP iteration of one signal per warp (see file comment, step 2).
template <typename YT>
__global__ void __launch_bounds__(256) ls_step_kernel(
    const YT *__restrict__ ys, const double *__restrict__ d64, const double *__restrict__ gram,
    int64_t p, int64_t t, int64_t n, int64_t n_pad, int64_t k_max, int64_t kw, int iter,
    double c_err, double dmax, TensorState st, int64_t *out_sel, double *out_coef,
    int64_t *out_count, double *out_rnorm, int64_t *out_scans) {
  extern __shared__ double lsm[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sig = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (sig >= p) return;
  if (st.status[sig] & (ST_DONE | ST_DELEGATE)) return;
  double *lin = lsm + wib * (kw * kw + 4 * kw);  // L^{-1} rows 0..k-1 (row-major)
  double *wv = lin + kw * kw;                      // w
  double *xv = wv + kw;                            // x
  double *gv = xv + kw;                            // G[new, S]
  double *zv = gv + kw;                            // z
  const int64_t k = iter;                          // atoms selected so far
  int64_t *sel = out_sel + sig * kw;
  const double *r = st.r64 + sig * n;

  // ---- candidates: drop taken atoms, rigorous error bound of the bf16 scan
  int cidx = -1;
  float cval = -1.0f;
  if (lane < NCAND) {
    cidx = st.cand_idx[sig * NCAND + lane];
    cval = st.cand_val[sig * NCAND + lane];
    for (int64_t i = 0; i < k && cidx >= 0; i++)
      if (sel[i] == cidx) cidx = -1;
    if (cidx < 0) cval = -1.0f;
  }
  const double E = c_err * st.rnorm[sig] * dmax;
  double best_apx = (double)cval;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best_apx = fmax(best_apx, __shfl_xor_sync(CDB_FULL_MASK, best_apx, o));
  // every candidate whose approximate value is within 2E of the best is re-scored
  const bool rescore = cidx >= 0 && (double)cval >= best_apx - 2.0 * E;
  const unsigned rmask = __ballot_sync(CDB_FULL_MASK, rescore);
  double unscored = rescore || cidx < 0 ? -1.0 : (double)cval;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) unscored = fmax(unscored, __shfl_xor_sync(CDB_FULL_MASK, unscored, o));
  unscored = fmax(unscored, (double)st.cand_drop[sig]);

  // exact fp64 correlations of the re-scored candidates (warp dot each)
  double best = -1.0;
  int64_t bestj = -1;
  for (unsigned m = rmask; m; m &= m - 1) {
    const int c = __ffs(m) - 1;
    const int64_t j = __shfl_sync(CDB_FULL_MASK, cidx, c);
    const double *dj = d64 + j * n;
    double acc = 0.0;
    for (int64_t i = lane; i < n; i += 32) acc = fma(__ldg(dj + i), r[i], acc);
    const double v = fabs(warp_sum(acc));
    if (v > best || (v == best && j < bestj)) {
      best = v;
      bestj = j;
    }
  }
  const int64_t scans_it = t - k;  // scans += c - k (_kernels.py:91)
  if (bestj < 0 || !(unscored + E < best)) {
    // uncertifiable (or no candidate): the exact engine redoes this signal
    if (lane == 0) st.status[sig] |= ST_DELEGATE;
    return;
  }
  if (lane == 0) out_scans[sig] += scans_it;
  if (best <= 0.0) {  // residual orthogonal to every atom (_kernels.py:104)
    if (lane == 0) st.status[sig] |= ST_DONE;
    return;
  }
  // ---- Cholesky append through the Gram row of the new atom
  const double *grow = gram + bestj * t;
  for (int64_t i = lane; i < k * kw; i += 32) lin[i] = st.linv[sig * kw * kw + i];
  for (int64_t i = lane; i < k; i += 32) {
    gv[i] = __ldg(grow + sel[i]);
    zv[i] = st.z[sig * kw + i];
  }
  const double gnn = __ldg(grow + bestj);
  __syncwarp();
  for (int64_t l = lane; l < k; l += 32) {
    double acc = 0.0;
    for (int64_t i = 0; i <= l; i++) acc = fma(lin[l * kw + i], gv[i], acc);
    wv[l] = acc;
  }
  __syncwarp();
  double ww = 0.0;
  for (int64_t l = lane; l < k; l += 32) ww = fma(wv[l], wv[l], ww);
  ww = warp_sum(ww);
  const double d2 = gnn - ww;
  if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {
    if (lane == 0) st.status[sig] |= ST_DELEGATE;
    return;
  }
  const double inv_d = 1.0 / sqrt(d2);
  // c_new = <d_new, r> = q_k^T r * d and q_k^T y = q_k^T r  =>  z_k = c_new / d
  double cnew = 0.0;
  {
    const double *dj = d64 + bestj * n;
    for (int64_t i = lane; i < n; i += 32) cnew = fma(__ldg(dj + i), r[i], cnew);
    cnew = warp_sum(cnew);
  }
  const double zk = cnew * inv_d;
  for (int64_t i = lane; i <= k; i += 32) {
    double v;
    if (i == k) {
      v = inv_d;
    } else {
      double acc = 0.0;
      for (int64_t l = i; l < k; l++) acc = fma(wv[l], lin[l * kw + i], acc);
      v = -acc * inv_d;
    }
    lin[k * kw + i] = v;
    st.linv[sig * kw * kw + k * kw + i] = v;
  }
  if (lane == 0) {
    zv[k] = zk;
    st.z[sig * kw + k] = zk;
    sel[k] = bestj;
  }
  __syncwarp();
  // ---- coefficients x = L^{-T} z (pick order)
  const int64_t kd = k + 1;
  for (int64_t i = lane; i < kd; i += 32) {
    double acc = 0.0;
    for (int64_t l = i; l < kd; l++) acc = fma(lin[l * kw + i], zv[l], acc);
    xv[i] = acc;
    out_coef[sig * kw + i] = acc;
  }
  __syncwarp();
  // ---- residual r = y - D_S x in fp64, its norm, its bf16 copy
  double *rw = st.r64 + sig * n;
  double rr = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    double ri = (double)ys[sig * n + i];
    for (int64_t l = 0; l < kd; l++) ri = fma(-xv[l], __ldg(d64 + sel[l] * n + i), ri);
    rw[i] = ri;
    st.r16[sig * n_pad + i] = __float2bfloat16_rn((float)ri);
    rr = fma(ri, ri, rr);
  }
  const double rnorm = sqrt(warp_sum(rr));
  if (lane == 0) {
    st.rnorm[sig] = rnorm;
    out_rnorm[sig] = rnorm;
    out_count[sig] = kd;
    const bool done = rnorm <= st.tol[sig] || kd >= k_max;
    if (done)
      st.status[sig] |= ST_DONE;
    else
      atomicAdd(st.active + iter, 1);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  }
  return fn;
}

bool make_map(CUtensorMap *m, const void *base, int64_t rows, int64_t cols_pad, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols_pad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols_pad * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

int64_t tensor_state_bytes(int64_t p, int64_t n, int64_t kw) {
  const int64_t n_pad = (n + BK - 1) / BK * BK;
  const int64_t p_pad = (p + BM - 1) / BM * BM;
  return p * n * 8 + p_pad * n_pad * 2 + p * kw * kw * 8 + p * kw * 8 + p * 8 * 2 + p * 4 +
         p * NCAND * 8 + p * 4;
}

cudaError_t run_tensor_chunk(const TensorArgs &a, cudaStream_t stream) {
  const int64_t p = a.p, n = a.n, kw = a.k_width, t = a.t;
  const int64_t n_pad = (n + BK - 1) / BK * BK;
  const int64_t p_pad = (p + BM - 1) / BM * BM;
  if (a.n_pad != n_pad) return cudaErrorInvalidValue;
  uint8_t *w = (uint8_t *)a.work;
  auto take = [&](int64_t bytes) {
    uint8_t *r = w;
    w += (bytes + 255) & ~int64_t(255);
    return r;
  };
  TensorState st{};
  st.r64 = (double *)take(p * n * 8);
  st.r16 = (__nv_bfloat16 *)take(p_pad * n_pad * 2);
  st.linv = (double *)take(p * kw * kw * 8);
  st.z = (double *)take(p * kw * 8);
  st.rnorm = (double *)take(p * 8);
  st.tol = (double *)take(p * 8);
  st.status = a.status;
  int *cidx = (int *)take(p * NCAND * 4);
  float *cval = (float *)take(p * NCAND * 4);
  float *cdrop = (float *)take(p * 4);
  st.cand_idx = cidx;
  st.cand_val = cval;
  st.cand_drop = cdrop;
  st.active = (int *)take((a.k_max + 1) * 4);
  cudaError_t e;
  if ((e = cudaMemsetAsync(st.r16, 0, p_pad * n_pad * 2, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(st.active, 0, (a.k_max + 1) * 4, stream)) != cudaSuccess) return e;

  CUtensorMap tm_a, tm_b;
  if (!make_map(&tm_a, st.r16, p_pad, n_pad, BM) || !make_map(&tm_b, a.d16, t, n_pad, BN))
    return cudaErrorInvalidValue;

  const unsigned wblocks = (unsigned)((p * 32 + 255) / 256);
  if (a.ys_f32)
    ls_init_kernel<float><<<wblocks, 256, 0, stream>>>((const float *)a.ys, p, n, n_pad, kw, a.eps,
                                                       st, a.out_sel, a.out_coef, a.out_count,
                                                       a.out_rnorm, a.out_scans, a.out_flag);
  else
    ls_init_kernel<double><<<wblocks, 256, 0, stream>>>((const double *)a.ys, p, n, n_pad, kw,
                                                        a.eps, st, a.out_sel, a.out_coef,
                                                        a.out_count, a.out_rnorm, a.out_scans,
                                                        a.out_flag);
  note_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;

  const size_t corr_smem = sizeof(CorrSmem) + 1024;
  if ((e = cudaFuncSetAttribute(corr_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)corr_smem)) != cudaSuccess)
    return e;
  const int64_t m_tiles = p_pad / BM;
  const unsigned corr_grid = (unsigned)(m_tiles < a.num_sms ? m_tiles : a.num_sms);
  const int64_t ls_per_warp = (int64_t)sizeof(double) * (kw * kw + 4 * kw);
  int ls_wpb = (int)((160 * 1024) / ls_per_warp);
  if (ls_wpb > 8) ls_wpb = 8;
  if (ls_wpb < 1) ls_wpb = 1;
  const size_t ls_smem = (size_t)ls_per_warp * ls_wpb;
  if (a.ys_f32) {
    if ((e = cudaFuncSetAttribute(ls_step_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ls_smem)) != cudaSuccess)
      return e;
  } else {
    if ((e = cudaFuncSetAttribute(ls_step_kernel<double>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ls_smem)) !=
        cudaSuccess)
      return e;
  }
  // rigorous bound of |c_bf16 - c| / (|r| |d|): bf16 rounding of both
  // operands (2u + u^2, u = 2^-8) plus fp32 accumulation over n_pad terms
  const double c_err = 2.0 * 0x1p-8 + 0x1p-16 + (double)(n_pad + 16) * 0x1p-23;
  const unsigned ls_grid = (unsigned)((p + ls_wpb - 1) / ls_wpb);
  for (int it = 0; it < a.k_max; it++) {
    corr_topk_kernel<<<corr_grid, THREADS, corr_smem, stream>>>(
        tm_a, tm_b, p, t, (int)(n_pad / BK), m_tiles, it ? st.active + it - 1 : nullptr, cidx,
        cval, cdrop);
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (a.ys_f32)
      ls_step_kernel<float><<<ls_grid, ls_wpb * 32, ls_smem, stream>>>(
          (const float *)a.ys, a.d64, a.gram, p, t, n, n_pad, a.k_max, kw, it, c_err, a.dmax, st,
          a.out_sel, a.out_coef, a.out_count, a.out_rnorm, a.out_scans);
    else
      ls_step_kernel<double><<<ls_grid, ls_wpb * 32, ls_smem, stream>>>(
          (const double *)a.ys, a.d64, a.gram, p, t, n, n_pad, a.k_max, kw, it, c_err, a.dmax, st,
          a.out_sel, a.out_coef, a.out_count, a.out_rnorm, a.out_scans);
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace cdb
