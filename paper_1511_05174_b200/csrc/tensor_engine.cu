// Tensor engine: batched OMP over large dictionaries with the correlation
// scan on the 5th-generation tensor cores and a certified fp64 selection.
//
// Per OMP iteration (all signals of the batch in lock-step):
//
//  1. corr_topk_kernel  C = R16 . D16^T on tcgen05 (fp16 x fp16 -> fp32 in
//     TMEM), operands staged by TMA with 128-byte swizzle, two 256-column
//     accumulator buffers so the epilogue of atom tile t overlaps the MMAs
//     of tile t+1.  The epilogue never writes C: each thread keeps, for its
//     signal row, the 8 largest |c| seen and the largest value it dropped.
//     Replaces the reference's scan, _kernels.py:94-103.
//  2. ls_step_kernel (one warp per signal, fp64)  re-scores the approximate
//     winners exactly (c_j = <d_j, r> in fp64) and CERTIFIES the pick: with
//     E the rigorous fp16/fp32 error bound of step 1, every atom outside
//     the re-scored set has |c| <= (its approximate value) + E < best exact.
//     Certified picks are therefore the exact fp64 argmax (ties -> lowest
//     index, as the reference's strict '>' scan).  An uncertifiable pick, or
//     a new atom within 1e-4 |a| of the span of the support, hands the
//     signal to the exact engine.  Then: Cholesky append of the support Gram
//     (G row gather, explicit L^{-1}), z_k = c_new / d (the reference's
//     q_k^T y), coefficients x = L^{-T} z, and the residual r = y - D_S x
//     rematerialised in fp64 from y (no drift), its exact norm for the stop
//     test (_kernels.py:156) and its scaled fp16 copy as the next GEMM operand.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "engines.h"
#include "sm100.cuh"

namespace cdb {
namespace {

constexpr int BMH = 128;         // rows per M half (one MMA, M = 128)
constexpr int BM = 2 * BMH;      // signals per CTA tile (two halves share each B stage)
constexpr int BN = 128;          // atoms per tile (MMA N)
constexpr int BK = 64;           // fp16 elements per 128-byte swizzled row chunk
constexpr int NCAND = 8;         // approximate candidates kept per signal
constexpr int EPI_WARPS = 8;     // 4 TMEM lane quarters x 2 M halves: one row per thread
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr uint32_t AH_BYTES = BMH * BK * 2;   // one M half, one K chunk (16 KB)
constexpr uint32_t B_BYTES = BN * BK * 2;     // one atom tile, one K chunk (16 KB)
constexpr uint32_t TMEM_COLS = 4 * BN;        // 2 buffers x 2 halves
constexpr int RES_KCHUNKS = 4;                // A resident when n_pad <= 256
constexpr int RES_BSTAGES = 4;
constexpr int STR_STAGES = 4;

struct CorrSmemRes {                                   // A resident in smem
  uint8_t a[RES_KCHUNKS][2][AH_BYTES];
  uint8_t b[RES_BSTAGES][B_BYTES];
  uint64_t full[RES_BSTAGES], empty[RES_BSTAGES], tfull[2], tempty[2], afull, aempty;
  uint32_t tmem_base;
};
struct CorrSmemStr {                                   // A streamed with B
  uint8_t st[STR_STAGES][2 * AH_BYTES + B_BYTES];
  uint64_t full[STR_STAGES], empty[STR_STAGES], tfull[2], tempty[2], afull, aempty;
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

template <bool A_RES, bool SPLIT>
__global__ void __launch_bounds__(THREADS, 1)
    corr_topk_kernel(const __grid_constant__ CUtensorMap tm_a,
                     const __grid_constant__ CUtensorMap tm_b, int64_t p, int64_t t,
                     int n_kchunks, int64_t m_tiles, const int *__restrict__ active,
                     int *__restrict__ cand_idx, float *__restrict__ cand_val,
                     float *__restrict__ cand_drop, int nsplit_arg) {
  // SPLIT = false compiles the single-part scan exactly as before the split
  const int nsplit = SPLIT ? nsplit_arg : 1;
  griddep_wait();  // the previous kernel's residuals and active count (PDL)
  griddep_launch();
  if (active && *active == 0) return;  // every signal already finished
  using Smem = typename std::conditional<A_RES, CorrSmemRes, CorrSmemStr>::type;
  constexpr int NST = A_RES ? RES_BSTAGES : STR_STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem &sm = *reinterpret_cast<Smem *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                       ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t_tiles = (int)((t + BN - 1) / BN);
  // work item = (signal tile mt, dictionary part q of nsplit): items of one
  // signal tile are adjacent, so the CTAs in flight share few signal tiles
  // (their A stays in L2) and stream the same dictionary parts together
  const int tpq = (t_tiles + nsplit - 1) / nsplit;
  const int64_t n_items = m_tiles * nsplit;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_a);
    sm100::tma_prefetch(&tm_b);
    for (int s = 0; s < NST; s++) {
      sm100::mbar_init(&sm.full[s], 1);
      sm100::mbar_init(&sm.empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      sm100::mbar_init(&sm.tfull[a], 1);
      sm100::mbar_init(&sm.tempty[a], EPI_WARPS * 32);
    }
    sm100::mbar_init(&sm.afull, 1);
    sm100::mbar_init(&sm.aempty, 1);
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
      uint32_t s = 0, ph = 0, aph = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int64_t mt = item / nsplit;
        const int tt0 = (int)(item % nsplit) * tpq, tt1 = tt0 + tpq < t_tiles ? tt0 + tpq : t_tiles;
        const int row0 = (int)(mt * BM);
        if constexpr (A_RES) {
          sm100::mbar_wait(&sm.aempty, aph ^ 1);
          sm100::mbar_expect_tx(&sm.afull, (uint32_t)n_kchunks * 2 * AH_BYTES);
          for (int kc = 0; kc < n_kchunks; kc++)
            for (int h = 0; h < 2; h++)
              sm100::tma_load_2d(sm.a[kc][h], &tm_a, &sm.afull, kc * BK, row0 + h * BMH);
          aph ^= 1;
        }
        for (int tt = tt0; tt < tt1; tt++) {
          for (int kc = 0; kc < n_kchunks; kc++) {
            sm100::mbar_wait(&sm.empty[s], ph ^ 1);
            if constexpr (A_RES) {
              sm100::mbar_expect_tx(&sm.full[s], B_BYTES);
              sm100::tma_load_2d(sm.b[s], &tm_b, &sm.full[s], kc * BK, tt * BN);
            } else {
              sm100::mbar_expect_tx(&sm.full[s], 2 * AH_BYTES + B_BYTES);
              sm100::tma_load_2d(sm.st[s], &tm_a, &sm.full[s], kc * BK, row0);
              sm100::tma_load_2d(sm.st[s] + AH_BYTES, &tm_a, &sm.full[s], kc * BK, row0 + BMH);
              sm100::tma_load_2d(sm.st[s] + 2 * AH_BYTES, &tm_b, &sm.full[s], kc * BK, tt * BN);
            }
            if (++s == NST) {
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
      constexpr uint32_t idesc = sm100::idesc_f16_f32(BMH, BN);
      uint32_t s = 0, ph = 0, acc = 0, acc_ph = 0, aph = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int tt0 = (int)(item % nsplit) * tpq, tt1 = tt0 + tpq < t_tiles ? tt0 + tpq : t_tiles;
        if constexpr (A_RES) {
          sm100::mbar_wait(&sm.afull, aph);
          aph ^= 1;
          sm100::tc_fence_after();
        }
        for (int tt = tt0; tt < tt1; tt++) {
          sm100::mbar_wait(&sm.tempty[acc], acc_ph ^ 1);
          sm100::tc_fence_after();
          for (int kc = 0; kc < n_kchunks; kc++) {
            sm100::mbar_wait(&sm.full[s], ph);
            sm100::tc_fence_after();
            uint32_t a0, a1, b;
            if constexpr (A_RES) {
              a0 = sm100::smem_u32(sm.a[kc][0]);
              a1 = sm100::smem_u32(sm.a[kc][1]);
              b = sm100::smem_u32(sm.b[s]);
            } else {
              a0 = sm100::smem_u32(sm.st[s]);
              a1 = a0 + AH_BYTES;
              b = a0 + 2 * AH_BYTES;
            }
#pragma unroll
            for (int k = 0; k < BK / 16; k++) {
              const uint64_t bd = sm100::desc_kmajor_sw128(b + k * 32);
              const uint32_t accum = (kc | k) != 0 ? 1u : 0u;
              sm100::mma_f16(tmem + (acc * 2 + 0) * BN, sm100::desc_kmajor_sw128(a0 + k * 32), bd,
                              idesc, accum);
              sm100::mma_f16(tmem + (acc * 2 + 1) * BN, sm100::desc_kmajor_sw128(a1 + k * 32), bd,
                              idesc, accum);
            }
            sm100::mma_commit(&sm.empty[s]);
            if (++s == NST) {
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
        if constexpr (A_RES) sm100::mma_commit(&sm.aempty);
      }
    }
  } else {
    // ------------------------------------------------ epilogue: top-k |c| per row
    const int ew = warp - 2;       // 0..7
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int half = ew >> 2;      // M half
    const int row = half * BMH + quarter * 32 + lane;
    uint32_t acc = 0, acc_ph = 0;
    // chunk-local column ids in registers (opaque to constant folding) so a
    // key is one LOP3 (mask | id) instead of two
    uint32_t cid[2][32];
    const uint32_t opaque0 = (uint32_t)threadIdx.x >> 16;  // 0 at runtime
#pragma unroll
    for (int i = 0; i < 64; i++) cid[i >> 5][i & 31] = opaque0 + (uint32_t)i;
    const uint32_t k63 = 63u + opaque0;  // kept in a register
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t mt = item / nsplit;
      const int q = (int)(item % nsplit);
      const int tt0 = q * tpq, tt1 = tt0 + tpq < t_tiles ? tt0 + tpq : t_tiles;
      float val[NCAND];
      int idx[NCAND];
      float dropped = -1.0f;
#pragma unroll
      for (int i = 0; i < NCAND; i++) {
        val[i] = -1.0f;
        idx[i] = -1;
      }
      for (int tt = tt0; tt < tt1; tt++) {
        sm100::mbar_wait(&sm.tfull[acc], acc_ph);
        sm100::tc_fence_after();
        const uint32_t tbase = tmem + (acc * 2 + half) * BN + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
        for (int c = 0; c < BN; c += 64) {
          float v[2][32];
          sm100::tmem_ld32(tbase + c, v[0]);
          sm100::tmem_ld32(tbase + c + 32, v[1]);
          // branchless top-2 of 64 columns on packed keys: |v| with its low 6
          // mantissa bits replaced by the column within the 64 (truncation
          // <= 2^-17 rel., inside c_err); everything else raises `dropped`
          uint32_t c1 = 0u, c2 = 0u, rest = 0u;
          const int jbase = tt * BN + c;
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            if (jbase + 32 * hh + 32 <= t) {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                // (bits | 63) & (0x7FFFFFC0 | id) == (bits & 0x7FFFFFC0) | id: one LOP3
                // (63 in a register, the id folded into the immediate)
                uint32_t ka, kb;
                asm("lop3.b32 %0, %1, %2, %3, 0xA8;"
                    : "=r"(ka)
                    : "r"(__float_as_uint(v[hh][i])), "r"(k63), "r"(0x7FFFFFC0u | (uint32_t)(32 * hh + i)));
                asm("lop3.b32 %0, %1, %2, %3, 0xA8;"
                    : "=r"(kb)
                    : "r"(__float_as_uint(v[hh][i + 1])), "r"(k63),
                      "r"(0x7FFFFFC0u | (uint32_t)(32 * hh + i + 1)));
                // merge the sorted pair (hi, lo) into (c1 >= c2) and `rest`:
                // c2' = max(min(c1,hi), c2, lo), third = max(min(c1,lo), min(c2,hi))
                const uint32_t hi = max(ka, kb), lo = min(ka, kb);
                const uint32_t n2 = max(max(min(c1, hi), c2), lo);
                rest = max(max(rest, min(c1, lo)), min(c2, hi));
                c1 = max(c1, hi);
                c2 = n2;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; i++) {
                uint32_t key = (__float_as_uint(v[hh][i]) & 0x7FFFFFC0u) | cid[hh][i];
                key = (jbase + 32 * hh + i < t) ? key : 0u;
                const uint32_t m = min(c1, key);
                c1 = max(c1, key);
                rest = max(rest, min(c2, m));
                c2 = max(c2, m);
              }
            }
          }
          dropped = fmaxf(dropped, __uint_as_float(rest & 0xFFFFFFC0u));
          if (c1) list_insert(val, idx, dropped, __uint_as_float(c1 & 0xFFFFFFC0u),
                              jbase + (int)(c1 & 0x3Fu));
          if (c2) list_insert(val, idx, dropped, __uint_as_float(c2 & 0xFFFFFFC0u),
                              jbase + (int)(c2 & 0x3Fu));
        }
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_ph ^= 1;
        }
      }
      const int64_t grow = mt * BM + row;
      if (grow < p) {  // nsplit > 1: partial lists [p][nsplit][NCAND], merged by merge_cands
        const int64_t slot = grow * nsplit + q;
#pragma unroll
        for (int i = 0; i < NCAND; i++) {
          cand_idx[slot * NCAND + i] = idx[i];
          cand_val[slot * NCAND + i] = val[i];
        }
        cand_drop[slot] = dropped;
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, TMEM_COLS);
  }
}

// The nsplit partial top-8 lists of a signal (one per dictionary part) ->
// its top-8 (by value, lower atom id on equal values) and `dropped` = the
// largest value left out (the parts' own dropped values included): warp per
// signal, lane = one partial candidate, its rank found against all 32.
__global__ void __launch_bounds__(256) merge_cands_kernel(const int *__restrict__ pidx,
                                                          const float *__restrict__ pval,
                                                          const float *__restrict__ pdrop,
                                                          int64_t p, int nsplit,
                                                          const int *__restrict__ active,
                                                          int *__restrict__ cand_idx,
                                                          float *__restrict__ cand_val,
                                                          float *__restrict__ cand_drop) {
  griddep_wait();
  griddep_launch();
  if (active && *active == 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t sig = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sig >= p) return;
  const int tot = nsplit * NCAND;  // <= 64: two partial candidates per lane
  int j[2];
  float v[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int e = lane + 32 * h;
    j[h] = e < tot ? pidx[sig * tot + e] : -1;
    v[h] = e < tot && j[h] >= 0 ? pval[sig * tot + e] : -1.0f;
  }
  int rank[2] = {0, 0};
  for (int q = 0; q < 64; q++) {
    const float vq = __shfl_sync(CDB_FULL_MASK, v[q >> 5], q & 31);
    const int jq = __shfl_sync(CDB_FULL_MASK, j[q >> 5], q & 31);
#pragma unroll
    for (int h = 0; h < 2; h++)
      rank[h] += (vq > v[h]) || (vq == v[h] && (unsigned)jq < (unsigned)j[h]) ||
                 (vq == v[h] && jq == j[h] && q < lane + 32 * h);
  }
  float drop = lane < nsplit ? pdrop[sig * nsplit + lane] : -1.0f;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    if (rank[h] < NCAND) {
      cand_idx[sig * NCAND + rank[h]] = j[h];
      cand_val[sig * NCAND + rank[h]] = v[h];
    } else {
      drop = fmaxf(drop, v[h]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) drop = fmaxf(drop, __shfl_xor_sync(CDB_FULL_MASK, drop, o));
  if (lane == 0) cand_drop[sig] = drop;
}

__global__ void to_f16_rows(const float *__restrict__ rows, int64_t p, int64_t n, int64_t n_pad,
                            __half *__restrict__ out) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= p * n_pad) return;
  const int64_t r = gid / n_pad, c = gid % n_pad;
  out[gid] = __float2half_rn(c < n ? rows[r * n + c] : 0.0f);
}

// debug pass: candidate values back in the dictionary's own units
__global__ void unscale_vals(float *__restrict__ val, float *__restrict__ drop, int64_t p,
                             float inv) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid < p * NCAND) val[gid] *= inv;
  if (gid < p) drop[gid] *= inv;
}

// ---------------------------------------------------------------- LS side
// Power-of-two scale of a signal's fp16 scan operand: with b >= |r~|^2 (the
// running |y|^2 - |z|^2, floored at 2^-40 |y|^2 against cancellation) every
// scaled element stays below 2^14, a factor 4 under the fp16 maximum, and the
// typical element |r~| / sqrt(N) keeps all 11 significand bits.  Writer and
// reader derive it from the same stored (rn2, yy) pair.  An operand that
// overflows anyway measures an infinite rounding error, so its picks are
// never certified (exact rescan).
// (Exponents are taken and powers of two built from the bit patterns: no
// libdevice slow-path calls inside the register-tuned operand kernels.)
__device__ __forceinline__ int scan_scale_exp(double rn2, double yy) {
  const double b = fmax(rn2, yy * 0x1p-40);
  if (!(b > 0x1p-200) || !(b < 0x1p200)) return 0;
  return 13 - ((((__double2hiint(b) >> 20) & 0x7ff) - 1023) >> 1);  // in [-87, 113]
}
__device__ __forceinline__ double pow2d(int e) { return __hiloint2double((1023 + e) << 20, 0); }
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// Store the fp16 scan operand element of s * r~ and return the squared rounding
// error of the value the scan sees, fp16(s v) / s - v.
__device__ __forceinline__ double put_r16(__half *dst, double v, double s, double inv_s) {
  const __half b = __float2half_rn((float)(v * s));
  *dst = b;
  const double e = (double)__half2float(b) * inv_s - v;
  return e * e;
}

// L^{-1} layout (shared and global): row stride kwp = kw rounded up to 16,
// element (l, i) at l * kwp + (i ^ (l & 15)).  Lanes walking a column (fixed
// i, l = lane) hit 16 distinct banks; lanes walking a row stay inside one
// aligned 128-byte block.
__device__ __forceinline__ int64_t lsw(int64_t l, int64_t i, int64_t kwp) {
  return l * kwp + (i ^ (l & 15));
}

struct TensorState {
  __half *r16;          // Ppad x n_pad   GEMM operand  fp16(s r~), r~ = y - D32_S x, s = scan_scale
  double *linv;         // P x kw x kwp   L^{-1}, swizzled rows (lsw)
  double *z;            // P x kw         q_i^T y
  double *rn2;          // P   |y|^2 - |z|^2   (= |r|^2 up to rounding)
  double *yy;           // P   |y|^2
  double *rt;           // P   |r~|  (operand of the fp16 scan)
  double *dr;           // P   bound on |r~ - r|
  double *rq;           // P   |fp16(s r~) / s - r~| (the scan operand's rounding, exact)
  double emax;          // max_j |fp16(dscale d_j) / dscale - d_j| (the dictionary operand's rounding)
  double dinv;          // 1 / (power-of-two scale of the dictionary operand)
  double *tol;          // P
  uint32_t *status;     // P   ST_DONE | ST_DELEGATE
  const int *cand_idx;
  const float *cand_val;
  const float *cand_drop;
  int *active;          // per iteration: signals still running after it
  int *rescans;         // count of exact rescans (uncertifiable picks)
  int *npending;        // per iteration: queued rescans
  int64_t *pending;     // queued signal ids
  int64_t *rs_j;        // rescan result: atom
  double *rs_c;         // rescan result: exact correlation
  double *rs_pv;        // per pending slot x RS_SPLIT: partial best |c|, atom, c
  int64_t *rs_pj;
  double *rs_pc;
  int *rs_cnt;          // per pending slot: parts done (reset by the last part)
  int64_t debug_sig;    // CDB_LS_DEBUG: printf trace of one signal
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
  const YT *y = ys + sig * n;
  double yy = 0.0, q2 = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    const double v = (double)y[i];
    yy = fma(v, v, yy);
  }
  yy = warp_sum(yy);
  const int e16 = scan_scale_exp(yy, yy);
  const double s16 = pow2d(e16), inv16 = pow2d(-e16);
  for (int64_t i = lane; i < n; i += 32)
    q2 += put_r16(st.r16 + sig * n_pad + i, (double)y[i], s16, inv16);
  q2 = warp_sum(q2);
  // |y| in the reference's _dot4 order (_kernels.py:27-47,71): lanes 0-3
  // run the four accumulator chains, the tail is added last
  const int64_t m4 = (n / 4) * 4;
  double part = 0.0;
  if (lane < 4)
    for (int64_t i = lane; i < m4; i += 4) {
      const double v = (double)y[i];
      part = __dadd_rn(part, __dmul_rn(v, v));
    }
  const double s0 = __shfl_sync(CDB_FULL_MASK, part, 0), s1 = __shfl_sync(CDB_FULL_MASK, part, 1);
  const double s2 = __shfl_sync(CDB_FULL_MASK, part, 2), s3 = __shfl_sync(CDB_FULL_MASK, part, 3);
  double tot = __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3);
  for (int64_t i = m4; i < n; i++) {
    const double v = (double)y[i];
    tot = __dadd_rn(tot, __dmul_rn(v, v));
  }
  const double ynorm = sqrt(tot);
  for (int64_t j = lane; j < kw; j += 32) {
    out_sel[sig * kw + j] = -1;
    out_coef[sig * kw + j] = 0.0;
  }
  if (lane == 0) {
    const double tol = eps[sig];
    st.tol[sig] = tol;
    st.yy[sig] = yy;
    st.rn2[sig] = yy;
    st.rt[sig] = sqrt(yy);
    st.dr[sig] = 0.0;
    st.rq[sig] = sqrt(q2) * (1.0 + 1e-12);
    st.status[sig] = ynorm <= tol ? ST_DONE : 0u;
    out_count[sig] = 0;
    out_rnorm[sig] = ynorm;
    out_scans[sig] = 0;
    out_flag[sig] = 0;
  }
}

// exact c_j = <d_j, y> - sum_s G[j, s] x_s  (fp64; the whole warp).  The
// gathered G[j, S] entries stay in the caller's registers (g0: s = lane,
// g1: s = lane + 32) so the winner's row is reused by the Cholesky update.
__device__ __forceinline__ double exact_corr(const double *__restrict__ d64,
                                             const double *__restrict__ gram, int64_t t, int n,
                                             int64_t j, const double *y, const int64_t *sel,
                                             const double *x, int k, int lane, double &g0,
                                             double &g1) {
  const double *dj = d64 + j * n;
  const double *gj = gram + j * t;
  g0 = lane < k ? __ldg(gj + sel[lane]) : 0.0;
  g1 = lane + 32 < k ? __ldg(gj + sel[lane + 32]) : 0.0;
  double acc = 0.0, acc2 = 0.0;
  int i = lane;
  for (; i + 32 < n; i += 64) {
    acc = fma(__ldg(dj + i), y[i], acc);
    acc2 = fma(__ldg(dj + i + 32), y[i + 32], acc2);
  }
  if (i < n) acc = fma(__ldg(dj + i), y[i], acc);
  acc += acc2;
  acc = fma(-g0, lane < k ? x[lane] : 0.0, acc);
  acc = fma(-g1, lane + 32 < k ? x[lane + 32] : 0.0, acc);
  for (int s = lane + 64; s < k; s += 32) acc = fma(-__ldg(gj + sel[s]), x[s], acc);
  return warp_sum(acc);
}

constexpr uint32_t ST_RESCAN = 4u;  // pick needs the exact full rescan
constexpr uint32_t ST_RESID = 8u;   // split mode: the next scan operand is still to be built

// Append atom `bestj` (exact correlation cbest) to the signal's support:
// Cholesky update through the Gram row, coefficients, stop test, and the
// fp16 operand of the next scan.  Whole warp; smem per warp as in ls_step.
__device__ void ls_update(const double *__restrict__ d64, const float *__restrict__ d32,
                          const double *__restrict__ gram, int64_t sig, int64_t t, int64_t n,
                          int64_t n_pad, int64_t k_max, int64_t kw, int iter, double dmax,
                          TensorState &st, int64_t *sel, int64_t *ssel, double *out_coef,
                          int64_t *out_count,
                          int64_t bestj, double cbest, double *lin, double *wv, double *xv,
                          double *gv, double *zv, const double *y, int lane, double g0, double g1,
                          double rn2_prev, double tol, double yy) {
  const int64_t k = iter;
  const int64_t ldl = (kw + 15) & ~int64_t(15);  // L^{-1} row stride (see lsw)
  const double *grow = gram + bestj * t;
  const double gnn = __ldg(grow + bestj);
  if (lane < k) gv[lane] = g0;
  if (lane + 32 < k) gv[lane + 32] = g1;
  for (int64_t i = lane + 64; i < k; i += 32) gv[i] = __ldg(grow + sel[i]);
  __syncwarp();
  for (int64_t l = lane; l < k; l += 32) {
    double acc = 0.0;
    for (int64_t i = 0; i <= l; i++) acc = fma(lin[lsw(l, i, ldl)], gv[i], acc);
    wv[l] = acc;
  }
  __syncwarp();
  double ww = 0.0;
  for (int64_t l = lane; l < k; l += 32) ww = fma(wv[l], wv[l], ww);
  ww = warp_sum(ww);
  const double d2 = gnn - ww;
  if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine decides
    if (lane == 0) st.status[sig] |= ST_DELEGATE;
    return;
  }
  const double inv_d = 1.0 / sqrt(d2);
  // <d_new, r> = d q_k^T r and q_k^T y = q_k^T r  =>  z_k = c_new / d
  const double zk = cbest * inv_d;
  for (int64_t i = lane; i <= k; i += 32) {
    double v;
    if (i == k) {
      v = inv_d;
    } else {
      double acc = 0.0;
      for (int64_t l = i; l < k; l++) acc = fma(wv[l], lin[lsw(l, i, ldl)], acc);
      v = -acc * inv_d;
    }
    lin[lsw(k, i, ldl)] = v;
    st.linv[sig * kw * ldl + lsw(k, i, ldl)] = v;
  }
  if (lane == 0) {
    zv[k] = zk;
    st.z[sig * kw + k] = zk;
    sel[k] = bestj;
    ssel[k] = bestj;
  }
  __syncwarp();
  const int64_t kd = k + 1;
  for (int64_t i = lane; i < kd; i += 32) {
    double acc = 0.0;
    for (int64_t l = i; l < kd; l++) acc = fma(lin[lsw(l, i, ldl)], zv[l], acc);
    xv[i] = acc;
    out_coef[sig * kw + i] = acc;
  }
  __syncwarp();
  // ---- stop test on |r|^2 = |y|^2 - |z|^2, exact residual inside the band
  const double rn2 = rn2_prev - zk * zk;
  const double gap = rn2 - tol * tol;
  bool stop;
  if (fabs(gap) > 1e-12 * yy) {
    stop = gap < 0.0;
  } else {
    double rr = 0.0;
    for (int64_t i = lane; i < n; i += 32) {
      double ri = y[i];
      for (int64_t l = 0; l < kd; l++) ri = fma(-xv[l], __ldg(d64 + ssel[l] * n + i), ri);
      rr = fma(ri, ri, rr);
    }
    stop = sqrt(warp_sum(rr)) <= tol;
  }
  if (lane == 0) {
    st.rn2[sig] = rn2;
    out_count[sig] = kd;
  }
  if (stop || kd >= k_max) {
    if (lane == 0) st.status[sig] |= ST_DONE;
    return;
  }
  // ---- next scan operand: r~ = y - D32_S x (fp64 accumulate) -> fp16(s r~).
  // 8 elements per lane per pass: each support atom row is read coalesced.
  double rr = 0.0, sx = 0.0, q2 = 0.0;
  const int e16 = scan_scale_exp(rn2, yy);
  const double s16 = pow2d(e16), inv16 = pow2d(-e16);
  for (int64_t i0 = 0; i0 < n; i0 += 256) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int64_t i = i0 + u * 32 + lane;
      acc[u] = i < n ? y[i] : 0.0;
    }
    int64_t l = 0;
    for (; l + 1 < kd; l += 2) {  // two support atoms per step: 16 loads in flight
      const float *row0 = d32 + ssel[l] * n;
      const float *row1 = d32 + ssel[l + 1] * n;
      const double x0 = xv[l], x1 = xv[l + 1];
      float v0[8], v1[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int64_t i = i0 + u * 32 + lane;
        v0[u] = i < n ? __ldg(row0 + i) : 0.0f;
        v1[u] = i < n ? __ldg(row1 + i) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) acc[u] = fma(-x1, (double)v1[u], fma(-x0, (double)v0[u], acc[u]));
    }
    if (l < kd) {
      const float *row = d32 + ssel[l] * n;
      const double xl = xv[l];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int64_t i = i0 + u * 32 + lane;
        if (i < n) acc[u] = fma(-xl, (double)__ldg(row + i), acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int64_t i = i0 + u * 32 + lane;
      if (i < n) {
        q2 += put_r16(st.r16 + sig * n_pad + i, acc[u], s16, inv16);
        rr = fma(acc[u], acc[u], rr);
      }
    }
  }
  for (int64_t l = lane; l < kd; l += 32) sx += fabs(xv[l]);
  rr = warp_sum(rr);
  sx = warp_sum(sx);
  q2 = warp_sum(q2);
  if (lane == 0) {
    st.rq[sig] = sqrt(q2) * (1.0 + 1e-12);
    st.rt[sig] = sqrt(rr);
    st.dr[sig] = 0x1p-24 * sx * dmax * 1.0000001;  // |(D64 - D32) x| bound
    atomicAdd(st.active + iter, 1);
  }
}

// One OMP iteration of one signal per warp (see file comment, step 2).
// resume == 0: certify the scan's candidates; resume == 1: take the pick
// the exact rescan produced for the signals listed in st.pending.
template <typename YT>
__global__ void __launch_bounds__(256, 3) ls_step_kernel(
    const YT *__restrict__ ys, const double *__restrict__ d64, const float *__restrict__ d32,
    const double *__restrict__ gram, int64_t p, int64_t t, int64_t n, int64_t n_pad,
    int64_t k_max, int64_t kw, int iter, double c_err, double dmax, TensorState st,
    int64_t *out_sel, double *out_coef, int64_t *out_count, int64_t *out_scans, int resume) {
  extern __shared__ double lsm[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ldl = (kw + 15) & ~int64_t(15);
  const int64_t per_warp = kw * ldl + 5 * kw + n;
  double *lin = lsm + wib * per_warp;  // L^{-1} rows (row-major)
  double *wv = lin + kw * ldl;         // w
  double *xv = wv + kw;                // x (current coefficients)
  double *gv = xv + kw;                // G[new, S]
  double *zv = gv + kw;                // z
  double *y = zv + kw;                 // the signal (fp64)
  const int64_t k = iter;              // atoms selected so far
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t count = resume ? (int64_t)st.npending[iter] : p;

  for (int64_t e = wid; e < count; e += nw) {
    const int64_t sig = resume ? st.pending[e] : e;
    if (!resume && (st.status[sig] & (ST_DONE | ST_DELEGATE))) continue;
    int64_t *sel = out_sel + sig * kw;  // global (written for the new atom)
    int64_t *ssel = (int64_t *)(y + n); // smem copy of the support ids
    // ---- independent loads first: signal, coefficients, z, support, L^{-1}, candidates
    int cidx = -1;
    float cval = -1.0f;
    if (!resume && lane < NCAND) {
      cidx = st.cand_idx[sig * NCAND + lane];
      cval = st.cand_val[sig * NCAND + lane];
    }
    const float cdrop = resume ? 0.0f : st.cand_drop[sig];
    const double rt = st.rt[sig], drs = st.dr[sig];
    const double rn2_prev = st.rn2[sig], tol_s = st.tol[sig], yy_s = st.yy[sig];
    for (int64_t i = lane; i < n; i += 32) y[i] = (double)ys[sig * n + i];
    for (int64_t i = lane; i < k; i += 32) {
      xv[i] = out_coef[sig * kw + i];
      zv[i] = st.z[sig * kw + i];
      ssel[i] = sel[i];
    }
    for (int64_t i = lane; i < k * ldl; i += 32) lin[i] = st.linv[sig * kw * ldl + i];
    __syncwarp();
    double best = -1.0, cbest = 0.0, bg0 = 0.0, bg1 = 0.0;
    int64_t bestj = -1;
    if (resume) {
      bestj = st.rs_j[sig];
      cbest = st.rs_c[sig];
      best = fabs(cbest);
      if (lane == 0) st.status[sig] &= ~ST_RESCAN;
      if (bestj >= 0) {
        const double *grow = gram + bestj * t;
        bg0 = lane < k ? __ldg(grow + ssel[lane]) : 0.0;
        bg1 = lane + 32 < k ? __ldg(grow + ssel[lane + 32]) : 0.0;
      }
    } else {
      // ---- candidates: drop taken atoms; rigorous bound E of the fp16 scan
      if (lane < NCAND) {
        for (int64_t i = 0; i < k && cidx >= 0; i++)
          if (ssel[i] == cidx) cidx = -1;
        if (cidx < 0) cval = -1.0f;
      }
      const double rq = st.rq[sig];  // E: rigorous bound of |c~ - <d, r>| (see c_err)
      const double vinv = pow2d(-scan_scale_exp(rn2_prev, yy_s)) * st.dinv;  // scan values carry both scales
      const double E = (c_err * (rt + rq) * 1.0079 + rq + drs) * dmax + st.emax * (rt + rq);
      double best_apx = (double)cval * vinv;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        best_apx = fmax(best_apx, __shfl_xor_sync(CDB_FULL_MASK, best_apx, o));
      const bool rescore = cidx >= 0 && (double)cval * vinv >= best_apx - 2.0 * E;
      const unsigned rmask = __ballot_sync(CDB_FULL_MASK, rescore);
      double unscored = rescore || cidx < 0 ? -1.0 : (double)cval * vinv;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        unscored = fmax(unscored, __shfl_xor_sync(CDB_FULL_MASK, unscored, o));
      unscored = fmax(unscored, (double)cdrop * vinv);
      for (unsigned m = rmask; m; m &= m - 1) {
        const int c = __ffs(m) - 1;
        const int64_t j = __shfl_sync(CDB_FULL_MASK, cidx, c);
        double g0, g1;
        const double cj = exact_corr(d64, gram, t, (int)n, j, y, ssel, xv, (int)k, lane, g0, g1);
        const double v = fabs(cj);
        if (v > best || (v == best && j < bestj)) {
          best = v;
          bestj = j;
          cbest = cj;
          bg0 = g0;
          bg1 = g1;
        }
      }
      if (bestj < 0 || !(unscored + E < best)) {
        // uncertifiable: queue for the CTA-wide exact rescan, resume later
        if (lane == 0) {
          st.status[sig] |= ST_RESCAN;
          st.pending[atomicAdd(st.npending + iter, 1)] = sig;
          atomicAdd(st.rescans, 1);
        }
        __syncwarp();
        continue;
      }
    }
    if (lane == 0) out_scans[sig] += t - k;  // scans += c - k (_kernels.py:91)
    if (bestj < 0 || best <= 0.0) {          // orthogonal break (_kernels.py:104)
      if (lane == 0) st.status[sig] |= ST_DONE;
      __syncwarp();
      continue;
    }
    ls_update(d64, d32, gram, sig, t, n, n_pad, k_max, kw, iter, dmax, st, sel, ssel, out_coef,
              out_count, bestj, cbest, lin, wv, xv, gv, zv, y, lane, bg0, bg1, rn2_prev, tol_s,
              yy_s);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- grouped LS step
// The LS step is bound by each signal's chain of dependent memory round trips,
// not by bandwidth, so throughput scales with signals in flight.  Here a warp
// runs NG = 32 / G signals, one per G-lane group (the signal stays in global
// memory; per-signal shared state is only L^{-1} and five k-vectors).  All
// warp-level primitives run on every lane (group-local reductions via
// width-G xor shuffles); per-group work is predicated by `act`, so groups in
// different states never diverge around a shuffle.  Same arithmetic as
// ls_step_kernel / ls_update.
template <int G>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(CDB_FULL_MASK, v, o);
  return v;
}
template <int G>
__device__ __forceinline__ double gmax(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(CDB_FULL_MASK, v, o));
  return v;
}

// YM > 0: N <= YM * G and every lane keeps its YM elements of y
// (i = gl + G m) in registers for both the re-score and the residual.
template <typename YT, int G, int YM = 0>
__global__ void __launch_bounds__(128, 6) ls_group_kernel(
    const YT *__restrict__ ys, const double *__restrict__ d64, const float *__restrict__ d32,
    const double *__restrict__ gram, int64_t p, int64_t t, int n, int64_t n_pad, int k_max,
    int kw, int iter, double c_err, double dmax, TensorState st, int64_t *out_sel,
    double *out_coef, int64_t *out_count, int64_t *out_scans, int resume, int split) {
  constexpr int NG = 32 / G;
  griddep_wait();  // the scan's candidates (PDL)
  griddep_launch();
  extern __shared__ double lsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gi = lane / G, gl = lane % G;
  const unsigned gbits = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (gi * G);
  const int ldl = (kw + 15) & ~15;  // L^{-1} row stride (see lsw)
  const int per_group = kw * ldl + 5 * kw;
  double *lin = lsm + (wib * NG + gi) * per_group;
  double *wv = lin + kw * ldl;
  double *xv = wv + kw;
  double *gv = xv + kw;
  double *zv = gv + kw;
  int64_t *ssel = (int64_t *)(zv + kw);
  const int k = iter;
  const int64_t slots = (int64_t)gridDim.x * (blockDim.x >> 5) * NG;
  const int64_t count = resume ? (int64_t)st.npending[iter] : p;

  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * NG; base < count;
       base += slots) {
    const int64_t e = base + gi;
    const bool valid = e < count;
    const int64_t sig = valid ? (resume ? st.pending[e] : e) : 0;
    bool act = valid && (resume || !(st.status[sig] & (ST_DONE | ST_DELEGATE)));
    int64_t *sel = out_sel + sig * kw;
    const YT *y = ys + sig * (int64_t)n;
    // ---- independent loads
    int cidx = -1;
    float cval = -1.0f;
    if (act && !resume && gl < NCAND) {
      cidx = st.cand_idx[sig * NCAND + gl];
      cval = st.cand_val[sig * NCAND + gl];
    }
    float cdrop = 0.0f;
    double rt = 0.0, drs = 0.0, rn2_prev = 0.0, tol = 0.0, yy = 1.0;
    if (act) {
      if (!resume) cdrop = st.cand_drop[sig];
      rt = st.rt[sig];
      drs = st.dr[sig];
      rn2_prev = st.rn2[sig];
      tol = st.tol[sig];
      yy = st.yy[sig];
      for (int i = gl; i < k; i += G) {
        xv[i] = out_coef[sig * kw + i];
        zv[i] = st.z[sig * kw + i];
        ssel[i] = sel[i];
      }
      for (int i = gl; i < k * ldl; i += G) lin[i] = st.linv[sig * kw * ldl + i];
    }
    YT yv[YM > 0 ? YM : 1];
    if constexpr (YM > 0) {
#pragma unroll
      for (int m = 0; m < YM; m++) {
        const int i = gl + G * m;
        yv[m] = act && i < n ? y[i] : (YT)0;
      }
    }
    __syncwarp();
    double best = -1.0, cbest = 0.0;
    int64_t bestj = -1;
    if (resume) {
      if (act) {
        bestj = st.rs_j[sig];
        cbest = st.rs_c[sig];
        best = fabs(cbest);
        if (gl == 0) st.status[sig] &= ~ST_RESCAN;
      }
    } else {
      // ---- candidates: drop taken atoms; rigorous bound E of the fp16 scan
      if (cidx >= 0) {
        for (int i = 0; i < k; i++)
          if (ssel[i] == cidx) cidx = -1;
        if (cidx < 0) cval = -1.0f;
      }
      const double rq = st.rq[sig];  // E: rigorous bound of |c~ - <d, r>| (see c_err)
      const double vinv = pow2d(-scan_scale_exp(rn2_prev, yy)) * st.dinv;  // scan values carry both scales
      const double E = (c_err * (rt + rq) * 1.0079 + rq + drs) * dmax + st.emax * (rt + rq);
      const double best_apx = gmax<G>((double)cval * vinv);
      const bool rescore = act && cidx >= 0 && (double)cval * vinv >= best_apx - 2.0 * E;
      const unsigned rm = (__ballot_sync(CDB_FULL_MASK, rescore) & gbits) >> (gi * G);
      double unsc = gmax<G>(rescore || cidx < 0 ? -1.0 : (double)cval * vinv);
      unsc = fmax(unsc, (double)cdrop * vinv);
      const int nre = __popc(rm);
      const int maxre = (int)__reduce_max_sync(CDB_FULL_MASK, (unsigned)nre);
      unsigned mm = rm;
      for (int r = 0; r < maxre; r++) {
        const int src = mm ? __ffs(mm) - 1 : 0;
        const bool on = mm != 0;
        if (mm) mm &= mm - 1;
        const int64_t j = __shfl_sync(CDB_FULL_MASK, (long long)cidx, gi * G + src);
        double acc = 0.0;
        if (on) {
          const double *dj = d64 + j * n;
          double a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int i = gl;
          if constexpr (YM > 0) {
#pragma unroll
            for (int m = 0; m < YM; m += 4) {  // y from registers, 4 atom loads in flight
              const int i0 = gl + G * m;
              const double d0 = i0 < n ? __ldg(dj + i0) : 0.0;
              const double d1 = i0 + G < n ? __ldg(dj + i0 + G) : 0.0;
              const double d2 = i0 + 2 * G < n ? __ldg(dj + i0 + 2 * G) : 0.0;
              const double d3 = i0 + 3 * G < n ? __ldg(dj + i0 + 3 * G) : 0.0;
              acc = fma(d0, (double)yv[m], acc);
              a1 = fma(d1, (double)yv[m + 1], a1);
              a2 = fma(d2, (double)yv[m + 2], a2);
              a3 = fma(d3, (double)yv[m + 3], a3);
            }
            i = n;
          }
          for (; i + 3 * G < n; i += 4 * G) {  // 8 loads in flight
            const double d0 = __ldg(dj + i), d1 = __ldg(dj + i + G), d2 = __ldg(dj + i + 2 * G),
                         d3 = __ldg(dj + i + 3 * G);
            const double y0 = (double)y[i], y1 = (double)y[i + G], y2 = (double)y[i + 2 * G],
                         y3 = (double)y[i + 3 * G];
            acc = fma(d0, y0, acc);
            a1 = fma(d1, y1, a1);
            a2 = fma(d2, y2, a2);
            a3 = fma(d3, y3, a3);
          }
          for (; i < n; i += G) acc = fma(__ldg(dj + i), (double)y[i], acc);
          acc += (a1 + a2) + a3;
          const double *gj = gram + j * t;
#pragma unroll 4
          for (int s2 = gl; s2 < k; s2 += G) acc = fma(-__ldg(gj + ssel[s2]), xv[s2], acc);
        }
        const double cj = gsum<G>(acc);
        if (on) {
          const double v = fabs(cj);
          if (v > best || (v == best && j < bestj)) {
            best = v;
            bestj = j;
            cbest = cj;
          }
        }
      }
      if (act && !(bestj >= 0 && unsc + E < best)) {
        // uncertifiable: queue for the CTA-wide exact rescan, resume later
        if (gl == 0) {
          st.status[sig] |= ST_RESCAN;
          st.pending[atomicAdd(st.npending + iter, 1)] = sig;
          atomicAdd(st.rescans, 1);
        }
        act = false;
      }
    }
    if (act && gl == 0) out_scans[sig] += t - k;  // scans += c - k (_kernels.py:91)
    if (act && (bestj < 0 || best <= 0.0)) {      // orthogonal break (_kernels.py:104)
      if (gl == 0) st.status[sig] |= ST_DONE;
      act = false;
    }
    // ---- Cholesky append through the Gram row of the new atom
    const double *grow = gram + (act ? bestj : 0) * t;
    if (act)
      for (int l = gl; l < k; l += G) gv[l] = __ldg(grow + ssel[l]);
    const double gnn = act ? __ldg(grow + bestj) : 1.0;
    __syncwarp();
    if (act)
      for (int l = gl; l < k; l += G) {
        double acc = 0.0;
        for (int i = 0; i <= l; i++) acc = fma(lin[lsw(l, i, ldl)], gv[i], acc);
        wv[l] = acc;
      }
    __syncwarp();
    double ww = 0.0;
    if (act)
      for (int l = gl; l < k; l += G) ww = fma(wv[l], wv[l], ww);
    ww = gsum<G>(ww);
    const double d2 = gnn - ww;
    if (act && !(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: exact engine
      if (gl == 0) st.status[sig] |= ST_DELEGATE;
      act = false;
    }
    const double inv_d = act ? 1.0 / sqrt(d2) : 0.0;
    const double zk = cbest * inv_d;  // q_k^T y = q_k^T r = <d_new, r> / d
    if (act) {
      for (int i = gl; i <= k; i += G) {
        double v;
        if (i == k) {
          v = inv_d;
        } else {
          double acc = 0.0;
          for (int l = i; l < k; l++) acc = fma(wv[l], lin[lsw(l, i, ldl)], acc);
          v = -acc * inv_d;
        }
        lin[lsw(k, i, ldl)] = v;
        st.linv[sig * kw * ldl + lsw(k, i, ldl)] = v;
      }
      if (gl == 0) {
        zv[k] = zk;
        st.z[sig * kw + k] = zk;
        sel[k] = bestj;
        ssel[k] = bestj;
      }
    }
    __syncwarp();
    const int kd = k + 1;
    if (act)
      for (int i = gl; i < kd; i += G) {
        double acc = 0.0;
        for (int l = i; l < kd; l++) acc = fma(lin[lsw(l, i, ldl)], zv[l], acc);
        xv[i] = acc;
        out_coef[sig * kw + i] = acc;
      }
    __syncwarp();
    // ---- stop test on |r|^2 = |y|^2 - |z|^2, exact residual inside the band
    const double rn2 = rn2_prev - zk * zk;
    const double gap = rn2 - tol * tol;
    const bool need_exact = act && !(fabs(gap) > 1e-12 * yy);
    bool stop = act && gap < 0.0;
    if (__any_sync(CDB_FULL_MASK, need_exact)) {
      double rr = 0.0;
      if (need_exact)
        for (int i = gl; i < n; i += G) {
          double ri = (double)y[i];
          for (int l = 0; l < kd; l++) ri = fma(-xv[l], __ldg(d64 + ssel[l] * n + i), ri);
          rr = fma(ri, ri, rr);
        }
      rr = gsum<G>(rr);
      if (need_exact) stop = sqrt(rr) <= tol;
    }
    if (act && gl == 0) {
      st.rn2[sig] = rn2;
      out_count[sig] = kd;
    }
    if (act && (stop || kd >= k_max)) {
      if (gl == 0) st.status[sig] |= ST_DONE;
      act = false;
    }
    // ---- next scan operand: r~ = y - D32_S x (fp64 accumulate) -> fp16
    //      (split mode: left to resid_split_kernel, flagged ST_RESID)
    double rr = 0.0, sx = 0.0, q2 = 0.0;
    if (act && !split) {
      const int e16 = scan_scale_exp(rn2, yy);
  const double s16 = pow2d(e16), inv16 = pow2d(-e16);
#pragma unroll
      for (int i0 = 0; i0 < (YM > 0 ? YM * G : n); i0 += 8 * G) {
        if (YM > 0 && i0 >= n) break;
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int i = i0 + u * G + gl;
          if constexpr (YM > 0)
            acc[u] = i < n ? (double)yv[i0 / G + u] : 0.0;
          else
            acc[u] = i < n ? (double)y[i] : 0.0;
        }
        int l = 0;
        for (; l + 3 < kd; l += 4) {  // 32 loads in flight before the FMAs
          float v[4][8];
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float *row = d32 + ssel[l + q] * n;
#pragma unroll
            for (int u = 0; u < 8; u++) {
              const int i = i0 + u * G + gl;
              v[q][u] = i < n ? __ldg(row + i) : 0.0f;
            }
          }
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const double xl = xv[l + q];
#pragma unroll
            for (int u = 0; u < 8; u++) acc[u] = fma(-xl, (double)v[q][u], acc[u]);
          }
        }
        for (; l < kd; l++) {
          const float *row = d32 + ssel[l] * n;
          const double xl = xv[l];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int i = i0 + u * G + gl;
            if (i < n) acc[u] = fma(-xl, (double)__ldg(row + i), acc[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int i = i0 + u * G + gl;
          if (i < n) {
            q2 += put_r16(st.r16 + sig * n_pad + i, acc[u], s16, inv16);
            rr = fma(acc[u], acc[u], rr);
          }
        }
      }
      for (int l = gl; l < kd; l += G) sx += fabs(xv[l]);
    }
    rr = gsum<G>(rr);
    sx = gsum<G>(sx);
    q2 = gsum<G>(q2);
    if (act && gl == 0) {
      if (split) {
        st.status[sig] |= ST_RESID;
      } else {
        st.rq[sig] = sqrt(q2) * (1.0 + 1e-12);
        st.rt[sig] = sqrt(rr);
        st.dr[sig] = 0x1p-24 * sx * dmax * 1.0000001;  // |(D64 - D32) x| bound
      }
      atomicAdd(st.active + iter, 1);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- wide LS step
// Long supports (kw > 32: cfg 4, K = 64) make L^{-1} too large to stage in
// shared memory (32 KB per signal left the grouped kernel 4 signals per SM,
// 5.4 ms per 111 k-signal launch on cfg 4 step 1).  Here one warp owns one
// signal and nothing per-signal is staged: L^{-1} stays in global memory as
// packed rows (row l holds l+1 entries at l(l+1)/2), read twice per
// iteration with coalesced row loads --
//   w = L^{-1} g      lanes own columns i, accumulate one partial per row,
//                     and a butterfly reduce-scatter (31 fp64 shuffles per
//                     32 rows) leaves lane l holding w_l;
//   v = L^{-T} w      lanes own columns i, rows l streamed with w_l broadcast,
// and the support's k-vectors (ids, coefficients, Gram row) live in
// registers, lane i holding entries i, i + 32, ...  The coefficients are
// updated in place, x_k = [x_{k-1}; 0] + z_k [-v / d; 1 / d] (the new row of
// L^{-1} is [-v^T / d, 1 / d]), so z never needs re-reading.  Certification,
// delegation, the stop rule and the scan counts are those of ls_step_kernel;
// the next scan operand is built by resid_split_kernel.
__device__ __forceinline__ int64_t lpk(int l) { return (int64_t)l * (l + 1) / 2; }


// 32 per-lane partials acc[m] (m = row within the block) -> lane l returns
// the warp-wide sum of partial l.
__device__ __forceinline__ double reduce_scatter32(double (&acc)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int m = 0; m < o; m++) {
      const double send = hi ? acc[m] : acc[m + o];
      const double keep = hi ? acc[m + o] : acc[m];
      acc[m] = keep + __shfl_xor_sync(CDB_FULL_MASK, send, o);
    }
  }
  return acc[0];
}

template <typename YT, int KR, int MB>
__global__ void __launch_bounds__(128, MB) ls_wide_kernel(
    const YT *__restrict__ ys, const double *__restrict__ d64, const double *__restrict__ gram,
    int64_t p, int64_t t, int n, int k_max, int kw, int iter, double c_err, double dmax,
    TensorState st, int64_t *out_sel, double *out_coef, int64_t *out_count, int64_t *out_scans,
    int resume) {
  griddep_wait();  // the scan's candidates (PDL)
  griddep_launch();
  __shared__ double wsm[4][32 * KR];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int k = iter;
  const int64_t kp = (int64_t)kw * (kw + 1) / 2;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t count = resume ? (int64_t)st.npending[iter] : p;
  double *wl = wsm[wib];

  for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; e < count; e += nw) {
    const int64_t sig = resume ? st.pending[e] : e;
    if (!resume && (st.status[sig] & (ST_DONE | ST_DELEGATE))) continue;
    int64_t *sel = out_sel + sig * kw;
    double *xo = out_coef + sig * kw;
    double *lin = st.linv + sig * kp;
    const YT *y = ys + sig * (int64_t)n;
    // the L^{-1} rows and the signal are needed only after the candidate
    // loads and the re-scores: start pulling them into L1 now
    {
      const char *lb = (const char *)lin;
      const int64_t lbytes = lpk(k) * 8;
      for (int64_t o = (int64_t)lane * 128; o < lbytes; o += 32 * 128)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(lb + o));
      const char *yb = (const char *)y;
      for (int64_t o = (int64_t)lane * 128; o < (int64_t)n * (int64_t)sizeof(YT); o += 32 * 128)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(yb + o));
    }
    int64_t sv[KR];
    double xv[KR];
#pragma unroll
    for (int r = 0; r < KR; r++) {
      const int i = lane + 32 * r;
      sv[r] = i < k ? sel[i] : -1;
      xv[r] = i < k ? xo[i] : 0.0;
    }
    int cidx = -1;
    float cval = -1.0f;
    if (!resume && lane < NCAND) {
      cidx = st.cand_idx[sig * NCAND + lane];
      cval = st.cand_val[sig * NCAND + lane];
    }
    const double rn2_prev = st.rn2[sig], tol = st.tol[sig], yy = st.yy[sig];
    double best = -1.0, cbest = 0.0;
    int64_t bestj = -1;
    double bg[KR], bgnn = 1.0;
#pragma unroll
    for (int r = 0; r < KR; r++) bg[r] = 0.0;
    if (resume) {
      bestj = st.rs_j[sig];
      cbest = st.rs_c[sig];
      best = fabs(cbest);
      if (lane == 0) st.status[sig] &= ~ST_RESCAN;
      if (bestj >= 0) {
        const double *grow = gram + bestj * t;
#pragma unroll
        for (int r = 0; r < KR; r++) bg[r] = sv[r] >= 0 ? __ldg(grow + sv[r]) : 0.0;
        bgnn = __ldg(grow + bestj);
      }
    } else {
      // ---- candidates: drop taken atoms (support ids are spread over the lanes)
#pragma unroll
      for (int c = 0; c < NCAND; c++) {
        const int j = __shfl_sync(CDB_FULL_MASK, cidx, c);
        bool hit = false;
#pragma unroll
        for (int r = 0; r < KR; r++) hit |= (j >= 0 && sv[r] == j);
        if (__any_sync(CDB_FULL_MASK, hit) && lane == c) {
          cidx = -1;
          cval = -1.0f;
        }
      }
      const float cdrop = st.cand_drop[sig];
      const double rt = st.rt[sig], drs = st.dr[sig], rq = st.rq[sig];
      const double vinv = pow2d(-scan_scale_exp(rn2_prev, yy)) * st.dinv;  // scan values carry both scales
      const double E = (c_err * (rt + rq) * 1.0079 + rq + drs) * dmax + st.emax * (rt + rq);
      double best_apx = (double)cval * vinv;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        best_apx = fmax(best_apx, __shfl_xor_sync(CDB_FULL_MASK, best_apx, o));
      const bool rescore = cidx >= 0 && (double)cval * vinv >= best_apx - 2.0 * E;
      const unsigned rmask = __ballot_sync(CDB_FULL_MASK, rescore);
      double unscored = rescore || cidx < 0 ? -1.0 : (double)cval * vinv;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        unscored = fmax(unscored, __shfl_xor_sync(CDB_FULL_MASK, unscored, o));
      unscored = fmax(unscored, (double)cdrop * vinv);
      for (unsigned m = rmask; m; m &= m - 1) {
        const int64_t j = __shfl_sync(CDB_FULL_MASK, cidx, __ffs(m) - 1);
        // exact c_j = <d_j, y> - G[j, S] x  (fp64)
        const double *dj = d64 + j * n;
        const double *gj = gram + j * t;
        double g[KR];
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int r = 0; r < KR; r++) g[r] = sv[r] >= 0 ? __ldg(gj + sv[r]) : 0.0;
        const double gjj = __ldg(gj + j);
        int i = lane;
        if (n == 512) {  // cfg 4 step 1: all 16 atom loads of a lane in flight at once
          double e[16];
#pragma unroll
          for (int q = 0; q < 16; q++) e[q] = __ldg(dj + lane + 32 * q);
#pragma unroll
          for (int q = 0; q < 16; q += 4) {
            a0 = fma(e[q], (double)y[lane + 32 * q], a0);
            a1 = fma(e[q + 1], (double)y[lane + 32 * (q + 1)], a1);
            a2 = fma(e[q + 2], (double)y[lane + 32 * (q + 2)], a2);
            a3 = fma(e[q + 3], (double)y[lane + 32 * (q + 3)], a3);
          }
          i = n;
        }
        for (; i + 96 < n; i += 128) {
          const double e0 = __ldg(dj + i), e1 = __ldg(dj + i + 32), e2 = __ldg(dj + i + 64),
                       e3 = __ldg(dj + i + 96);
          a0 = fma(e0, (double)y[i], a0);
          a1 = fma(e1, (double)y[i + 32], a1);
          a2 = fma(e2, (double)y[i + 64], a2);
          a3 = fma(e3, (double)y[i + 96], a3);
        }
        for (; i < n; i += 32) a0 = fma(__ldg(dj + i), (double)y[i], a0);
        double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
        for (int r = 0; r < KR; r++) acc = fma(-g[r], xv[r], acc);
        const double cj = warp_sum(acc);
        const double v = fabs(cj);
        if (v > best || (v == best && j < bestj)) {
          best = v;
          bestj = j;
          cbest = cj;
          bgnn = gjj;
#pragma unroll
          for (int r = 0; r < KR; r++) bg[r] = g[r];
        }
      }
      if (bestj < 0 || !(unscored + E < best)) {
        // uncertifiable: queue for the exact rescan, resume later
        if (lane == 0) {
          st.status[sig] |= ST_RESCAN;
          st.pending[atomicAdd(st.npending + iter, 1)] = sig;
          atomicAdd(st.rescans, 1);
        }
        continue;
      }
    }
    if (lane == 0) out_scans[sig] += t - k;  // scans += c - k (_kernels.py:91)
    if (bestj < 0 || best <= 0.0) {          // orthogonal break (_kernels.py:104)
      if (lane == 0) st.status[sig] |= ST_DONE;
      continue;
    }
    // ---- w = L^{-1} g   (g = G[S, new]; lane-owned columns, reduce-scatter per 32 rows)
    double w[KR];
#pragma unroll
    for (int b = 0; b < KR; b++) {
      w[b] = 0.0;
      if (32 * b >= k) continue;  // warp-uniform
      double acc[32];
#pragma unroll
      for (int m = 0; m < 32; m++) {
        const int l = 32 * b + m;
        double a = 0.0;
        if (l < k) {
          const double *row = lin + lpk(l);
#pragma unroll
          for (int r = 0; r <= b; r++) {
            const int i = lane + 32 * r;
            if (i <= l) a = fma(row[i], bg[r], a);
          }
        }
        acc[m] = a;
      }
      w[b] = reduce_scatter32(acc, lane);
      wl[32 * b + lane] = w[b];
    }
    __syncwarp();
    double ww = 0.0;
#pragma unroll
    for (int b = 0; b < KR; b++)
      if (lane + 32 * b < k) ww = fma(w[b], w[b], ww);
    ww = warp_sum(ww);
    const double gnn = bgnn;
    const double d2 = gnn - ww;
    if (!(d2 > GRAM_DELEGATE_D2 * gnn)) {  // near rank deficiency: the exact engine decides
      if (lane == 0) st.status[sig] |= ST_DELEGATE;
      __syncwarp();
      continue;
    }
    const double inv_d = 1.0 / sqrt(d2);
    const double zk = cbest * inv_d;  // q_k^T y = q_k^T r = <d_new, r> / d
    // ---- v = L^{-T} w (rows streamed, w_l broadcast from shared memory)
    double v[KR];
#pragma unroll
    for (int r = 0; r < KR; r++) v[r] = 0.0;
    int l = 0;
    for (; l + 3 < k; l += 4) {
      const double w0 = wl[l], w1 = wl[l + 1], w2 = wl[l + 2], w3 = wl[l + 3];
      const double *r0 = lin + lpk(l);
#pragma unroll
      for (int r = 0; r < KR; r++) {
        const int i = lane + 32 * r;
        const double *rw = r0;
        if (i <= l) v[r] = fma(rw[i], w0, v[r]);
        rw += l + 1;
        if (i <= l + 1) v[r] = fma(rw[i], w1, v[r]);
        rw += l + 2;
        if (i <= l + 2) v[r] = fma(rw[i], w2, v[r]);
        rw += l + 3;
        if (i <= l + 3) v[r] = fma(rw[i], w3, v[r]);
      }
    }
    for (; l < k; l++) {
      const double wv = wl[l];
      const double *rw = lin + lpk(l);
#pragma unroll
      for (int r = 0; r < KR; r++) {
        const int i = lane + 32 * r;
        if (i <= l) v[r] = fma(rw[i], wv, v[r]);
      }
    }
    // ---- append row k of L^{-1}, update x, record the pick
    double *nrow = lin + lpk(k);
#pragma unroll
    for (int r = 0; r < KR; r++) {
      const int i = lane + 32 * r;
      if (i < k) {
        const double u = -v[r] * inv_d;
        nrow[i] = u;
        xv[r] = fma(zk, u, xv[r]);
        xo[i] = xv[r];
      } else if (i == k) {
        nrow[i] = inv_d;
        xv[r] = zk * inv_d;
        xo[i] = xv[r];
        sv[r] = bestj;
        sel[i] = bestj;
      }
    }
    if (lane == 0) st.z[sig * kw + k] = zk;
    const int kd = k + 1;
    // ---- stop test on |r|^2 = |y|^2 - |z|^2, exact residual inside the band
    const double rn2 = rn2_prev - zk * zk;
    const double gap = rn2 - tol * tol;
    bool stop = gap < 0.0;
    if (!(fabs(gap) > 1e-12 * yy)) {
      __syncwarp();  // x and the ids written above by the other lanes
      double rr = 0.0;
      for (int i = lane; i < n; i += 32) {
        double ri = (double)y[i];
        for (int s = 0; s < kd; s++) ri = fma(-xo[s], __ldg(d64 + sel[s] * n + i), ri);
        rr = fma(ri, ri, rr);
      }
      stop = sqrt(warp_sum(rr)) <= tol;
    }
    if (lane == 0) {
      st.rn2[sig] = rn2;
      out_count[sig] = kd;
      if (stop || kd >= k_max) {
        st.status[sig] |= ST_DONE;
      } else {
        st.status[sig] |= ST_RESID;
        atomicAdd(st.active + iter, 1);
      }
    }
    __syncwarp();
  }
}

// Split-mode scan operand (large N): r~ = y - D32_S x -> fp16 for every signal
// flagged ST_RESID, one CTA per signal -- 8 elements x 4 atom rows = 32 loads
// in flight per thread, so the kd x N fp32 row stream runs near HBM speed
// instead of at the LS kernel's occupancy (its per-signal L^{-1} state allows
// only a few signals per SM).  Same arithmetic as the fused path.
template <typename YT, int BT>
__global__ void __launch_bounds__(BT) resid_split_kernel(const YT *__restrict__ ys,
                                                          const float *__restrict__ d32, int64_t p,
                                                          int64_t n, int64_t n_pad, int64_t kw,
                                                          double dmax, TensorState st,
                                                          const int64_t *out_sel,
                                                          const double *out_coef,
                                                          const int64_t *out_count) {
  extern __shared__ double xsm[];
  double *xv = xsm;                         // kw
  int64_t *ssel = (int64_t *)(xv + kw);     // kw
  __shared__ double red[3][BT / 32];
  __shared__ int e16s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the next signal's status, count and code entries (thread l < kw) are
  // loaded one signal ahead (resid_f32_kernel: 12% on cfg 4 step 1)
  auto meta = [&](int64_t s, uint32_t &stt, int &kd, double &x, int64_t &sel) {
    stt = s < p ? st.status[s] : 0u;
    kd = s < p ? (int)out_count[s] : 0;
    x = s < p && tid < kw ? out_coef[s * kw + tid] : 0.0;
    sel = s < p && tid < kw ? out_sel[s * kw + tid] : 0;
  };
  uint32_t n_st;
  int n_kd;
  double n_x;
  int64_t n_sel;
  meta(blockIdx.x, n_st, n_kd, n_x, n_sel);
  for (int64_t sig = blockIdx.x; sig < p; sig += gridDim.x) {
    const uint32_t c_st = n_st;
    const int kd = n_kd;
    const double cx = n_x;
    const int64_t csel = n_sel;
    meta(sig + gridDim.x, n_st, n_kd, n_x, n_sel);
    if (!(c_st & ST_RESID)) continue;  // uniform across the CTA
    for (int l = tid; l < kd; l += BT) {  // entry tid prefetched; l >= BT only if kw > BT
      xv[l] = l == tid ? cx : out_coef[sig * kw + l];
      ssel[l] = l == tid ? csel : out_sel[sig * kw + l];
    }
    // the operand's scale exponent waits in shared memory: nothing of it is
    // live across the register-tight row loop
    if (tid == 0) e16s = scan_scale_exp(st.rn2[sig], st.yy[sig]);
    __syncthreads();
    const YT *y = ys + sig * n;
    double rr = 0.0, q2 = 0.0;
    for (int64_t i0 = 0; i0 < n; i0 += 8 * BT) {
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int64_t i = i0 + u * BT + tid;
        acc[u] = i < n ? (double)y[i] : 0.0;
      }
      int l = 0;
      for (; l + 3 < kd; l += 4) {
        float v[4][8];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const float *row = d32 + ssel[l + q] * n;
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int64_t i = i0 + u * BT + tid;
            v[q][u] = i < n ? __ldg(row + i) : 0.0f;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const double xl = xv[l + q];
#pragma unroll
          for (int u = 0; u < 8; u++) acc[u] = fma(-xl, (double)v[q][u], acc[u]);
        }
      }
      for (; l < kd; l++) {
        const float *row = d32 + ssel[l] * n;
        const double xl = xv[l];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int64_t i = i0 + u * BT + tid;
          if (i < n) acc[u] = fma(-xl, (double)__ldg(row + i), acc[u]);
        }
      }
      const int e16 = e16s;
      const double s16 = pow2d(e16), inv16 = pow2d(-e16);
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int64_t i = i0 + u * BT + tid;
        if (i < n) {
          q2 += put_r16(st.r16 + sig * n_pad + i, acc[u], s16, inv16);
          rr = fma(acc[u], acc[u], rr);
        }
      }
    }
    double sx = 0.0;
    for (int l = tid; l < kd; l += blockDim.x) sx += fabs(xv[l]);
    rr = warp_sum(rr);
    sx = warp_sum(sx);
    q2 = warp_sum(q2);
    if (lane == 0) {
      red[0][warp] = rr;
      red[1][warp] = sx;
      red[2][warp] = q2;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0, c = 0.0;
      for (int w = 0; w < BT / 32; w++) {
        a += red[0][w];
        b += red[1][w];
        c += red[2][w];
      }
      st.rq[sig] = sqrt(c) * (1.0 + 1e-12);
      st.rt[sig] = sqrt(a);
      st.dr[sig] = 0x1p-24 * b * dmax * 1.0000001;  // |(D64 - D32) x| bound
      st.status[sig] &= ~ST_RESID;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ float4 ldg_nc_f4(const float4 *p) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Split-mode scan operand for long rows (N = 1024 J <= 4096: cfg 4 full OMP),
// the row stream on the bulk-copy engine: one producer lane walks the same
// signal list as the consumers and keeps a ring of RB_S whole fp32 atom rows
// (4 N bytes each) in flight with 1-D cp.async.bulk copies that complete on
// mbarriers, so the bytes in flight per SM (2 CTAs x RB_S x 16 KB) no longer
// depend on registers; 256 consumer threads read each landed row from shared
// memory (16-byte, conflict-free) and run the same fp64 FMA chain in the same
// order as resid_split_kernel -- bit-identical operands and bounds.  The
// producer runs ahead across signal boundaries: the next signal's rows land
// while the consumers convert and store the current operand.
constexpr int RB_T = 256;  // consumer threads
constexpr int RB_S = 6;    // ring stages
template <typename YT, int J>
__global__ void __launch_bounds__(RB_T + 32) resid_bulk_kernel(
    const YT *__restrict__ ys, const float *__restrict__ d32, int64_t p, int64_t n, int64_t n_pad,
    int64_t kw, double dmax, TensorState st, const int64_t *out_sel, const double *out_coef,
    const int64_t *out_count) {
  extern __shared__ __align__(128) unsigned char rbsm[];
  float *ring = (float *)rbsm;                                  // RB_S x n
  double *xv = (double *)(rbsm + (size_t)RB_S * n * 4);         // kw
  uint64_t *full = (uint64_t *)(xv + kw), *empty = full + RB_S;  // RB_S each
  __shared__ double red[3][RB_T / 32];
  __shared__ int e16s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < RB_S; s++) {
      sm100::mbar_init(full + s, 1);
      sm100::mbar_init(empty + s, RB_T / 32);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t row_bytes = (uint32_t)(n * 4);
  uint32_t cnt = 0;  // rows issued (producer) / consumed (consumers): same sequence
  if (warp == RB_T / 32) {
    // ---- producer warp (lane 0 issues; all lanes hold the support ids)
    for (int64_t sig = blockIdx.x; sig < p; sig += gridDim.x) {
      if (!(st.status[sig] & ST_RESID)) continue;
      const int kd = (int)out_count[sig];
      const int64_t id0 = lane < kd ? out_sel[sig * kw + lane] : 0;
      const int64_t id1 = lane + 32 < kd ? out_sel[sig * kw + lane + 32] : 0;
      for (int l = 0; l < kd; l++, cnt++) {
        const int64_t id = __shfl_sync(CDB_FULL_MASK, l < 32 ? id0 : id1, l & 31);
        if (lane == 0) {
          const uint32_t stage = cnt % RB_S;
          sm100::mbar_wait(empty + stage, ((cnt / RB_S) & 1) ^ 1);
          sm100::mbar_expect_tx(full + stage, row_bytes);
          sm100::bulk_load(ring + (size_t)stage * n, d32 + id * n, row_bytes, full + stage);
        }
      }
    }
    return;
  }
  // ---- consumers
  for (int64_t sig = blockIdx.x; sig < p; sig += gridDim.x) {
    if (!(st.status[sig] & ST_RESID)) continue;  // uniform across the CTA
    const int kd = (int)out_count[sig];
    asm volatile("bar.sync 1, %0;" ::"n"(RB_T) : "memory");  // the previous signal's xv is consumed
    double sx = 0.0;
    if (tid < kd) {
      const double c = out_coef[sig * kw + tid];
      xv[tid] = c;
      sx = fabs(c);
    }
    if (tid == 0) e16s = scan_scale_exp(st.rn2[sig], st.yy[sig]);
    asm volatile("bar.sync 1, %0;" ::"n"(RB_T) : "memory");
    const YT *y = ys + sig * n;
    double acc[J][4];
#pragma unroll
    for (int j = 0; j < J; j++) {
      const int64_t i = 4 * (tid + (int64_t)RB_T * j);
      if constexpr (sizeof(YT) == 4) {
        const float4 v = *(const float4 *)(y + i);
        acc[j][0] = (double)v.x, acc[j][1] = (double)v.y, acc[j][2] = (double)v.z,
        acc[j][3] = (double)v.w;
      } else {
        const double2 a = *(const double2 *)(y + i), b = *(const double2 *)(y + i + 2);
        acc[j][0] = (double)a.x, acc[j][1] = (double)a.y, acc[j][2] = (double)b.x,
        acc[j][3] = (double)b.y;
      }
    }
    for (int l = 0; l < kd; l++, cnt++) {
      const uint32_t stage = cnt % RB_S;
      sm100::mbar_wait(full + stage, (cnt / RB_S) & 1);
      const double xl = -xv[l];
      const float4 *row = (const float4 *)(ring + (size_t)stage * n) + tid;
      float4 v[J];
#pragma unroll
      for (int j = 0; j < J; j++) v[j] = row[RB_T * j];
#pragma unroll
      for (int j = 0; j < J; j++) {
        acc[j][0] = fma(xl, (double)v[j].x, acc[j][0]);
        acc[j][1] = fma(xl, (double)v[j].y, acc[j][1]);
        acc[j][2] = fma(xl, (double)v[j].z, acc[j][2]);
        acc[j][3] = fma(xl, (double)v[j].w, acc[j][3]);
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(empty + stage);
    }
    // ---- fp16(s r~) with its exact rounding error, |r~|^2
    const int e16 = e16s;
    const double s16 = pow2d(e16), inv16 = pow2d(-e16);
    double rr = 0.0, q2 = 0.0;
#pragma unroll
    for (int j = 0; j < J; j++) {
      __half b[4];
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const double a = acc[j][c];
        b[c] = __float2half_rn((float)(a * s16));
        const double e = (double)__half2float(b[c]) * inv16 - a;
        q2 = fma(e, e, q2);
        rr = fma(a, a, rr);
      }
      __half2 lo, hi;
      lo.x = b[0], lo.y = b[1], hi.x = b[2], hi.y = b[3];
      uint2 pk;
      pk.x = *(uint32_t *)&lo;
      pk.y = *(uint32_t *)&hi;
      *(uint2 *)(st.r16 + sig * n_pad + 4 * (tid + (int64_t)RB_T * j)) = pk;
    }
    rr = warp_sum(rr);
    sx = warp_sum(sx);
    q2 = warp_sum(q2);
    if (lane == 0) {
      red[0][warp] = rr;
      red[1][warp] = sx;
      red[2][warp] = q2;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(RB_T) : "memory");
    if (tid == 0) {
      double a = 0.0, b = 0.0, c = 0.0;
      for (int w = 0; w < RB_T / 32; w++) {
        a += red[0][w];
        b += red[1][w];
        c += red[2][w];
      }
      st.rq[sig] = sqrt(c) * (1.0 + 1e-12);
      st.rt[sig] = sqrt(a);
      st.dr[sig] = 0x1p-24 * b * dmax * 1.0000001;  // |(D64 - D32) x| bound
      st.status[sig] &= ~ST_RESID;
    }
  }
}

// fp32 split-mode scan operand: the same r~ = y - D32_S x, accumulated in
// fp32 with 16-byte loads (V float4 per thread per atom row, 8 rows in
// flight), packed fp16 stores.  The scan's error budget charges the fp32
// arithmetic exactly (dr below): with u = 2^-24 and g = (k+1) u / (1 - (k+1) u)
// the FMA chain y32 - sum_l x32_l d32_l has |r~ - r| <= |y32 - y| +
// sum_l |x32_l d32_l - x_l d_l| + g (|y32| + sum_l |x32_l| |d32_l|), so
//   |r~ - r| <= (u + g (1 + u)) |y| + (2.0001 u + g (1 + u)^2) sum_l |x_l| dmax.
// Needs n == 4 * BT * V.
template <typename YT, int BT, int V, int G>
__global__ void __launch_bounds__(BT) resid_f32_kernel(const YT *__restrict__ ys,
                                                        const float *__restrict__ d32, int64_t p,
                                                        int64_t n, int64_t n_pad, int64_t kw,
                                                        double dmax, TensorState st,
                                                        const int64_t *out_sel,
                                                        const double *out_coef,
                                                        const int64_t *out_count) {
  extern __shared__ double xsm[];
  float *xf = (float *)xsm;                         // kw fp32 coefficients
  const float **rows = (const float **)(xsm + kw);  // kw row pointers
  __shared__ double red[3][BT / 32];
  __shared__ int e16s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the next signal's status, count and (thread l < kw) code entry are loaded
  // one signal ahead, so a signal starts without three dependent round trips
  auto meta = [&](int64_t s, uint32_t &stt, int &kd, double &x, int64_t &sel) {
    stt = s < p ? st.status[s] : 0u;
    kd = s < p ? (int)out_count[s] : 0;
    x = s < p && tid < kw ? out_coef[s * kw + tid] : 0.0;
    sel = s < p && tid < kw ? out_sel[s * kw + tid] : 0;
  };
  uint32_t n_st;
  int n_kd;
  double n_x;
  int64_t n_sel;
  meta(blockIdx.x, n_st, n_kd, n_x, n_sel);
  for (int64_t sig = blockIdx.x; sig < p; sig += gridDim.x) {
    const uint32_t c_st = n_st;
    const int kd = n_kd;
    const double cx = n_x;
    const int64_t csel = n_sel;
    meta(sig + gridDim.x, n_st, n_kd, n_x, n_sel);
    if (!(c_st & ST_RESID)) continue;  // uniform across the CTA
    double sx = 0.0;
    if (tid < kd) {  // kw <= BT (64 or 128 threads, K <= 64)
      xf[tid] = (float)cx;
      rows[tid] = d32 + csel * n;
      sx = fabs(cx);
    }
    sx = warp_sum(sx);
    if (lane == 0) red[1][warp] = sx;
    if (tid == 0) e16s = scan_scale_exp(st.rn2[sig], st.yy[sig]);  // read after the row loop
    __syncthreads();
    float4 acc[V];
    const YT *y = ys + sig * n;
#pragma unroll
    for (int v = 0; v < V; v++) {
      const int64_t i = 4 * (tid + (int64_t)v * BT);
      acc[v] = make_float4((float)y[i], (float)y[i + 1], (float)y[i + 2], (float)y[i + 3]);
    }
    // software-pipelined over groups of G rows: the next group's loads are
    // issued before the current group's FMAs (G * V 16-byte loads in flight)
    int l = 0;
    if (kd >= G) {
      float4 cur[G][V];
#pragma unroll
      for (int q = 0; q < G; q++)
#pragma unroll
        for (int v = 0; v < V; v++) cur[q][v] = ldg_nc_f4((const float4 *)rows[q] + tid + v * BT);
      for (; l + G - 1 < kd; l += G) {
        float4 nxt[G][V];
        const bool more = l + 2 * G - 1 < kd;
        if (more) {
#pragma unroll
          for (int q = 0; q < G; q++)
#pragma unroll
            for (int v = 0; v < V; v++)
              nxt[q][v] = ldg_nc_f4((const float4 *)rows[l + G + q] + tid + v * BT);
        }
#pragma unroll
        for (int q = 0; q < G; q++) {
          const float xl = -xf[l + q];
#pragma unroll
          for (int v = 0; v < V; v++) {
            acc[v].x = fmaf(xl, cur[q][v].x, acc[v].x);
            acc[v].y = fmaf(xl, cur[q][v].y, acc[v].y);
            acc[v].z = fmaf(xl, cur[q][v].z, acc[v].z);
            acc[v].w = fmaf(xl, cur[q][v].w, acc[v].w);
          }
        }
        if (more) {
#pragma unroll
          for (int q = 0; q < G; q++)
#pragma unroll
            for (int v = 0; v < V; v++) cur[q][v] = nxt[q][v];
        }
      }
    }
    for (; l < kd; l++) {
      const float xl = -xf[l];
#pragma unroll
      for (int v = 0; v < V; v++) {
        const float4 t = __ldg((const float4 *)rows[l] + tid + v * BT);
        acc[v].x = fmaf(xl, t.x, acc[v].x);
        acc[v].y = fmaf(xl, t.y, acc[v].y);
        acc[v].z = fmaf(xl, t.z, acc[v].z);
        acc[v].w = fmaf(xl, t.w, acc[v].w);
      }
    }
    float rr = 0.0f, q2 = 0.0f;
    const int e16 = e16s;
    const float s16 = pow2f(e16), inv16 = pow2f(-e16);
#pragma unroll
    for (int v = 0; v < V; v++) {
      const float e[4] = {acc[v].x, acc[v].y, acc[v].z, acc[v].w};
      __half b[4];
#pragma unroll
      for (int c = 0; c < 4; c++) {
        b[c] = __float2half_rn(e[c] * s16);
        const float d = __half2float(b[c]) * inv16 - e[c];  // exact in fp32
        q2 = fmaf(d, d, q2);
        rr = fmaf(e[c], e[c], rr);
      }
      __half2 lo, hi;
      lo.x = b[0];
      lo.y = b[1];
      hi.x = b[2];
      hi.y = b[3];
      uint2 pk;
      pk.x = *(uint32_t *)&lo;
      pk.y = *(uint32_t *)&hi;
      *(uint2 *)(st.r16 + sig * n_pad + 4 * (tid + (int64_t)v * BT)) = pk;
    }
    const double rrd = warp_sum((double)rr), q2d = warp_sum((double)q2);
    if (lane == 0) {
      red[0][warp] = rrd;
      red[2][warp] = q2d;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0, c = 0.0;
      for (int w = 0; w < BT / 32; w++) {
        a += red[0][w];
        b += red[1][w];
        c += red[2][w];
      }
      // fp32 sums of n squares: relative error <= n u; margins 2^-10 cover n <= 2^14
      st.rq[sig] = sqrt(c) * (1.0 + 0x1p-10);
      st.rt[sig] = sqrt(a) * (1.0 + 0x1p-10);
      const double u = 0x1p-24, g = (kd + 1) * u / (1.0 - (kd + 1) * u);
      st.dr[sig] = (u + g * (1.0 + u)) * sqrt(st.yy[sig]) * 1.0000001 +
                   (2.0001 * u + g * (1.0 + u) * (1.0 + u)) * b * dmax * 1.0000001;
      st.status[sig] &= ~ST_RESID;
    }
    __syncthreads();
  }
}

// Exact fp64 argmax over every non-taken atom for the queued signals.  The
// queue is cut into groups of RG signals and the atoms into parts; one CTA
// work item = (group, part): it materialises the RG exact residuals
// r = y - D64_S x and their taken-atom masks in shared memory, then streams
// its slice of the fp64 dictionary once for the whole group (each row feeds
// RG residuals, so the L2 / HBM traffic is 1/RG of a per-signal scan).  A
// warp pass covers 32/RG rows, i.e. 32 accumulators per lane, folded by a
// butterfly reduce-scatter (31 shuffles) that leaves lane l the sum of
// accumulator l.  Each part publishes (|c|, j, c) per signal; the last part of
// a group to finish reduces the partials (max |c|, lowest index on ties) into
// rs_j / rs_c.  The part count is chosen on the device from the queue length
// so that even a handful of queued signals fills the grid.
constexpr int RS_SPLIT = 16;  // partial slots per signal (buffer sizing)

template <int NV>
__device__ __forceinline__ double fold_lanes(double (&v)[NV], int lane) {
#pragma unroll
  for (int off = NV / 2; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int h = 0; h < off; h++) {
      const double send = up ? v[h] : v[h + off];
      const double keep = up ? v[h + off] : v[h];
      v[h] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

template <typename YT, int RG>
__global__ void __launch_bounds__(512) rescan_kernel(const YT *__restrict__ ys,
                                                     const double *__restrict__ d64, int64_t p,
                                                     int64_t t, int64_t n, int64_t kw, int iter,
                                                     TensorState st, const int64_t *out_sel,
                                                     const double *out_coef) {
  constexpr int ROWS = 32 / RG;
  constexpr int NW = 16;
  extern __shared__ double rsm[];
  __shared__ double sv[NW][RG];
  __shared__ int64_t sj[NW][RG];
  __shared__ double sc[NW][RG];
  __shared__ int last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t count = st.npending[iter];
  if (count == 0) return;
  const int64_t tw = (t + 31) / 32;
  double *r = rsm;                                     // RG x n
  double *x = r + RG * n;                              // RG x kw
  int64_t *sel = (int64_t *)(x + RG * kw);             // RG x kw
  uint32_t *taken = (uint32_t *)(sel + RG * kw);       // RG x tw
  const int64_t groups = (count + RG - 1) / RG;
  int64_t nparts = (2 * (int64_t)gridDim.x + groups - 1) / groups;
  if (nparts < 16) nparts = 16;
  if (nparts > (t + 63) / 64) nparts = (t + 63) / 64;
  if (nparts > p * RS_SPLIT / count) nparts = p * RS_SPLIT / count;
  if (nparts < 1) nparts = 1;
  const int64_t per = (t + nparts - 1) / nparts;
  const int64_t k = iter;
  for (int64_t w = blockIdx.x; w < groups * nparts; w += gridDim.x) {
    const int64_t g = w / nparts, part = w % nparts;
    const int64_t e0 = g * RG;
    const int ng = (int)(count - e0 < RG ? count - e0 : RG);
    for (int64_t i = threadIdx.x; i < RG * tw; i += blockDim.x) taken[i] = 0u;
    for (int64_t i = threadIdx.x; i < RG * kw; i += blockDim.x) {
      const int s = (int)(i / kw);
      const int64_t l = i % kw;
      const bool ok = s < ng && l < k;
      const int64_t sig = ok ? st.pending[e0 + s] : 0;
      x[i] = ok ? out_coef[sig * kw + l] : 0.0;
      sel[i] = ok ? out_sel[sig * kw + l] : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ng * (int)k; i += blockDim.x) {
      const int s = i / (int)k;
      const int64_t j = sel[s * kw + i % (int)k];
      atomicOr(&taken[s * tw + (j >> 5)], 1u << (j & 31));
    }
    // r_s = y_s - D64_S x_s, exact fp64 (zero for the unused group slots)
    for (int64_t i = threadIdx.x; i < RG * n; i += blockDim.x) {
      const int s = (int)(i / n);
      const int64_t c = i % n;
      double ri = 0.0;
      if (s < ng) {
        const int64_t sig = st.pending[e0 + s];
        ri = (double)ys[sig * n + c];
        for (int64_t l = 0; l < k; l++)
          ri = fma(-x[s * kw + l], __ldg(d64 + sel[s * kw + l] * n + c), ri);
      }
      r[i] = ri;
    }
    __syncthreads();
    const int64_t jlo = part * per, jhi = jlo + per < t ? jlo + per : t;
    double best = -1.0, cbest = 0.0;
    int64_t bestj = -1;
    const int my_s = lane % RG, my_row = lane / RG;
    for (int64_t j0 = jlo + (int64_t)warp * ROWS; j0 < jhi; j0 += NW * ROWS) {
      const double *rows[ROWS];
#pragma unroll
      for (int q = 0; q < ROWS; q++) rows[q] = d64 + (j0 + q < jhi ? j0 + q : jlo) * n;
      double acc[32];
#pragma unroll
      for (int q = 0; q < 32; q++) acc[q] = 0.0;
#pragma unroll(RG == 8 ? 2 : 1)
      for (int64_t i = lane; i < n; i += 32) {
        double dv[ROWS], rv[RG];
#pragma unroll
        for (int q = 0; q < ROWS; q++) dv[q] = __ldg(rows[q] + i);
#pragma unroll
        for (int s = 0; s < RG; s++) rv[s] = r[s * n + i];
#pragma unroll
        for (int q = 0; q < ROWS; q++)
#pragma unroll
          for (int s = 0; s < RG; s++) acc[q * RG + s] = fma(dv[q], rv[s], acc[q * RG + s]);
      }
      const double cj = fold_lanes<32>(acc, lane);
      const int64_t j = j0 + my_row;
      if (my_s < ng && j < jhi && !((taken[my_s * tw + (j >> 5)] >> (j & 31)) & 1u)) {
        const double v = fabs(cj);
        if (v > best || (v == best && j < bestj)) {
          best = v;
          bestj = j;
          cbest = cj;
        }
      }
    }
    // lanes sharing my_s: lane ^ RG, ^ 2RG, ...
#pragma unroll
    for (int off = RG; off < 32; off <<= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int64_t oj = __shfl_xor_sync(0xffffffffu, bestj, off);
      const double oc = __shfl_xor_sync(0xffffffffu, cbest, off);
      if (oj >= 0 && (bestj < 0 || ov > best || (ov == best && oj < bestj))) {
        best = ov;
        bestj = oj;
        cbest = oc;
      }
    }
    if (lane < RG) {
      sv[warp][lane] = best;
      sj[warp][lane] = bestj;
      sc[warp][lane] = cbest;
    }
    __syncthreads();
    if (threadIdx.x < ng) {
      const int s = threadIdx.x;
      double b = -1.0, c = 0.0;
      int64_t bj = -1;
      for (int q = 0; q < NW; q++)
        if (sj[q][s] >= 0 && (bj < 0 || sv[q][s] > b || (sv[q][s] == b && sj[q][s] < bj))) {
          b = sv[q][s];
          bj = sj[q][s];
          c = sc[q][s];
        }
      const int64_t slot = (e0 + s) * nparts + part;
      st.rs_pv[slot] = b;
      st.rs_pj[slot] = bj;
      st.rs_pc[slot] = c;
      __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st.rs_cnt[g], 1) == (int)nparts - 1;
    __syncthreads();
    if (last && threadIdx.x < ng) {  // every part of the group published: reduce
      __threadfence();
      const int64_t e = e0 + threadIdx.x;
      double b = -1.0, c = 0.0;
      int64_t bj = -1;
      for (int64_t q = 0; q < nparts; q++) {
        const double v = __ldcg(st.rs_pv + e * nparts + q);
        const int64_t j = __ldcg(st.rs_pj + e * nparts + q);
        if (j >= 0 && (bj < 0 || v > b || (v == b && j < bj))) {
          b = v;
          bj = j;
          c = __ldcg(st.rs_pc + e * nparts + q);
        }
      }
      const int64_t sig = st.pending[e];
      st.rs_j[sig] = bj;
      st.rs_c[sig] = c;
    }
    if (last && threadIdx.x == 0) st.rs_cnt[g] = 0;
    __syncthreads();
  }
}


// ---------------------------------------------------------------- tiled rescan
// For large dictionaries (every group of the kernel above would stream the
// whole fp64 dictionary from HBM or L2; see rescan_tiled) the queued rescans of one
// iteration are computed as the fp64 GEMM C = R D64^T over all queued
// residuals R at once, tiled 64 signals x 128 atoms per CTA (8 x 8 register
// blocking: 2 B of shared-memory traffic per FMA, i.e. FP64-pipe bound), with
// the masked argmax fused into the epilogue: each tile publishes
// (max |c|, lowest atom, c) per signal, and the last atom tile of a signal
// tile to finish reduces the partials into rs_j / rs_c.  Work items run
// signal-tile-fastest so the CTAs sharing an atom tile are co-resident and
// the dictionary is read from HBM about once per iteration.  Queues longer
// than `cap` signals run in several passes (a pass past the queue's end
// exits at once).
constexpr int RT_S = 64, RT_A = 128, RT_K = 16;

template <typename YT>
__global__ void __launch_bounds__(256) rescan_residual_kernel(
    const YT *__restrict__ ys, const double *__restrict__ d64, int64_t t, int64_t n, int64_t kw,
    int iter, TensorState st, const int64_t *out_sel, const double *out_coef, int64_t base,
    int64_t cap, double *__restrict__ rbuf, uint32_t *__restrict__ tbits) {
  extern __shared__ double rrs[];
  double *x = rrs;                       // kw
  int64_t *sel = (int64_t *)(x + kw);    // kw
  const int64_t count = st.npending[iter];
  const int64_t end = count < base + cap ? count : base + cap;
  const int64_t tw = (t + 31) / 32;
  const int64_t k = iter;
  for (int64_t e = base + blockIdx.x; e < end; e += gridDim.x) {
    const int64_t sig = st.pending[e], slot = e - base;
    for (int64_t l = threadIdx.x; l < k; l += blockDim.x) {
      x[l] = out_coef[sig * kw + l];
      sel[l] = out_sel[sig * kw + l];
    }
    uint32_t *tb = tbits + slot * tw;
    for (int64_t i = threadIdx.x; i < tw; i += blockDim.x) tb[i] = 0u;
    __syncthreads();
    if (threadIdx.x < k) {
      const int64_t j = sel[threadIdx.x];
      atomicOr(&tb[j >> 5], 1u << (j & 31));
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      double ri = (double)ys[sig * n + i];
      for (int64_t l = 0; l < k; l++) ri = fma(-x[l], __ldg(d64 + sel[l] * n + i), ri);
      rbuf[slot * n + i] = ri;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) rescan_tile_kernel(
    const double *__restrict__ d64, int64_t t, int64_t n, int iter, TensorState st, int64_t base,
    int64_t cap, const double *__restrict__ rbuf, const uint32_t *__restrict__ tbits,
    double *__restrict__ pv, int *__restrict__ pj, double *__restrict__ pc, int *tcnt) {
  constexpr int SA = RT_S + 1, SB = RT_A + 1;  // padded rows: conflict-free transposed stores
  extern __shared__ double tsm[];
  double *As = tsm;                // RT_K x SA   residual chunk, k-major
  double *Bs = As + RT_K * SA;     // RT_K x SB   atom chunk, k-major
  __shared__ int last;
  int64_t count = st.npending[iter] - base;
  if (count > cap) count = cap;
  if (count <= 0) return;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t s_tiles = (count + RT_S - 1) / RT_S, a_tiles = (t + RT_A - 1) / RT_A;
  const int64_t tw = (t + 31) / 32;
  for (int64_t w = blockIdx.x; w < s_tiles * a_tiles; w += gridDim.x) {
    const int64_t stile = w % s_tiles, at = w / s_tiles;
    const int64_t s0 = stile * RT_S, a0 = at * RT_A;
    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[i][j] = 0.0;
    for (int64_t k0 = 0; k0 < n; k0 += RT_K) {
#pragma unroll
      for (int q = 0; q < RT_S * RT_K / 128; q++) {
        const int idx = tid + 128 * q, s = idx / RT_K, kk = idx % RT_K;
        As[kk * SA + s] =
            (s0 + s < count && k0 + kk < n) ? rbuf[(s0 + s) * n + k0 + kk] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < RT_A * RT_K / 128; q++) {
        const int idx = tid + 128 * q, a = idx / RT_K, kk = idx % RT_K;
        Bs[kk * SB + a] =
            (a0 + a < t && k0 + kk < n) ? __ldg(d64 + (a0 + a) * n + k0 + kk) : 0.0;
      }
      __syncthreads();
#pragma unroll 4
      for (int kk = 0; kk < RT_K; kk++) {
        double av[8], bv[8];
#pragma unroll
        for (int i = 0; i < 8; i++) av[i] = As[kk * SA + ty + 8 * i];
#pragma unroll
        for (int j = 0; j < 8; j++) bv[j] = Bs[kk * SB + tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 8; i++)
#pragma unroll
          for (int j = 0; j < 8; j++) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
    // ---- masked argmax: my 8 atoms (ascending), then across the 16 tx lanes
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const int64_t s = s0 + ty + 8 * i;
      double best = -1.0, cb = 0.0;
      int bj = -1;
      if (s < count) {
        const uint32_t *tb = tbits + s * tw;
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int64_t a = a0 + tx + 16 * j;
          if (a < t && !((__ldg(tb + (a >> 5)) >> (a & 31)) & 1u)) {
            const double v = fabs(acc[i][j]);
            if (v > best) {
              best = v;
              bj = (int)a;
              cb = acc[i][j];
            }
          }
        }
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
        const double oc = __shfl_xor_sync(0xffffffffu, cb, off);
        if (oj >= 0 && (bj < 0 || ov > best || (ov == best && oj < bj))) {
          best = ov;
          bj = oj;
          cb = oc;
        }
      }
      if (tx == 0 && s < count) {
        pv[s * a_tiles + at] = best;
        pj[s * a_tiles + at] = bj;
        pc[s * a_tiles + at] = cb;
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(&tcnt[stile], 1) == (int)a_tiles - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      for (int si = tid; si < RT_S; si += blockDim.x) {
        const int64_t s = s0 + si;
        if (s >= count) break;
        double b = -1.0, c = 0.0;
        int bjj = -1;
        for (int64_t q = 0; q < a_tiles; q++) {
          const double v = __ldcg(pv + s * a_tiles + q);
          const int j = __ldcg(pj + s * a_tiles + q);
          if (j >= 0 && (bjj < 0 || v > b || (v == b && j < bjj))) {
            b = v;
            bjj = j;
            c = __ldcg(pc + s * a_tiles + q);
          }
        }
        const int64_t sig = st.pending[base + s];
        st.rs_j[sig] = bjj;
        st.rs_c[sig] = c;
      }
      if (tid == 0) tcnt[stile] = 0;
    }
    __syncthreads();
  }
}

// Buffers of the tiled rescan (stream-ordered allocations, freed at the end
// of the chunk).
struct TileRescan {
  int64_t cap = 0, a_tiles = 0;
  double *r = nullptr, *pv = nullptr, *pc = nullptr;
  uint32_t *tb = nullptr;
  int *pj = nullptr, *cnt = nullptr;
  void *mem = nullptr;
  cudaStream_t stream = nullptr;
  ~TileRescan() {
    if (mem) cudaFreeAsync(mem, stream);
  }
};

// Tiled when the dictionary is large, or mid-sized with long supports (the
// queue then holds hundreds of signals per iteration); CDB_RESCAN=tile|group.
bool rescan_tiled(int64_t t, int64_t n, int64_t k_max) {
  const char *m = getenv("CDB_RESCAN");
  if (m && !strcmp(m, "tile")) return true;
  if (m && !strcmp(m, "group")) return false;
  return t * n >= (int64_t(1) << 22) || (t * n >= (int64_t(1) << 20) && k_max >= 32);
}

cudaError_t tile_rescan_alloc(TileRescan &tr, int64_t p, int64_t t, int64_t n,
                              cudaStream_t stream) {
  // residual rows of the queued signals: up to 1 GiB, so a whole chunk of a
  // small-N problem is one (residual, tile) launch pair per iteration (the
  // pairs beyond the queue's length exit at once but still cost a launch)
  int64_t cap = (int64_t(1024) << 20) / (8 * n);
  cap = cap / RT_S * RT_S;
  if (cap < RT_S) cap = RT_S;
  if (cap > p) cap = (p + RT_S - 1) / RT_S * RT_S;
  tr.cap = cap;
  tr.a_tiles = (t + RT_A - 1) / RT_A;
  const int64_t tw = (t + 31) / 32;
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  const int64_t b_r = al(cap * n * 8), b_tb = al(cap * tw * 4), b_p = al(cap * tr.a_tiles * 8),
                b_j = al(cap * tr.a_tiles * 4), b_c = al((cap / RT_S + 1) * 4);
  tr.stream = stream;
  cudaError_t e = cudaMallocAsync(&tr.mem, b_r + b_tb + 2 * b_p + b_j + b_c, stream);
  if (e != cudaSuccess) return e;
  uint8_t *w = (uint8_t *)tr.mem;
  tr.r = (double *)w;
  tr.tb = (uint32_t *)(w += b_r);
  tr.pv = (double *)(w += b_tb);
  tr.pc = (double *)(w += b_p);
  tr.pj = (int *)(w += b_p);
  tr.cnt = (int *)(w += b_j);
  return cudaMemsetAsync(tr.cnt, 0, b_c, stream);
}

template <typename YT>
cudaError_t launch_rescan_tiled_t(const TensorArgs &a, const TensorState &st, TileRescan &tr,
                                  int64_t t, int64_t n, int64_t kw, int it, cudaStream_t stream) {
  const size_t tsm = sizeof(double) * RT_K * ((RT_S + 1) + (RT_A + 1));
  const size_t rsm = 16 * (size_t)kw;
  for (int64_t base = 0; base < a.p; base += tr.cap) {
    rescan_residual_kernel<YT><<<(unsigned)(a.num_sms * 4), 256, rsm, stream>>>(
        (const YT *)a.ys, a.d64, t, n, kw, it, st, a.out_sel, a.out_coef, base, tr.cap, tr.r,
        tr.tb);
    note_launch();
    rescan_tile_kernel<<<(unsigned)(a.num_sms * 3), 128, tsm, stream>>>(
        a.d64, t, n, it, st, base, tr.cap, tr.r, tr.tb, tr.pv, tr.pj, tr.pc, tr.cnt);
    note_launch();
  }
  return cudaGetLastError();
}

// Signals per rescan group: as many as fit 200 KB of shared memory (r, x,
// sel, taken per signal), at most 8.
size_t rescan_smem(int rg, int64_t t, int64_t n, int64_t kw) {
  return (size_t)rg * (8 * n + 16 * kw + 4 * ((t + 31) / 32)) + 64;
}

template <typename YT>
cudaError_t launch_rescan_t(const TensorArgs &a, const TensorState &st, int64_t t, int64_t n,
                            int64_t kw, int it, cudaStream_t stream) {
  const size_t lim = 200 * 1024;
  int rg = 8;
  while (rg > 1 && rescan_smem(rg, t, n, kw) > lim) rg >>= 1;
  const size_t sm = rescan_smem(rg, t, n, kw);
  if (sm > 227 * 1024) return cudaErrorInvalidValue;
  const void *f = rg == 8   ? (const void *)rescan_kernel<YT, 8>
                  : rg == 4 ? (const void *)rescan_kernel<YT, 4>
                  : rg == 2 ? (const void *)rescan_kernel<YT, 2>
                            : (const void *)rescan_kernel<YT, 1>;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int per_sm = sm <= 100 * 1024 ? 2 : 1;
  const unsigned grid = (unsigned)(a.num_sms * per_sm);
  const YT *ys = (const YT *)a.ys;
  switch (rg) {
    case 8: rescan_kernel<YT, 8><<<grid, 512, sm, stream>>>(ys, a.d64, a.p, t, n, kw, it, st, a.out_sel, a.out_coef); break;
    case 4: rescan_kernel<YT, 4><<<grid, 512, sm, stream>>>(ys, a.d64, a.p, t, n, kw, it, st, a.out_sel, a.out_coef); break;
    case 2: rescan_kernel<YT, 2><<<grid, 512, sm, stream>>>(ys, a.d64, a.p, t, n, kw, it, st, a.out_sel, a.out_coef); break;
    default: rescan_kernel<YT, 1><<<grid, 512, sm, stream>>>(ys, a.d64, a.p, t, n, kw, it, st, a.out_sel, a.out_coef); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_rescan(const TensorArgs &a, const TensorState &st, int64_t t, int64_t n,
                          int64_t kw, int it, cudaStream_t stream) {
  return a.ys_f32 ? launch_rescan_t<float>(a, st, t, n, kw, it, stream)
                  : launch_rescan_t<double>(a, st, t, n, kw, it, stream);
}

// Final residual norms (the reported rnorm): sqrt(|y|^2 - |z|^2) when that is
// tight, else the exact |y - D64_S x|.
template <typename YT>
__global__ void __launch_bounds__(256) ls_final_kernel(const YT *__restrict__ ys,
                                                       const double *__restrict__ d64, int64_t p,
                                                       int64_t n, int64_t kw, TensorState st,
                                                       const int64_t *out_sel,
                                                       const double *out_coef,
                                                       const int64_t *out_count,
                                                       double *out_rnorm) {
  const int64_t sig = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sig >= p || (st.status[sig] & ST_DELEGATE)) return;
  const int64_t kd = out_count[sig];
  if (kd == 0) return;
  // |r|^2 = |y|^2 - |z|^2 is accurate to ~1e-16 |y|^2 / |r|^2 relative:
  // re-materialise the residual only when that is not tight (as gram_engine)
  const double rn2 = st.rn2[sig];
  if (rn2 > 1e-6 * st.yy[sig]) {
    if (lane == 0) out_rnorm[sig] = sqrt(rn2);
    return;
  }
  const int64_t *sel = out_sel + sig * kw;
  const double *x = out_coef + sig * kw;
  double rr = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    double ri = (double)ys[sig * n + i];
    for (int64_t l = 0; l < kd; l++) ri = fma(-x[l], __ldg(d64 + sel[l] * n + i), ri);
    rr = fma(ri, ri, rr);
  }
  rr = warp_sum(rr);
  if (lane == 0) out_rnorm[sig] = sqrt(rr);
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
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// Full-dictionary scans that stream the signal operand (N_pad > the resident
// limit: cfg 4 full OMP) split the dictionary into this many parts per signal
// tile (CDB_CORR_SPLIT overrides; 1 = off): work items (tile, part), the parts'
// top-8 lists merged by merge_cands_kernel.
constexpr int kMaxCorrSplit = 8;

int64_t tensor_state_bytes(int64_t p, int64_t n, int64_t kw) {
  const int64_t n_pad = (n + BK - 1) / BK * BK;
  const int64_t p_pad = (p + BM - 1) / BM * BM;
  return p_pad * n_pad * 2 + p * kw * ((kw + 15) & ~int64_t(15)) * 8 + p * kw * 8 + p * 8 * 6 + p * NCAND * 8 + p * 4 +
         p * 8 * 3 + p * (3 * 8 * RS_SPLIT + 4) + 4 * 4096 + 24 * 256 +
         p * kMaxCorrSplit * (NCAND * 8 + 4);  // partial candidate lists of a split scan
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
  st.r16 = (__half *)take(p_pad * n_pad * 2);
  st.linv = (double *)take(p * kw * ((kw + 15) & ~int64_t(15)) * 8);
  st.z = (double *)take(p * kw * 8);
  st.rn2 = (double *)take(p * 8);
  st.yy = (double *)take(p * 8);
  st.rt = (double *)take(p * 8);
  st.dr = (double *)take(p * 8);
  st.rq = (double *)take(p * 8);
  st.emax = a.emax;
  st.dinv = 1.0 / a.dscale;
  st.tol = (double *)take(p * 8);
  st.status = a.status;
  int *cidx = (int *)take(p * NCAND * 4);
  float *cval = (float *)take(p * NCAND * 4);
  float *cdrop = (float *)take(p * 4);
  st.cand_idx = cidx;
  st.cand_val = cval;
  st.cand_drop = cdrop;
  int *pidx = (int *)take(p * kMaxCorrSplit * NCAND * 4);
  float *pval = (float *)take(p * kMaxCorrSplit * NCAND * 4);
  float *pdrop = (float *)take(p * kMaxCorrSplit * 4);
  st.active = (int *)take((a.k_max + 1) * 4);
  st.npending = (int *)take((a.k_max + 1) * 4);
  st.pending = (int64_t *)take(p * 8);
  st.rs_j = (int64_t *)take(p * 8);
  st.rs_c = (double *)take(p * 8);
  st.rs_pv = (double *)take(p * RS_SPLIT * 8);
  st.rs_pj = (int64_t *)take(p * RS_SPLIT * 8);
  st.rs_pc = (double *)take(p * RS_SPLIT * 8);
  st.rs_cnt = (int *)take(p * 4);
  st.rescans = a.rescans;
  st.debug_sig = getenv("CDB_LS_DEBUG") ? atoll(getenv("CDB_LS_DEBUG")) : -1;
  cudaError_t e;
  if ((e = cudaMemsetAsync(st.r16, 0, p_pad * n_pad * 2, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(st.active, 0, (a.k_max + 1) * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(st.npending, 0, (a.k_max + 1) * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(st.rs_cnt, 0, p * 4, stream)) != cudaSuccess) return e;

  CUtensorMap tm_a, tm_b;
  if (!make_map(&tm_a, st.r16, p_pad, n_pad, BMH) || !make_map(&tm_b, a.d16, t, n_pad, BN))
    return cudaErrorInvalidValue;

  const unsigned wblocks = (unsigned)((p * 32 + 255) / 256);
  {
  ProfScope _ps("ls_init", stream);
  if (a.ys_f32)
    ls_init_kernel<float><<<wblocks, 256, 0, stream>>>((const float *)a.ys, p, n, n_pad, kw, a.eps,
                                                       st, a.out_sel, a.out_coef, a.out_count,
                                                       a.out_rnorm, a.out_scans, a.out_flag);
  else
    ls_init_kernel<double><<<wblocks, 256, 0, stream>>>((const double *)a.ys, p, n, n_pad, kw,
                                                        a.eps, st, a.out_sel, a.out_coef,
                                                        a.out_count, a.out_rnorm, a.out_scans,
                                                        a.out_flag);
  }
  note_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;

  const bool a_res = n_pad / BK <= RES_KCHUNKS;
  const size_t corr_smem = (a_res ? sizeof(CorrSmemRes) : sizeof(CorrSmemStr)) + 1024;
  if ((e = cudaFuncSetAttribute(a_res ? corr_topk_kernel<true, false> : corr_topk_kernel<false, false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)corr_smem)) !=
      cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(a_res ? corr_topk_kernel<true, true> : corr_topk_kernel<false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)corr_smem)) !=
      cudaSuccess)
    return e;
  const int64_t m_tiles = p_pad / BM;
  int nsplit = 1;
  if (!a_res && (t + BN - 1) / BN >= 32) nsplit = 4;  // 1 / 2 / 4 / 8: 708 / 593 / 482 / 488 ms (cfg 4 full, 65k)
  if (const char *v = getenv("CDB_CORR_SPLIT")) {
    const int q = atoi(v);
    nsplit = q >= 1 && q <= kMaxCorrSplit ? q : nsplit;
  }
  const int64_t corr_items = m_tiles * nsplit;
  unsigned corr_grid = (unsigned)(corr_items < a.num_sms ? corr_items : a.num_sms);
  if (const char *cap = getenv("CDB_CORR_GRID_CAP")) {
    const int c = atoi(cap);
    if (c > 0 && (unsigned)c < corr_grid) corr_grid = (unsigned)c;
  }
  const int64_t ls_per_warp = (int64_t)sizeof(double) * (kw * ((kw + 15) & ~int64_t(15)) + 5 * kw + n);
  int ls_wpb = (int)((160 * 1024) / ls_per_warp);
  if (ls_wpb > 8) ls_wpb = 8;
  if (ls_wpb < 1) ls_wpb = 1;
  const size_t ls_smem = (size_t)ls_per_warp * ls_wpb;
  if (a.ys_f32)
    e = cudaFuncSetAttribute(ls_step_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ls_smem);
  else
    e = cudaFuncSetAttribute(ls_step_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ls_smem);
  if (e != cudaSuccess) return e;
  // E = c_err (|r~| + rq)(1 + 2^-7) dmax + emax (|r~| + rq) + dmax (rq + dr):
  // the fp16 operands' rounding is charged exactly as measured (in unscaled
  // units; the power-of-two operand scales cancel exactly) -- emax =
  // max_j |d^_j - d_j| (dictionary), rq = |r^ - r~| (per signal,
  // per iteration), via <d^, r^> - <d, r~> = <d^ - d, r^> + <d, r^ - r~> --
  // and c_err covers the fp32 accumulation over n_pad terms and the
  // truncation of the packed epilogue keys (2^-18; 2^-15 kept as margin),
  // relative to |d^| |r^| <= dmax (1 + 2^-8) (|r~| + rq).
  const double c_err = (double)(n_pad + 16) * 0x1p-23 + 0x1p-15;
  const unsigned ls_grid = (unsigned)((p + ls_wpb - 1) / ls_wpb);
  // grouped LS kernel: 8-lane groups (4 signals per warp) when the per-signal
  // state is small, whole warps otherwise; CDB_LS_LEGACY=1 forces ls_step
  const int64_t grp_bytes = 8 * (kw * ((kw + 15) & ~int64_t(15)) + 5 * kw);
  // lanes per signal in the grouped LS kernel: 16 measured best on cfg 1
  // (8: 10.3 M, 16: 10.9 M signals/s); whole warps when the state is large
  int lsg_g = 4 * 2 * grp_bytes <= 96 * 1024 ? 16 : 32;
  if (const char *g = getenv("CDB_LS_G")) {
    const int v = atoi(g);
    if ((v == 8 && 4 * grp_bytes <= 48 * 1024) || v == 16 || v == 32) lsg_g = v;
  }
  const int64_t lsg_per_block = 4 * (32 / lsg_g) * grp_bytes;  // 4 warps per block
  int64_t lsg_smem = lsg_per_block;
  if (getenv("CDB_LS_LEGACY") || lsg_per_block > 200 * 1024) lsg_smem = 0;
  const unsigned lsg_grid = (unsigned)((p + 4 * (32 / lsg_g) - 1) / (4 * (32 / lsg_g)));
  if (lsg_smem > 0) {
    auto set = [&](const void *f) {
      return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsg_smem);
    };
    if ((e = set((const void *)ls_group_kernel<float, 8>)) != cudaSuccess) return e;
    if ((e = set((const void *)ls_group_kernel<float, 16>)) != cudaSuccess) return e;
    if ((e = set((const void *)ls_group_kernel<float, 16, 16>)) != cudaSuccess) return e;
    if ((e = set((const void *)ls_group_kernel<double, 16, 16>)) != cudaSuccess) return e;
    if ((e = set((const void *)ls_group_kernel<double, 16>)) != cudaSuccess) return e;
    if ((e = set((const void *)ls_group_kernel<double, 8>)) != cudaSuccess) return e;
    if ((e = set((const void *)ls_group_kernel<float, 32>)) != cudaSuccess) return e;
    if ((e = set((const void *)ls_group_kernel<double, 32>)) != cudaSuccess) return e;
  }
  const bool tiled = rescan_tiled(t, n, a.k_max);
  // programmatic dependent launch for the scan / least-squares pairs (not
  // while per-kernel events are recorded: they would time the overlap)
  const bool pdl = pdl_enabled() && !prof_active();
  // large N: build the scan operand in its own kernel (CDB_LS_SPLIT=0|1 overrides)
  int split = n > 256 ? 1 : 0;
  // N = 128 with K <= 32 (cfg 2 zero-tree step 1): the warp-per-signal LS kernel
  // plus the one-warp fp32 operand kernel beat the grouped kernel with its fused
  // operand, 18.6 + 9.3 vs 39.2 ms per 200 k signals (zero-tree 2.95 M -> 3.55 M/s)
  if (n == 128 && kw <= 32 && !(getenv("CDB_RESID_F32") && atoi(getenv("CDB_RESID_F32")) == 0))
    split = 1;
  if (const char *v = getenv("CDB_LS_SPLIT")) split = atoi(v) ? 1 : 0;
  // long supports: the wide LS kernel (L^{-1} in global memory, warp per signal);
  // CDB_LS_WIDE=0|1 overrides
  int wide_kr = kw <= 32 ? 1 : (kw <= 64 ? 2 : (kw <= 128 ? 4 : 0));
  // ... and short supports whose operand is built by its own kernel anyway
  // (N > 256): cfg 2 full OMP (N = 1024, K = 32), 200 k signals: ls_step 41.9 ->
  // 24.2 ms, 1.24 M -> 1.39 M signals/s; with the operand fused into the grouped
  // kernel (N <= 256: cfg 1 full OMP) the wide kernel + its operand pass lose
  // (7.5 -> 10.4 ms per 100 k)
  bool wide = (kw > 32 || split) && wide_kr > 0;
  if (const char *v = getenv("CDB_LS_WIDE")) wide = atoi(v) != 0 && wide_kr > 0;
  if (wide) split = 1;
  TileRescan tr;
  if (tiled && (e = tile_rescan_alloc(tr, p, t, n, stream)) != cudaSuccess) return e;
  for (int it = 0; it < a.k_max; it++) {
    {
    ProfScope _ps("corr_topk", stream);
    auto kern = a_res ? corr_topk_kernel<true, false> : corr_topk_kernel<false, false>;
    if (nsplit == 1) {
      e = launch_k(pdl, kern, corr_grid, THREADS, corr_smem, stream, tm_a, tm_b, p, t,
                   (int)(n_pad / BK), m_tiles, it ? st.active + it - 1 : nullptr, cidx, cval, cdrop,
                   1);
    } else {
      auto kern_s = a_res ? corr_topk_kernel<true, true> : corr_topk_kernel<false, true>;
      e = launch_k(pdl, kern_s, corr_grid, THREADS, corr_smem, stream, tm_a, tm_b, p, t,
                   (int)(n_pad / BK), m_tiles, it ? st.active + it - 1 : nullptr, pidx, pval, pdrop,
                   nsplit);
      if (e == cudaSuccess) {
        note_launch();
        e = launch_k(pdl, merge_cands_kernel, (unsigned)((p * 32 + 255) / 256), 256, 0, stream,
                     (const int *)pidx, (const float *)pval, (const float *)pdrop, p, nsplit,
                     it ? (const int *)(st.active + it - 1) : (const int *)nullptr, cidx, cval,
                     cdrop);
      }
    }
    if (e != cudaSuccess) return e;
    }
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    for (int resume = 0; resume < 2; resume++) {
      if (resume) {
        ProfScope _ps("rescan", stream);
        if (tiled)
          e = a.ys_f32 ? launch_rescan_tiled_t<float>(a, st, tr, t, n, kw, it, stream)
                       : launch_rescan_tiled_t<double>(a, st, tr, t, n, kw, it, stream);
        else
          e = launch_rescan(a, st, t, n, kw, it, stream);
        if (e != cudaSuccess) return e;
        note_launch();
      }
      ProfScope _ps(resume ? "ls_resume" : "ls_step", stream);
      if (wide) {
        const unsigned grid = resume ? (unsigned)(a.num_sms * 8) : (unsigned)((p + 3) / 4);
        // blocks per SM the register budget targets (CDB_LSW_MINB=4|5|6 for A/B)
        // (cfg 4 step 1 per 1M: 4 / 5 / 6 -> 514 / 462 / 472 ms)
        static const int lsw_mb = getenv("CDB_LSW_MINB") ? atoi(getenv("CDB_LSW_MINB")) : 5;
#define CDB_WIDE_MB(YT_, KR_, MB_)                                                              \
  e = launch_k(pdl, ls_wide_kernel<YT_, KR_, MB_>, grid, 128, 0, stream, (const YT_ *)a.ys,     \
               a.d64, a.gram, p, t, (int)n, (int)a.k_max, (int)kw, it, c_err, a.dmax, st,       \
               a.out_sel, a.out_coef, a.out_count, a.out_scans, resume);
#define CDB_WIDE(YT_, KR_)                                                                      \
  if (lsw_mb == 5) { CDB_WIDE_MB(YT_, KR_, 5) }                                                 \
  else if (lsw_mb == 6) { CDB_WIDE_MB(YT_, KR_, 6) }                                            \
  else { CDB_WIDE_MB(YT_, KR_, 4) }
        if (a.ys_f32) {
          if (wide_kr == 1) { CDB_WIDE(float, 1) } else if (wide_kr == 2) { CDB_WIDE(float, 2) } else { CDB_WIDE(float, 4) }
        } else {
          if (wide_kr == 1) { CDB_WIDE(double, 1) } else if (wide_kr == 2) { CDB_WIDE(double, 2) } else { CDB_WIDE(double, 4) }
        }
#undef CDB_WIDE
#undef CDB_WIDE_MB
      } else if (lsg_smem > 0) {
        const unsigned grid = resume ? (unsigned)(a.num_sms * 4) : lsg_grid;
        if (lsg_g == 8) {
          if (a.ys_f32)
            e = launch_k(pdl, ls_group_kernel<float, 8>, grid, 128, lsg_smem, stream,
                (const float *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
          else
            e = launch_k(pdl, ls_group_kernel<double, 8>, grid, 128, lsg_smem, stream,
                (const double *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
        } else if (lsg_g == 16 && n <= 256) {
          if (a.ys_f32)
            e = launch_k(pdl, ls_group_kernel<float, 16, 16>, grid, 128, lsg_smem, stream,
                (const float *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
          else
            e = launch_k(pdl, ls_group_kernel<double, 16, 16>, grid, 128, lsg_smem, stream,
                (const double *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
        } else if (lsg_g == 16) {
          if (a.ys_f32)
            e = launch_k(pdl, ls_group_kernel<float, 16>, grid, 128, lsg_smem, stream,
                (const float *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
          else
            e = launch_k(pdl, ls_group_kernel<double, 16>, grid, 128, lsg_smem, stream,
                (const double *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
        } else {
          if (a.ys_f32)
            e = launch_k(pdl, ls_group_kernel<float, 32>, grid, 128, lsg_smem, stream,
                (const float *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
          else
            e = launch_k(pdl, ls_group_kernel<double, 32>, grid, 128, lsg_smem, stream,
                (const double *)a.ys, a.d64, a.d32, a.gram, p, t, (int)n, n_pad, (int)a.k_max,
                (int)kw, it, c_err, a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans,
                resume, split);
        }
      } else {
        const unsigned grid = resume ? (unsigned)a.num_sms : ls_grid;
        if (a.ys_f32)
          ls_step_kernel<float><<<grid, ls_wpb * 32, ls_smem, stream>>>(
              (const float *)a.ys, a.d64, a.d32, a.gram, p, t, n, n_pad, a.k_max, kw, it, c_err,
              a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans, resume);
        else
          ls_step_kernel<double><<<grid, ls_wpb * 32, ls_smem, stream>>>(
              (const double *)a.ys, a.d64, a.d32, a.gram, p, t, n, n_pad, a.k_max, kw, it, c_err,
              a.dmax, st, a.out_sel, a.out_coef, a.out_count, a.out_scans, resume);
      }
      if (e != cudaSuccess) return e;
      note_launch();
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (split && (wide || lsg_smem > 0) && it + 1 < a.k_max) {  // the next scan's operand
      ProfScope _ps("ls_resid", stream);
      const size_t xs = 16 * (size_t)kw;
      // threads per signal: N / 8 (8 elements each), 64..256
      const int bt = n >= 2048 ? 256 : (n >= 1024 ? 128 : 64);
      const unsigned g = (unsigned)(a.num_sms * (2048 / bt));
      // fp32 vectorised operand build when n = 4 * BT * V (CDB_RESID_F32=0: fp64 kernel)
      static const bool f32_ok = !(getenv("CDB_RESID_F32") && atoi(getenv("CDB_RESID_F32")) == 0);
      const size_t xs32 = 16 * (size_t)kw;
      // rows per pipeline group (CDB_RESID_G overrides).  Measured per 200 k cfg 2
      // signals: N = 1024 (full OMP) 8 / 6 / 4 -> 53.1 / 41.4 / 44.2 ms; N = 128 (step 1,
      // one warp per signal) 9.3 / 9.8 / 6.5 ms; N = 512 (cfg 4 step 1, per 131 k
      // signals) 51.3 / 41.7 / 45.0 ms
      static const int rg_env = getenv("CDB_RESID_G") ? atoi(getenv("CDB_RESID_G")) : 0;
      const int rg = rg_env ? rg_env : (n == 1024 || n == 512 ? 6 : (n == 128 ? 4 : 8));
#define CDB_RESID32G(BT_, V_, G_)                                                               \
  if (a.ys_f32)                                                                                 \
    resid_f32_kernel<float, BT_, V_, G_><<<g, BT_, xs32, stream>>>(                             \
        (const float *)a.ys, a.d32, p, n, n_pad, kw, a.dmax, st, a.out_sel, a.out_coef,         \
        a.out_count);                                                                           \
  else                                                                                          \
    resid_f32_kernel<double, BT_, V_, G_><<<g, BT_, xs32, stream>>>(                            \
        (const double *)a.ys, a.d32, p, n, n_pad, kw, a.dmax, st, a.out_sel, a.out_coef,        \
        a.out_count);
#define CDB_RESID32(BT_, V_)                                                                    \
  if (rg == 4) { CDB_RESID32G(BT_, V_, 4) }                                                     \
  else if (rg == 6) { CDB_RESID32G(BT_, V_, 6) }                                                \
  else { CDB_RESID32G(BT_, V_, 8) }
      bool done32 = false;
      if (f32_ok && kw <= 64) {  // one code entry per thread (BT >= 64)
        done32 = true;
        // N = 4096 (cfg 4 full OMP) stays on the fp64 kernel: measured 1988 vs
        // 6287 ms per 250 k signals (register-bound) and 37% more exact rescans
        // from the looser fp32 bound
        // (N = 512 as 128 threads x one float4 per row: 44.6 ms at best per 131 k cfg-4
        // signals against 41.7 ms for 64 threads x two)
        if (n == 4 * 64 * 2) { CDB_RESID32(64, 2) }
        else if (n == 4 * 128 * 2) { CDB_RESID32(128, 2) }
        else if (n == 4 * 64 * 1) { CDB_RESID32(64, 1) }
        else if (n == 4 * 32 * 1 && kw <= 32) {  // one warp per signal (cfg 2 step 1)
          const unsigned g = (unsigned)(a.num_sms * 32);
          CDB_RESID32(32, 1)
        }
        else done32 = false;
      }
#undef CDB_RESID32
#undef CDB_RESID32G
      // long rows: the bulk-copy ring (CDB_RESID_BULK=0: the register-pipelined kernel)
      static const bool bulk_ok = !(getenv("CDB_RESID_BULK") && atoi(getenv("CDB_RESID_BULK")) == 0);
      // (measured per 65,536 signals, K = 32, bulk vs register-pipelined: N = 3072
      // 50.2 vs 61.3 ms; N = 2048 46.3 vs 56.8 ms with a 134 MB fp32 dictionary but
      // 38.5 vs 33.4 ms with an L2-resident one; N = 1024 93.2 vs 55.0 ms)
      const bool bulk_n = n >= 3072 || (n == 2048 && t * n * 4 > (int64_t(96) << 20));
      if (!done32 && bulk_ok && bulk_n && n % 1024 == 0 && n <= 4096 && kw <= 64) {
        done32 = true;
        const size_t bsm = (size_t)RB_S * n * 4 + 8 * (size_t)kw + 16 * RB_S;
        const unsigned bg = (unsigned)(a.num_sms * 2);
#define CDB_RESIDB(J_)                                                                          \
  {                                                                                             \
    auto kf = resid_bulk_kernel<float, J_>;                                                     \
    auto kd_ = resid_bulk_kernel<double, J_>;                                                   \
    if (a.ys_f32) {                                                                             \
      e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);      \
      if (e == cudaSuccess)                                                                     \
        kf<<<bg, RB_T + 32, bsm, stream>>>((const float *)a.ys, a.d32, p, n, n_pad, kw, a.dmax, \
                                           st, a.out_sel, a.out_coef, a.out_count);             \
    } else {                                                                                    \
      e = cudaFuncSetAttribute(kd_, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);     \
      if (e == cudaSuccess)                                                                     \
        kd_<<<bg, RB_T + 32, bsm, stream>>>((const double *)a.ys, a.d32, p, n, n_pad, kw,       \
                                            a.dmax, st, a.out_sel, a.out_coef, a.out_count);    \
    }                                                                                           \
  }
        if (n == 1024) CDB_RESIDB(1)
        else if (n == 2048) CDB_RESIDB(2)
        else if (n == 3072) CDB_RESIDB(3)
        else CDB_RESIDB(4)
#undef CDB_RESIDB
        if (e != cudaSuccess) return e;
      }
      if (!done32) {
#define CDB_RESID(BT_)                                                                          \
  if (a.ys_f32)                                                                                 \
    resid_split_kernel<float, BT_><<<g, BT_, xs, stream>>>((const float *)a.ys, a.d32, p, n,    \
                                                           n_pad, kw, a.dmax, st, a.out_sel,    \
                                                           a.out_coef, a.out_count);            \
  else                                                                                          \
    resid_split_kernel<double, BT_><<<g, BT_, xs, stream>>>((const double *)a.ys, a.d32, p, n,  \
                                                            n_pad, kw, a.dmax, st, a.out_sel,   \
                                                            a.out_coef, a.out_count);
      if (bt == 256) {
        CDB_RESID(256)
      } else if (bt == 128) {
        CDB_RESID(128)
      } else {
        CDB_RESID(64)
      }
      }
#undef CDB_RESID
      note_launch();
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  ProfScope _ps("ls_final", stream);
  if (a.ys_f32)
    ls_final_kernel<float><<<wblocks, 256, 0, stream>>>((const float *)a.ys, a.d64, p, n, kw, st,
                                                        a.out_sel, a.out_coef, a.out_count,
                                                        a.out_rnorm);
  else
    ls_final_kernel<double><<<wblocks, 256, 0, stream>>>((const double *)a.ys, a.d64, p, n, kw, st,
                                                         a.out_sel, a.out_coef, a.out_count,
                                                         a.out_rnorm);
  note_launch();
  return cudaGetLastError();
}

// One correlation pass on caller-provided residual rows (debug / unit tests):
// r16 = fp16(rows) (P x n fp32 device), candidate lists out (values divided
// by the dictionary operand's scale).
cudaError_t debug_corr_topk(const void *d16, double dscale, int64_t t, int64_t n,
                            const float *rows, int64_t p, int *cand_idx, float *cand_val,
                            float *cand_drop, int grid_cap, cudaStream_t stream) {
  const int64_t n_pad = (n + BK - 1) / BK * BK;
  const int64_t p_pad = (p + BM - 1) / BM * BM;
  __half *r16 = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&r16, p_pad * n_pad * 2, stream);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(r16, 0, p_pad * n_pad * 2, stream);
  to_f16_rows<<<(unsigned)((p * n_pad + 255) / 256), 256, 0, stream>>>(rows, p, n, n_pad, r16);
  CUtensorMap tm_a, tm_b;
  if (!make_map(&tm_a, r16, p_pad, n_pad, BMH) || !make_map(&tm_b, d16, t, n_pad, BN))
    return cudaErrorInvalidValue;
  const bool a_res = n_pad / BK <= RES_KCHUNKS;
  const size_t corr_smem = (a_res ? sizeof(CorrSmemRes) : sizeof(CorrSmemStr)) + 1024;
  auto kern = a_res ? corr_topk_kernel<true, false> : corr_topk_kernel<false, false>;
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)corr_smem)) != cudaSuccess)
    return e;
  const int64_t m_tiles = p_pad / BM;
  int64_t grid = m_tiles < 148 ? m_tiles : 148;
  if (grid_cap > 0 && grid > grid_cap) grid = grid_cap;
  kern<<<(unsigned)grid, THREADS, corr_smem, stream>>>(tm_a, tm_b, p, t, (int)(n_pad / BK),
                                                       m_tiles, nullptr, cand_idx, cand_val,
                                                       cand_drop, 1);
  note_launch();
  unscale_vals<<<(unsigned)((p * NCAND + 255) / 256), 256, 0, stream>>>(cand_val, cand_drop, p,
                                                                        (float)(1.0 / dscale));
  e = cudaGetLastError();
  cudaFreeAsync(r16, stream);
  return e;
}

}  // namespace cdb
