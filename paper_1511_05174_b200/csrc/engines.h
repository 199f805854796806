// Internal engine interfaces (host side) of the crossdict B200 library.
#pragma once
#include <utility>
#include <cstdint>
#include <cuda_runtime.h>

#include "candidates.cuh"

namespace cdb {

void note_launch(int n = 1);

// Device-time profiler (cdb_profile_*): CUDA events recorded on the launching
// stream around each kernel launch, summed per kernel name.
void prof_begin(const char *name, cudaStream_t stream);
void prof_end(const char *name, cudaStream_t stream);
bool prof_active();  // per-kernel events are being recorded
bool pdl_enabled();  // CDB_PDL (default 1): programmatic dependent launch

// Launch `kern` with the programmatic-stream-serialization attribute when
// `pdl`: the kernel may start while its predecessor drains, and must call
// griddep_wait() before reading the predecessor's output.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), unsigned grid, unsigned block,
                     size_t smem, cudaStream_t stream, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
struct ProfScope {
  const char *name;
  cudaStream_t stream;
  ProfScope(const char *n, cudaStream_t s) : name(n), stream(s) { prof_begin(n, s); }
  ~ProfScope() { prof_end(name, stream); }
};

// ---------------------------------------------------------------- exact
struct ExactArgs {
  const double *mat_t;   // T x N fp64
  int64_t t, n;
  int64_t ys_stride;     // elements between signal rows
  const int64_t *sig_ids;  // optional: process only these signals
  int64_t p_count;       // number of signals to process (len(sig_ids) or P)
  const int *p_count_dev;  // optional: the count lives on the device (<= p_count)
  const int32_t *rows;     // optional coded mode: per-signal effective rows, m_sig[p]
                           // of them, each `fan` source coordinates (row p at
                           // rows + p * rows_stride; see eff_at in common.cuh)
  const int64_t *m_sig;
  int fan;
  int sum_order;           // eff_at ord: 0 sequential list, 1 numpy pairwise slots
  int64_t rows_stride;
  int64_t k_max;         // budget (clipped per signal when cands.clip)
  int64_t k_width;       // output row width
  const double *eps;
  Cands cands;
  int64_t *out_sel;
  double *out_coef;
  int64_t *out_count;
  double *out_rnorm;
  int64_t *out_scans;
  uint8_t *out_flag;
  double *work;          // warps * work_stride doubles
  int64_t work_stride;
};
int64_t exact_work_stride(int64_t n, int64_t k_width, int64_t max_cands);
cudaError_t launch_exact(const ExactArgs &args, const void *ys, bool ys_f32, int warps,
                         cudaStream_t stream);

// ---------------------------------------------------------------- gram
struct GramArgs {
  const double *d64;     // T x N fp64 atoms (rows)
  const double *gram;    // T x T fp64 Gram matrix
  int64_t t, n;
  int64_t ys_stride;
  int64_t p;             // signals in this launch
  int64_t p_offset;      // first signal of this launch
  int64_t k_max, k_width;
  const double *eps;
  Cands cands;
  int64_t max_cands;     // upper bound of cands.count(p) over the batch
  int64_t *out_sel;
  double *out_coef;
  int64_t *out_count;
  double *out_rnorm;
  int64_t *out_scans;
  uint8_t *out_flag;
  uint32_t *status;      // per-signal status bits (ST_DELEGATE ...)
  double *hwork;         // optional global H storage when it does not fit smem
  const char *tag;       // profiler name
  const double *alpha0_in;  // optional precomputed <d_{C_j}, y> (P x max_cands)
  int prefetch_runner;      // CTA kernel: L2-prefetch the runner-up's Gram slice
};
// Shared-memory bytes per warp of the Gram engine (H in smem or global), and
// the doubles of one signal's H (global scratch when it does not fit smem).
int64_t gram_h_doubles(int64_t max_cands, int64_t k_width);
int64_t gram_total_smem(int64_t max_cands, int64_t k_width, int64_t n, bool h_in_smem);
cudaError_t launch_gram(const GramArgs &args, const void *ys, bool ys_f32, int max_smem_per_block,
                        int num_sms, cudaStream_t stream);
// Streamed H (H larger than a warp's shared memory): persistent warps, the
// first nr rows of each warp's H in shared memory, the rest in a per-warp
// global slot of slot_doubles (args.hwork = warps * slot_doubles doubles).
struct GramStreamPlan {
  bool ok;
  bool cta;   // CTA per signal (gram_cta_kernel): warps = CTAs, per_warp_smem = per CTA
  bool reg;   // H on chip (gram_reg_kernel, cta too): nr = register rows
  bool tma;   // cta: rows [nr, k) streamed through a shared-memory ring by bulk copies
  int cpt;    // cta: candidates per thread
  int wpb, nr;
  int64_t per_warp_smem, warps, slot_doubles;
};
// Shared-memory-sized H that still goes to the CTA-per-signal kernel: 128 < S <= 256
// candidates with a precomputed alpha0, every H row in the CTA's third of shared
// memory (cfg 2 step 2: S = 256, K = 32).
bool gram_cta_preferred(int64_t max_cands, int64_t k_width, int64_t n, bool has_alpha0);
GramStreamPlan gram_stream_plan(int64_t max_cands, int64_t k_width, int64_t n, bool stage_y,
                                int max_smem_per_block, int num_sms);

// ---------------------------------------------------------------- resident
struct ResidentArgs {
  const double *d64;     // T x N fp64 atoms (rows)
  const double *gram;    // T x T fp64 Gram matrix (optional)
  int64_t t, n;
  int64_t p;
  int64_t k_max, k_width;
  const double *eps;
  Cands cands;
  int64_t max_cands;
  int64_t *out_sel;
  double *out_coef;
  int64_t *out_count;
  double *out_rnorm;
  int64_t *out_scans;
  uint8_t *out_flag;
  uint32_t *status;
  int64_t per_warp;      // filled by the launcher
  int64_t t_pad;         // filled by the launcher
  const char *tag;
};
bool resident_fits(int64_t n, int64_t t, int64_t kw, int64_t max_cands, int smem_optin);
cudaError_t launch_resident(const ResidentArgs &args, const void *ys, bool ys_f32, int smem_optin,
                            int num_sms, cudaStream_t stream);

// ---------------------------------------------------------------- tensor
struct TensorArgs {
  const void *ys;
  bool ys_f32;
  int64_t p, n, n_pad, t, k_max, k_width;
  const double *eps;
  const double *d64;
  const void *d16;
  const float *d32;      // T x N fp32 atoms (residual materialisation)
  const double *gram;
  double dmax;           // max atom norm (error bound)
  double emax;           // max |fp16(dscale d_j) / dscale - d_j| (error bound)
  double dscale;         // power-of-two scale of the fp16 dictionary operand
  int *rescans;          // device counter of inline exact rescans
  int64_t *out_sel;
  double *out_coef;
  int64_t *out_count;
  double *out_rnorm;
  int64_t *out_scans;
  uint8_t *out_flag;
  uint32_t *status;
  void *work;            // tensor_state_bytes(p, n, k_width) bytes
  int num_sms;
  const char *tag;       // profiler name prefix
};
int64_t tensor_state_bytes(int64_t p, int64_t n, int64_t kw);
cudaError_t run_tensor_chunk(const TensorArgs &args, cudaStream_t stream);
cudaError_t debug_corr_topk(const void *d16, double dscale, int64_t t, int64_t n,
                            const float *rows, int64_t p, int *cand_idx, float *cand_val,
                            float *cand_drop, int grid_cap, cudaStream_t stream);

// ---------------------------------------------------------------- helpers
cudaError_t launch_quant_err_max(const double *d64, const void *d16, int64_t t, int64_t n,
                                 int64_t n_pad, double scale, double *out, cudaStream_t stream);
cudaError_t launch_row_norm_max(const double *d64, int64_t t, int64_t n, double *out,
                                cudaStream_t stream);
cudaError_t launch_downsample(const void *ys, bool ys_f32, int64_t p, int64_t n,
                              const int64_t *fine_shape, const int64_t *factors, int rank,
                              double *y_low, int64_t n_low, cudaStream_t stream,
                              double rel = 0.0, double *eps_low = nullptr,
                              double *eps_fine = nullptr);
cudaError_t launch_row_tol(const void *ys, bool ys_f32, int64_t p, int64_t n, double rel,
                           double *eps, cudaStream_t stream);
cudaError_t launch_sort_blocks(const int64_t *low_sel, const int64_t *low_count, int64_t p,
                               int64_t k1, int64_t *blocks, cudaStream_t stream);
cudaError_t launch_gram_matrix(const double *d64, int64_t t, int64_t n, double *gram,
                               cudaStream_t stream);
cudaError_t launch_to_f16(const double *d64, int64_t t, int64_t n, int64_t n_pad, double scale,
                          void *d16, cudaStream_t stream);
bool route_alpha0_dmma(int64_t q, int64_t n);
cudaError_t launch_route_alpha0(const double *d64, int64_t t_low, int64_t n, int64_t q,
                               const void *ys, bool ys_f32, const int64_t *blocks,
                               const int64_t *nb, int64_t p, int64_t k1, int64_t smax,
                               double *alpha0, void *work, cudaStream_t stream);
int64_t route_work_bytes(int64_t t_low, int64_t p, int64_t k1, int64_t n, bool ys_f32);

// ---------------------------------------------------------------- patch pipeline ends
cudaError_t launch_extract_patches(const void *signal, bool f32, int rank, const int64_t *sig,
                                   const int64_t *pat, const int64_t *str, int remove_dc,
                                   double *rows, double *dc, int num_sms, cudaStream_t stream);
cudaError_t launch_reconstruct_aggregate(const double *d64, int64_t n, const int64_t *sel,
                                         const double *coef, int64_t kw, int64_t p,
                                         const double *dc, int rank, const int64_t *sig,
                                         const int64_t *pat, const int64_t *str, double *est,
                                         double *out, unsigned long long *uncovered, int num_sms,
                                         cudaStream_t stream);
cudaError_t launch_aggregate(const double *rows, const double *dc, int rank, const int64_t *sig,
                             const int64_t *pat, const int64_t *str, double *out,
                             unsigned long long *uncovered, cudaStream_t stream);
cudaError_t launch_to_f32(const double *d64, int64_t count, float *d32, cudaStream_t stream);
// n x len column block -> len x n rows (fp32 or fp64)
cudaError_t launch_cols_to_rows(const void *cols, bool f32, int64_t n, int64_t len, void *rows,
                                cudaStream_t stream);
cudaError_t launch_collect_delegates(const uint32_t *status, int64_t p, int64_t *ids,
                                     int *count, cudaStream_t stream);

// K-SVD update stage (ksvd_engine.cu): one persistent CTA over the atoms.
struct KsvdArgs {
  const double *y;        // M x N signal rows
  double *e;              // M x N residual rows (in/out)
  double *d;              // T x N atom rows (in/out)
  const int64_t *ptr;     // T + 1: users of atom j are sig[ptr[j] .. ptr[j+1])
  const int64_t *sig;     // ascending signal ids per atom
  double *val;            // code entries x[j, sig] (in/out)
  int64_t n, m, t, threshold;
  int64_t smem_b;         // doubles of shared memory for the Gram matrix
  double *ej;             // scratch: max users x N
  double *bglob;          // scratch: N x N (Gram matrix beyond smem_b)
  uint32_t *taken;        // M bits, zeroed
  int64_t *replaced;      // out
  long long *prof;        // optional phase times (ns, 16 slots; CDB_KSVD_PROF=1)
};
size_t ksvd_update_smem(int64_t n, int64_t smem_b);
cudaError_t launch_ksvd_update(const KsvdArgs &a, size_t smem, cudaStream_t stream);

}  // namespace cdb
