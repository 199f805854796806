/*
 * crossdict_b200.h -- C ABI of the B200 batched-OMP / zero-tree-OMP engine.
 *
 * This is the drop-in boundary for the reference package `crossdict`
 * (/root/reference/pkg/src/crossdict).  The reference has exactly one
 * compiled seam on this path, the numba kernel
 *
 *     omp_batch_kernel(mat_t, ys, k_max, eps, allowed, restricted,
 *                      out_sel, out_coef, out_count, out_rnorm, out_scans,
 *                      out_flag)                           (_kernels.py:50-168)
 *
 * bound into crossdict.pursuit by `from ._kernels import omp_batch_kernel`
 * (pursuit.py:32) and called only from pursuit._run_kernel (pursuit.py:234-250).
 * cdb_omp_batch() below takes the same arguments, in the same dtypes and
 * layouts, plus a dictionary handle (the device-resident form of `mat_t`) and
 * a CUDA stream.  The batched zero-tree driver (crossscale.py:235-283) is one
 * more entry point so that its grouping/routing runs on the device.
 *
 * Conventions (mirroring the reference seam, pursuit.py:240-245):
 *   - plain pointers and sizes; arrays are C-contiguous; int64/fp64/uint8 as
 *     in the reference; every pointer may be HOST or DEVICE memory (detected
 *     per pointer; host buffers are staged through the stream);
 *   - the caller allocates every output; the library overwrites them
 *     entirely (it does not rely on the caller's -1 / 0 pre-initialisation);
 *   - no exceptions cross the ABI; every function returns a cdb_status;
 *     validation that the reference performs in Python (ConfigError,
 *     DimensionError, DomainError) stays in the host layer, the ABI only
 *     re-checks sizes and returns CDB_ERR_ARG;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *     stream-ordered and return after the outputs are complete (host
 *     outputs) or enqueued (device outputs).
 */
#ifndef CROSSDICT_B200_H
#define CROSSDICT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CDB_OK = 0,
    CDB_ERR_ARG = 1,      /* size / pointer argument invalid                   */
    CDB_ERR_CUDA = 2,     /* a CUDA runtime call failed (see cdb_last_error)   */
    CDB_ERR_NOMEM = 3,    /* device or pinned allocation failed                */
    CDB_ERR_NODEV = 4,    /* no sm_100 device available                        */
    CDB_ERR_FORMAT = 5,   /* malformed .csd file (crossdict FormatError)       */
    CDB_ERR_CHECKSUM = 6  /* .csd CRC-32 mismatch (crossdict ChecksumError)    */
} cdb_status;

/* Opaque device-resident dictionary (atoms as rows, T x N). */
typedef struct cdb_dictionary cdb_dictionary;

/* Message for the last non-OK status on this thread. */
const char *cdb_last_error(void);

/* Library / device facts: writes the SM count and compute capability. */
cdb_status cdb_device_info(int *sm_count, int *cc_major, int *cc_minor);

/*
 * Stage a dictionary on the current device.
 * Replaces: tensor.py:124-129 (Dictionary.atoms_t, the T x N C-contiguous
 * kernel operand) and pursuit.py:96-123 (DenseColumns.mat_t).
 * atoms_t: T x N fp64 row-major (one atom per row), host or device.
 * Builds the fp64 copy, the bf16 tensor-core operand, squared norms and,
 * when T*T*8 bytes <= gram_budget_bytes, the fp64 Gram matrix.
 */
cdb_status cdb_dictionary_create(const double *atoms_t, int64_t t, int64_t n,
                                 int64_t gram_budget_bytes, void *stream,
                                 cdb_dictionary **out);
cdb_status cdb_dictionary_destroy(cdb_dictionary *dict);
/* Bytes of device memory held by the handle. */
int64_t cdb_dictionary_bytes(const cdb_dictionary *dict);

/* Engine selection for cdb_omp_batch / cdb_zero_tree_batch. */
typedef enum {
    CDB_ENGINE_AUTO = 0,     /* pick per problem shape (default)               */
    CDB_ENGINE_EXACT = 1,    /* warp-per-signal fp64 restatement of the kernel  */
    CDB_ENGINE_GRAM = 2,     /* signal-stationary fp64 Gram/Cholesky OMP        */
    CDB_ENGINE_TENSOR = 3,   /* tcgen05 bf16 correlation + certified fp64 LS    */
    CDB_ENGINE_RESIDENT = 4  /* dictionary resident in smem, fp64, warp/signal  */
} cdb_engine;

/*
 * Batched OMP.  Replaces omp_batch_kernel (_kernels.py:50-168) as called by
 * pursuit._run_kernel (pursuit.py:234-250).
 *   ys       : P x N signals as rows (pursuit.py:433 `ys_rows`); fp64, or fp32
 *              when ys_is_f32 != 0 (a compact exact input, e.g. fp32 data)
 *   eps      : P absolute residual tolerances (pursuit.py:434-437)
 *   allowed  : P x S ascending 0-based candidate ids, read only when
 *              restricted != 0 (pursuit.py:421-422), else may be NULL
 *   out_sel  : P x k_max int64, pick order, -1 padded
 *   out_coef : P x k_max fp64, aligned with out_sel
 *   out_count, out_scans : P int64;  out_rnorm : P fp64;  out_flag : P uint8
 */
cdb_status cdb_omp_batch(const cdb_dictionary *dict, const void *ys, int ys_is_f32,
                         int64_t p, int64_t k_max, const double *eps,
                         const int64_t *allowed, int64_t s_allowed, int restricted,
                         int64_t *out_sel, double *out_coef, int64_t *out_count,
                         double *out_rnorm, int64_t *out_scans, uint8_t *out_flag,
                         int engine, void *stream);

/*
 * Batched OMP on the reference's own column batch (omp_many_arrays' `ys`,
 * pursuit.py:388-441, before its host transpose at pursuit.py:433): element
 * (i, p) at ys_cols[i * ld + p], ld >= P, fp64 or fp32 (ys_is_f32), HOST
 * memory; staged, transposed on the device and pipelined as in
 * cdb_zero_tree_batch_cols.  eps: P host tolerances, or NULL for
 * rel_tol * ||y_p|| computed on the device (pursuit.py:434-437).  All
 * candidates (no restriction); host outputs as cdb_omp_batch.
 */
cdb_status cdb_omp_batch_cols(const cdb_dictionary *dict, const void *ys_cols, int ys_is_f32,
                              int64_t ld, int64_t p, int64_t k_max, const double *eps,
                              double rel_tol, int64_t *out_sel, double *out_coef,
                              int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                              uint8_t *out_flag, int engine, void *stream);

/*
 * Block-restricted batched OMP: allowed = blocks * q + [0, q)
 * (pursuit.py:417-423, the `allowed_blocks` / `block_q` form).
 * blocks: P x nb int64, each row ascending, 0-based block ids.
 * k_max is the caller's already clipped budget min(K, nb*q, N).
 */
cdb_status cdb_omp_batch_blocked(const cdb_dictionary *dict, const void *ys, int ys_is_f32,
                                 int64_t p, int64_t k_max, const double *eps,
                                 const int64_t *blocks, int64_t nb, int64_t q,
                                 int64_t *out_sel, double *out_coef, int64_t *out_count,
                                 double *out_rnorm, int64_t *out_scans, uint8_t *out_flag,
                                 int engine, void *stream);

/*
 * Masked batched OMP (the per-patch mask operators of
 * crossdict pipelines._recover_operator, pipelines.py:256-322, sensing.py:
 * 222-231): signal p is measured on the m[p] coordinates rows[p][0..m[p])
 * (ascending, int32, row stride N) of the atoms, i.e. OMP over the compacted
 * effective dictionary E_p = D[rows_p, :] with the m[p] measurements in
 * ys[p][0..m[p]) (fp64, row stride N); budget min(k_max, T, m[p]).  Runs the
 * exact engine: selections, coefficients and residuals follow the
 * reference's arithmetic on E_p.
 */
cdb_status cdb_omp_batch_masked(const cdb_dictionary *dict, const double *ys,
                                const int32_t *rows, const int64_t *m, int64_t p, int64_t k_max,
                                const double *eps, int64_t *out_sel, double *out_coef,
                                int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                                uint8_t *out_flag, void *stream);

/*
 * Coded batched OMP (general form; crossdict
 * pipelines._recover_operator pipelines.py:256-322 with sensing.patch_problem
 * sensing.py:205-279, and the Phi zero-tree steps of crossscale.zero_tree_omp
 * crossscale.py:194-222 per patch): signal p is measured through its own
 * operator with m[p] <= m_stride outputs.  Effective row i of signal p sums
 * the atom coordinates rows[(p*m_stride + i)*fan + u], u < fan (fan 1: a
 * gather -- masks, channel mosaics, angular sampling; fan F: a binary
 * temporal code), in numpy's order for the reference's
 * E_p = phi_p.apply_matrix(D): sum_order 0 = sequential over the listed
 * sources (the list ends at the first -1; C-contiguous columns), 1 =
 * numpy's pairwise_sum over all fan slots, -1 slots being 0.0 (the frame
 * axis contiguous: zero-tree step-2 columns, or a single column; fan <= 128).  ys is
 * P x m_stride fp64 (first m[p] used).  blocks (P x nb_max, ascending, or
 * NULL for all T atoms; nb NULL -> nb_max each) restricts the candidates to
 * blocks*q + [0,q) in that order -- the reference's local OMP over
 * D_high[:, allowed] -- and outputs are global atom ids.  Budget
 * min(k_max, candidates, m[p]) per signal.  Exact engine: selections,
 * coefficients, residuals and scans follow the reference's arithmetic.
 * m_stride <= N.  Host or device pointers.
 */
cdb_status cdb_omp_batch_coded(const cdb_dictionary *dict, const double *ys, int64_t m_stride,
                               const int32_t *rows, int64_t fan, int sum_order,
                               const int64_t *m, int64_t p,
                               int64_t k_max, const double *eps, const int64_t *blocks,
                               int64_t nb_max, const int64_t *nb, int64_t q, int64_t *out_sel,
                               double *out_coef, int64_t *out_count, double *out_rnorm,
                               int64_t *out_scans, uint8_t *out_flag, void *stream);

/*
 * K-SVD dictionary-update stage (SURVEY §8 row f1 follow-on; crossdict
 * learn._update_stage, learn.py:169-199): sequential rank-one refits of the
 * T atoms.  y_rows / e_rows: M x N fp64 signal and residual rows (e = y - D X
 * on entry, updated in place); d_rows: T x N atom rows (updated in place);
 * the code matrix X as a per-atom CSR: the users of atom j are
 * atom_sig[atom_ptr[j] .. atom_ptr[j+1]) (ascending signal ids) with values
 * vals[...] (updated in place; dead atoms' entries zeroed); nnz =
 * atom_ptr[T]; max_users = max_j |users_j|.  An atom with fewer than
 * `threshold` users is re-seeded from the not-yet-taken signal with the
 * largest residual norm; the others take the leading singular triple of
 * E_j (sign: largest-magnitude entry of the atom positive; the reference's
 * LAPACK sign is arbitrary).  *replaced = number of re-seeded atoms.
 * N <= ~160 (the Gram matrix of the update lives in shared memory up to
 * there, in global memory beyond).  Host or device pointers.
 */
cdb_status cdb_ksvd_update(int64_t n, int64_t m, int64_t t, const double *y_rows, double *e_rows,
                           double *d_rows, const int64_t *atom_ptr, const int64_t *atom_sig,
                           double *vals, int64_t nnz, int64_t max_users, int64_t threshold,
                           int64_t *replaced, void *stream);

/*
 * Ragged block-restricted batched OMP: signal p may use its first nb[p]
 * block ids of row p of blocks (P x nb_max, ascending within the used
 * prefix); budget min(k_max, nb[p]*q, N) per signal; outputs k_max wide.
 * One call for what crossdict's K-SVD coding stage issues as one
 * cdb_omp_batch_blocked per distinct block count (learn.py:240-262).
 */
cdb_status cdb_omp_batch_blocked_ragged(const cdb_dictionary *dict, const void *ys, int ys_is_f32,
                                        int64_t p, int64_t k_max, const double *eps,
                                        const int64_t *blocks, int64_t nb_max, const int64_t *nb,
                                        int64_t q, int64_t *out_sel, double *out_coef,
                                        int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                                        uint8_t *out_flag, int engine, void *stream);

/*
 * Batched zero-tree OMP.  Replaces crossscale.zero_tree_many_arrays
 * (crossscale.py:235-283) and, with phi_mode != 0, the Phi-composed
 * two-step solve of zero_tree_omp (crossscale.py:169-232) on precomputed
 * effective dictionaries.
 *   low, high      : step-1 / step-2 dictionaries (T_high = q * T_low)
 *   fine_shape, factors, rank : the ScaleSpec (scaling.py:20-61); used for
 *                    the block-mean downsample W y when phi_mode == 0
 *   ys             : P x N rows (N = fine size, or M when phi_mode != 0)
 *   k1             : step-1 budget (k_low, or min(k_low, M, T_low) for Phi)
 *   k_high         : step-2 budget; per signal min(k_high, nb*q, N)
 *   rel_tol        : REL_RESIDUAL_TOL (pursuit.py:37), read at call time by
 *                    the host layer; step-1 tolerances use ||W y|| (identity)
 *   low_*  outputs : width k1;   high_* outputs : width k_high
 * Returns wall-clock-free results; per-step device times (ms) are written to
 * step_ms[2] when non-NULL (the reference's `timings` dict, crossscale.py:283).
 */
cdb_status cdb_zero_tree_batch(const cdb_dictionary *low, const cdb_dictionary *high,
                               const int64_t *fine_shape, const int64_t *factors, int rank,
                               const void *ys, int ys_is_f32, int64_t p,
                               int64_t k1, int64_t k_high, double rel_tol, int phi_mode,
                               int64_t *low_sel, double *low_coef, int64_t *low_count,
                               double *low_rnorm, int64_t *low_scans, uint8_t *low_flag,
                               int64_t *high_sel, double *high_coef, int64_t *high_count,
                               double *high_rnorm, int64_t *high_scans, uint8_t *high_flag,
                               int engine, float *step_ms, void *stream);

/*
 * Batched zero-tree OMP on the reference's own column batch.  Same as
 * cdb_zero_tree_batch, but ys_cols is the N x P (M x P with phi_mode) batch
 * exactly as crossscale.zero_tree_many_arrays receives it (crossscale.py:
 * 235-283; element (i, p) at ys_cols[i * ld + p], ld >= P, fp64 or fp32 when
 * ys_is_f32), in HOST memory (pageable is fine): the transpose the reference
 * makes at pursuit.py:433 happens on the device.  Host threads stage slabs of
 * columns into page-locked memory -- as fp32 when every value is fp32-exact
 * (the engines then read fp32 rows) -- while earlier chunks compute.
 * Outputs as cdb_zero_tree_batch (host or device).
 */
cdb_status cdb_zero_tree_batch_cols(const cdb_dictionary *low, const cdb_dictionary *high,
                                    const int64_t *fine_shape, const int64_t *factors, int rank,
                                    const void *ys_cols, int ys_is_f32, int64_t ld, int64_t p,
                                    int64_t k1, int64_t k_high, double rel_tol, int phi_mode,
                                    int64_t *low_sel, double *low_coef, int64_t *low_count,
                                    double *low_rnorm, int64_t *low_scans, uint8_t *low_flag,
                                    int64_t *high_sel, double *high_coef, int64_t *high_count,
                                    double *high_rnorm, int64_t *high_scans, uint8_t *high_flag,
                                    int engine, float *step_ms, void *stream);

/* Device-time profiler: when enabled, every kernel launch is bracketed by
 * CUDA events on its own stream.  cdb_profile_enable(1) also clears the
 * records.  cdb_profile_read aggregates per kernel name: up to max_entries
 * names (name_len bytes each), total milliseconds and launch counts; it
 * returns the number of distinct kernels recorded. */
void cdb_profile_enable(int on);
int cdb_profile_read(int max_entries, char *names, int name_len, double *ms, int64_t *launches);

/* Test hook: one tcgen05 correlation pass (the tensor engine's scan) on
 * caller residual rows.  rows: P x N fp32 DEVICE; outputs DEVICE: the 8
 * largest |<d_j, bf16(r)>| per row (cand_idx/cand_val, P x 8) and the largest
 * value not kept (cand_drop, P).  grid_cap > 0 limits the persistent grid. */
cdb_status cdb_debug_corr_topk(const cdb_dictionary *dict, const float *rows, int64_t p,
                               int *cand_idx, float *cand_val, float *cand_drop, int grid_cap,
                               void *stream);

/* ---- patch pipeline ends ------------------------------
 * Geometry: a rank-r (1..4) row-major signal of extents signal_shape, patch
 * windows of patch_shape at every multiple of stride (crossdict
 * patchwork.extract_patches, patchwork.py:58-89): P = prod((ext - pe) / st + 1)
 * positions in row-major order, N = prod(patch_shape).
 *
 * cdb_extract_patches: rows_out (P x N fp64, the reference's columns
 * transposed -- the layout cdb_omp_batch / cdb_zero_tree_batch take) and,
 * with remove_dc, the per-patch means dc_out (P) subtracted from the rows.
 * signal fp32 (is_f32) or fp64; every pointer host or device. */
cdb_status cdb_extract_patches(const void *signal, int is_f32, int rank,
                               const int64_t *signal_shape, const int64_t *patch_shape,
                               const int64_t *stride, int remove_dc, double *rows_out,
                               double *dc_out, void *stream);

/* cdb_reconstruct_aggregate: est_p = D_S x_p (+ dc_p when dc != NULL) from a
 * solve's sel / coef rows (P x k_width, sel -1 padded; the atoms of `dict`),
 * then overlap-add averaging into out (signal_shape, fp64): the reference's
 * `dictionary.atoms @ coef` + aggregate_patches(add_dc) (pipelines.py:246,
 * patchwork.py:92-122) without the dense T x P coefficient matrix.  Cells no
 * patch covers are 0; their number goes to *uncovered (host int64). */
cdb_status cdb_reconstruct_aggregate(const cdb_dictionary *dict, const int64_t *sel,
                                     const double *coef, int64_t k_width, int64_t p,
                                     const double *dc, int rank, const int64_t *signal_shape,
                                     const int64_t *patch_shape, const int64_t *stride,
                                     double *out, int64_t *uncovered, void *stream);

/* cdb_aggregate_patches: overlap-add averaging of caller patch values
 * (rows: P x N fp64, the columns transposed; dc != NULL re-adds the means
 * first) -- crossdict aggregate_patches (patchwork.py:92-122). */
cdb_status cdb_aggregate_patches(const double *rows, const double *dc, int rank,
                                 const int64_t *signal_shape, const int64_t *patch_shape,
                                 const int64_t *stride, double *out, int64_t *uncovered,
                                 void *stream);

/* ---- .csd model files (crossdict fileio.py:216-256) ----
 * Layout (little-endian): "CSDM", version u32 (=1), scale count u32 (1 or 2),
 * one record per scale coarse -> fine (patch rank u32, extents u32 x rank,
 * N, T, K, Q u32, atoms fp64 column-major N x T), CRC-32 of every preceding
 * byte.  The column-major atom block is exactly the T x N row layout
 * cdb_dictionary_create takes.
 *
 * cdb_csd_read verifies the CRC before parsing (a mismatch refuses the file,
 * CDB_ERR_CHECKSUM) and every structural rule of the reference loader
 * (CDB_ERR_FORMAT, message as the reference's).  Call it with atoms == NULL
 * to get the scale count and the per-scale geometry; then again with one
 * caller buffer of N*T doubles per scale to receive the atoms (T x N rows). */
typedef struct {
    int32_t rank;
    int64_t extents[4];
    int64_t n, t, k, q;
} cdb_csd_scale;
cdb_status cdb_csd_read(const char *path, int32_t *scale_count, cdb_csd_scale *scales,
                        double *const *atoms_t);
/* The same parse over an in-memory file image (read the file once, parse the
 * header, size the buffers, parse the same bytes again: no window for the file
 * to change between the calls).  capacity[s] (optional): doubles available in
 * atoms_t[s]; a scale larger than its buffer is refused (CDB_ERR_ARG). */
cdb_status cdb_csd_parse(const uint8_t *data, int64_t size, const char *name,
                         int32_t *scale_count, cdb_csd_scale *scales, double *const *atoms_t,
                         const int64_t *capacity);

/* Host layout helper: rows[j][i] = cols[i][j] for an n x p column batch (the
 * reference's N x P signal matrix) into p x n rows (the kernel layout; the
 * copy crossdict makes at pursuit.py:433).  elem_size 4 or 8; blocked and
 * split over `threads` host threads (<= 0: all cores).  Writing into pinned
 * memory lets the batch calls pipeline their host copies. */
cdb_status cdb_rows_from_cols(const void *cols, int64_t n, int64_t p, int elem_size, void *rows,
                              int threads);

/* 1 when two host buffers hold the same nbytes bytes, else 0 (memcmp split over
 * `threads` host threads, <= 0: all cores).  The host layer confirms a cached
 * device dictionary against its stored host copy with it, so a matrix the
 * caller changed in place (pursuit.py:84-94 keeps no such cache: the reference
 * re-reads `columns` on every call) is staged again. */
int cdb_host_equal(const void *a, const void *b, int64_t nbytes, int threads);

/* Number of kernels this library has launched since load (instrumentation). */
int64_t cdb_launch_count(void);

/* Engine used by the last OMP pass on this thread, how many of its signals
 * were handed to the exact engine, and how many picks needed an inline exact
 * rescan (tensor engine) -- instrumentation. */
void cdb_last_run_info(int *engine, int *delegated, int *rescans);

#ifdef __cplusplus
}
#endif

#endif /* CROSSDICT_B200_H */
