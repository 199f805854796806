// C ABI (include/crossdict_b200.h): dictionary staging, engine selection and
// the batched OMP / zero-tree drivers.  Host code only; kernels live in the
// *_engine.cu / helpers.cu translation units.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <string>
#include <array>
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>
#include <algorithm>

#include "../../include/crossdict_b200.h"
#include "engines.h"

struct cdb_dictionary {
  int64_t t = 0, n = 0, n_pad = 0;
  double *d64 = nullptr;   // T x N fp64 atoms (rows)
  double *gram = nullptr;  // T x T fp64 (optional)
  void *d16 = nullptr;     // T x n_pad fp16(dscale * d) (tensor-core operand)
  float *d32 = nullptr;    // T x N fp32 (residual materialisation of the scan operand)
  double dmax = 0.0;       // largest atom norm
  double emax = 0.0;       // largest |fp16(dscale d_j) / dscale - d_j| (tensor-engine certification)
  double dscale = 1.0;     // power of two: the largest atom norm lands in [2^8, 2^9)
  int64_t bytes = 0;
  int device = -1;         // CUDA device holding the arrays
};

namespace {

thread_local std::string g_last_error;
thread_local int g_last_engine = 0;     // engine the last run_omp used
// delegated / rescan counts of the last run_omp live in a persistent device
// buffer that the kernels count into; only cdb_last_run_info copies them to
// the host (after a device sync).  No copy is ever queued on the compute
// stream: a small D2H there would wait behind a pipeline's output copies on
// the copy engine and stall the next chunk.
// per thread and per device: [0] delegated, [1] rescans
constexpr int kMaxDevices = 64;
thread_local int *g_diag_per_dev[kMaxDevices] = {};
thread_local int *g_diag = nullptr;  // the current device's counters
int *diag_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int *&slot = g_diag_per_dev[dev];
  if (!slot) {
    cudaMalloc((void **)&slot, 2 * sizeof(int));
    cudaMemset(slot, 0, 2 * sizeof(int));
  }
  g_diag = slot;
  return slot;
}
void diag_clear(cudaStream_t st) { cudaMemsetAsync(diag_dev(), 0, 2 * sizeof(int), st); }
std::atomic<int64_t> g_launches{0};

cdb_status fail(cdb_status st, const std::string &msg) {
  g_last_error = msg;
  return st;
}

#define CDB_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(CDB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
  } while (0)

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Stream-ordered device scratch that frees itself.
struct DevBuf {
  void *ptr = nullptr;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  ~DevBuf() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
  cudaError_t alloc(size_t bytes, cudaStream_t s) {
    stream = s;
    if (bytes == 0) bytes = 16;
    return cudaMallocAsync(&ptr, bytes, s);
  }
  template <typename T>
  T *as() const {
    return (T *)ptr;
  }
};

// An input array usable on the device (copied when it lives on the host).
struct InArr {
  const void *dev = nullptr;
  DevBuf buf;
  cudaError_t bind(const void *p, size_t bytes, cudaStream_t s) {
    if (!p || is_device_ptr(p)) {
      dev = p;
      return cudaSuccess;
    }
    cudaError_t e = buf.alloc(bytes, s);
    if (e != cudaSuccess) return e;
    dev = buf.ptr;
    return cudaMemcpyAsync(buf.ptr, p, bytes, cudaMemcpyHostToDevice, s);
  }
};

// An output array written on the device and copied back when host-resident.
struct OutArr {
  void *host = nullptr;
  void *dev = nullptr;
  size_t bytes = 0;
  DevBuf buf;
  cudaError_t bind(void *p, size_t nbytes, cudaStream_t s) {
    bytes = nbytes;
    if (p && is_device_ptr(p)) {
      dev = p;
      return cudaSuccess;
    }
    host = p;
    cudaError_t e = buf.alloc(nbytes, s);
    dev = buf.ptr;
    return e;
  }
  cudaError_t finish(cudaStream_t s) {
    if (!host || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
  }
};

// An array read and written on the device: copied in, and back when host-resident.
struct IoArr {
  void *host = nullptr;
  void *dev = nullptr;
  size_t bytes = 0;
  DevBuf buf;
  cudaError_t bind(void *p, size_t nbytes, cudaStream_t s) {
    bytes = nbytes;
    if (!p || is_device_ptr(p)) {
      dev = p;
      return cudaSuccess;
    }
    host = p;
    cudaError_t e = buf.alloc(nbytes, s);
    if (e != cudaSuccess) return e;
    dev = buf.ptr;
    return cudaMemcpyAsync(dev, p, nbytes, cudaMemcpyHostToDevice, s);
  }
  cudaError_t finish(cudaStream_t s) {
    if (!host || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
  }
};

struct Outs {
  OutArr sel, coef, count, rnorm, scans, flag;
  cudaError_t bind(int64_t p, int64_t kw, int64_t *s, double *c, int64_t *cnt, double *rn,
                   int64_t *sc, uint8_t *fl, cudaStream_t st) {
    cudaError_t e;
    if ((e = sel.bind(s, sizeof(int64_t) * p * kw, st)) != cudaSuccess) return e;
    if ((e = coef.bind(c, sizeof(double) * p * kw, st)) != cudaSuccess) return e;
    if ((e = count.bind(cnt, sizeof(int64_t) * p, st)) != cudaSuccess) return e;
    if ((e = rnorm.bind(rn, sizeof(double) * p, st)) != cudaSuccess) return e;
    if ((e = scans.bind(sc, sizeof(int64_t) * p, st)) != cudaSuccess) return e;
    return flag.bind(fl, sizeof(uint8_t) * p, st);
  }
  cudaError_t finish(cudaStream_t st) {
    cudaError_t e;
    for (OutArr *o : {&sel, &coef, &count, &rnorm, &scans, &flag})
      if ((e = o->finish(st)) != cudaSuccess) return e;
    return cudaSuccess;
  }
  bool any_host() const {
    return sel.host || coef.host || count.host || rnorm.host || scans.host || flag.host;
  }
};

struct DevInfo {
  int sms = 0, smem_optin = 0, major = 0, minor = 0;
};

cdb_status device_info(DevInfo &di) {
  int dev = 0;
  CDB_CUDA(cudaGetDevice(&dev));
  static int pool_configured = -1;
  if (pool_configured != dev) {
    // keep freed stream-ordered scratch cached in the pool: the engines
    // allocate hundreds of MB of state per call
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_configured = dev;
  }
  CDB_CUDA(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
  CDB_CUDA(cudaDeviceGetAttribute(&di.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  CDB_CUDA(cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, dev));
  CDB_CUDA(cudaDeviceGetAttribute(&di.minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (di.major != 10) return fail(CDB_ERR_NODEV, "device is not sm_100 (B200)");
  return CDB_OK;
}

constexpr int64_t kGramSmemLimit = 100 * 1024;       // per-warp smem for H in smem
constexpr int64_t kGramPreferBytes = 24 * 1024;      // auto: gram over resident below this
constexpr int64_t kScratchBudget = int64_t(4) << 30;  // per-call global scratch cap

// Warps per SM for exact-engine launches: the kernel is latency-bound (a warp
// per signal), so as many as its registers allow (CDB_EXACT_WPS overrides).
int64_t exact_warps_per_sm() {
  static const int64_t w = getenv("CDB_EXACT_WPS") ? atoll(getenv("CDB_EXACT_WPS")) : 16;
  return w > 0 ? w : 16;
}

// Run the exact engine over `count` signals (all, or the ids in sig_ids).
cdb_status run_exact(const cdb_dictionary *d, const void *ys, bool f32, int64_t count,
                     const int64_t *sig_ids, int64_t k_max, int64_t kw, const double *eps,
                     const cdb::Cands &cands, int64_t max_cands, Outs &o, const DevInfo &di,
                     cudaStream_t st, const int *count_dev = nullptr,
                     const int32_t *rows = nullptr, const int64_t *m_sig = nullptr,
                     int fan = 1, int64_t m_stride = 0, int sum_order = 0) {
  if (count <= 0) return CDB_OK;
  cdb::ExactArgs a{};
  a.mat_t = d->d64;
  a.t = d->t;
  a.n = d->n;
  a.ys_stride = rows ? m_stride : d->n;
  a.sig_ids = sig_ids;
  a.p_count = count;
  a.p_count_dev = count_dev;
  a.rows = rows;
  a.m_sig = m_sig;
  a.fan = fan;
  a.sum_order = sum_order;
  a.rows_stride = m_stride * fan;
  a.k_max = k_max;
  a.k_width = kw;
  a.eps = eps;
  a.cands = cands;
  a.out_sel = o.sel.dev ? (int64_t *)o.sel.dev : nullptr;
  a.out_coef = (double *)o.coef.dev;
  a.out_count = (int64_t *)o.count.dev;
  a.out_rnorm = (double *)o.rnorm.dev;
  a.out_scans = (int64_t *)o.scans.dev;
  a.out_flag = (uint8_t *)o.flag.dev;
  a.work_stride = cdb::exact_work_stride(d->n, kw, max_cands);
  // a device-side count is usually tiny (delegations are rare): few warps
  const int64_t wmax = count_dev ? (int64_t)di.sms : (int64_t)di.sms * exact_warps_per_sm();
  int64_t warps = count < wmax ? count : wmax;
  const int64_t cap = kScratchBudget / (8 * a.work_stride);
  if (warps > cap) warps = cap < 4 ? 4 : cap;
  warps = (warps + 3) & ~int64_t(3);
  DevBuf work;
  CDB_CUDA(work.alloc(sizeof(double) * a.work_stride * warps, st));
  a.work = work.as<double>();
  CDB_CUDA(cdb::launch_exact(a, ys, f32, (int)warps, st));
  return CDB_OK;
}

// Signals an engine handed over (status ST_DELEGATE) -> exact engine.  The
// count stays on the device: the exact kernel reads it, so nothing here
// waits for the GPU (a host-buffer pipeline keeps queueing chunks).
cdb_status finish_delegates(const cdb_dictionary *d, const void *ys, bool f32, int64_t p,
                            int64_t k_max, int64_t kw, const double *eps, const cdb::Cands &cands,
                            int64_t max_cands, Outs &o, const uint32_t *status, const DevInfo &di,
                            cudaStream_t st) {
  DevBuf ids;
  CDB_CUDA(ids.alloc(sizeof(int64_t) * p, st));
  int *cnt = diag_dev();  // [0]: zeroed by run_omp's diag_clear
  CDB_CUDA(cdb::launch_collect_delegates(status, p, ids.as<int64_t>(), cnt, st));
  return run_exact(d, ys, f32, p, ids.as<int64_t>(), k_max, kw, eps, cands, max_cands, o, di, st,
                   cnt);
}

cdb_status run_tensor(const cdb_dictionary *d, const void *ys, bool f32, int64_t p, int64_t k_max,
                      int64_t kw, const double *eps, const cdb::Cands &cands, Outs &o,
                      const DevInfo &di, cudaStream_t st) {
  DevBuf status;
  CDB_CUDA(status.alloc(sizeof(uint32_t) * p, st));
  CDB_CUDA(cudaMemsetAsync(status.ptr, 0, sizeof(uint32_t) * p, st));
  const int64_t per = cdb::tensor_state_bytes(1 << 16, d->n, kw) / (1 << 16) + 1;
  // State per chunk.  When the fp16 dictionary operand stays L2-resident
  // (<= 32 MiB: every zero-tree step 1) a quarter of the device memory
  // (45 GB on a B200, capped at 48 GiB): configs[4] step 1 on 1M signals is one
  // 34 GB chunk instead of nine 4 GiB chunks -- 64 instead of 576 launches of
  // every per-iteration kernel and no partial waves between chunks (1.747 ->
  // 1.650 s per 1M signals).  A scan that streams its dictionary from HBM
  // (configs[4] full OMP, 128 MB) keeps 4 GiB chunks: the CTAs sharing a
  // dictionary part drift apart over a long launch and lose the L2 reuse
  // (corr_topk 7.9 -> 9.3 s per 1M signals in one chunk).
  // CDB_TENSOR_SCRATCH_GB overrides; an allocation that fails is retried at
  // half the size.
  int64_t budget = kScratchBudget;
  if (2 * d->t * d->n_pad <= (int64_t(32) << 20)) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
      budget = std::min<int64_t>(std::max<int64_t>((int64_t)(total_b / 4), kScratchBudget),
                                 int64_t(48) << 30);
    else
      cudaGetLastError();
  }
  if (const char *v = getenv("CDB_TENSOR_SCRATCH_GB")) {  // A/B switch: state per chunk
    const int64_t gb = atoll(v);
    if (gb >= 1 && gb <= 64) budget = gb << 30;
  }
  int64_t chunk = 0;
  DevBuf work;
  for (;; budget /= 2) {
    chunk = budget / per;
    if (chunk < 128) chunk = 128;
    if (chunk > p) chunk = p;
    const cudaError_t ae =
        work.alloc((size_t)cdb::tensor_state_bytes(chunk, d->n, kw) + 65536, st);
    if (ae == cudaSuccess) break;
    work.ptr = nullptr;
    cudaGetLastError();  // clear the allocation failure before the smaller retry
    if (ae != cudaErrorMemoryAllocation || chunk <= 128 || budget <= (int64_t(1) << 28))
      return fail(CDB_ERR_NOMEM, "tensor engine state allocation");
  }
  const size_t ysz = f32 ? 4 : 8;
  for (int64_t off = 0; off < p; off += chunk) {
    cdb::TensorArgs a{};
    a.p = (p - off) < chunk ? (p - off) : chunk;
    a.ys = (const uint8_t *)ys + off * d->n * ysz;
    a.ys_f32 = f32;
    a.n = d->n;
    a.n_pad = d->n_pad;
    a.t = d->t;
    a.k_max = k_max;
    a.k_width = kw;
    a.eps = eps + off;
    a.d64 = d->d64;
    a.d16 = d->d16;
    a.d32 = d->d32;
    a.gram = d->gram;
    a.rescans = diag_dev() + 1;  // zeroed by run_omp's diag_clear
    a.dmax = d->dmax;
    a.emax = d->emax;
    a.dscale = d->dscale;
    a.out_sel = (int64_t *)o.sel.dev + off * kw;
    a.out_coef = (double *)o.coef.dev + off * kw;
    a.out_count = (int64_t *)o.count.dev + off;
    a.out_rnorm = (double *)o.rnorm.dev + off;
    a.out_scans = (int64_t *)o.scans.dev + off;
    a.out_flag = (uint8_t *)o.flag.dev + off;
    a.status = status.as<uint32_t>() + off;
    a.work = work.ptr;
    a.num_sms = di.sms;
    CDB_CUDA(cdb::run_tensor_chunk(a, st));
  }
  return finish_delegates(d, ys, f32, p, k_max, kw, eps, cands, d->t, o, status.as<uint32_t>(),
                          di, st);
}

// The Gram engine beats the resident one when its per-signal state is small
// (>= ~13 signals per SM: cfg 0 full 32.7 vs 28.3 M/s, both steps of cfg 0's
// zero-tree); with a larger H (cfg 1 step 1: 32 KB per signal) resident wins.
// Full-dictionary scans whose Gram-engine state leaves at most four signals per
// SM go to the tensor engine when the batch is large enough to amortise its
// per-iteration launches (cfg 3 zero-tree step 1: T_low = 256, K = 24, 50 KB of H
// per signal: 19.2 -> 14.1 ms per 100 k signals, zero-tree 3.13 M -> 3.73 M/s).
constexpr int64_t kTensorPreferBytes = 40 * 1024;
constexpr int64_t kTensorPreferSignals = 16384;

bool gram_preferred(const cdb_dictionary *d, int64_t max_cands, int64_t kw) {
  return d->gram && max_cands > 0 && max_cands <= 512 && kw <= 64 &&
         cdb::gram_total_smem(max_cands, kw, d->n, true) <= kGramPreferBytes;
}

// The OMP driver shared by every entry point: picks the engine.
//   exact  : any problem (reference restatement)
//   gram   : Gram matrix available; H (max_cands x k) kept in smem when it fits
//   tensor : full-dictionary scans (mode 0) with a Gram matrix
// auto = gram when H fits in shared memory (small candidate sets: zero-tree
// steps, small dictionaries), tensor for large full-dictionary scans.
cdb_status run_omp(const cdb_dictionary *d, const void *ys, bool f32, int64_t p, int64_t k_max,
                   int64_t kw, const double *eps, const cdb::Cands &cands, int64_t max_cands,
                   Outs &o, int engine, const DevInfo &di, cudaStream_t st,
                   const char *tag = nullptr, const double *alpha0 = nullptr) {
  if (p <= 0) return CDB_OK;
  static const bool force_onchip = getenv("CDB_GRAM_ONCHIP") && atoi(getenv("CDB_GRAM_ONCHIP")) != 0;
  const bool h_smem = cdb::gram_total_smem(max_cands, kw, d->n, true) <= kGramSmemLimit &&
                      !(force_onchip && alpha0 && max_cands > 128) &&
                      !cdb::gram_cta_preferred(max_cands, kw, d->n, alpha0 != nullptr);
  const bool resident = cdb::resident_fits(d->n, d->t, kw, max_cands, di.smem_optin);
  if (engine == CDB_ENGINE_RESIDENT && !resident) engine = CDB_ENGINE_AUTO;  // a preference
  const bool gram_small = gram_preferred(d, max_cands, kw);
  if (engine == CDB_ENGINE_AUTO) {
    if (resident && max_cands > 0 && !gram_small)
      engine = CDB_ENGINE_RESIDENT;
    else if (!d->gram || max_cands <= 0)
      engine = CDB_ENGINE_EXACT;
    else if (h_smem && !(cands.mode == 0 && p >= kTensorPreferSignals &&
                         cdb::gram_total_smem(max_cands, kw, d->n, true) > kTensorPreferBytes))
      engine = CDB_ENGINE_GRAM;
    else if (cands.mode == 0)
      engine = CDB_ENGINE_TENSOR;
    else
      engine = CDB_ENGINE_GRAM;
  }
  if ((engine == CDB_ENGINE_GRAM || engine == CDB_ENGINE_TENSOR) && !d->gram)
    return fail(CDB_ERR_ARG, "engine needs the dictionary's Gram matrix (raise the budget)");
  if (engine == CDB_ENGINE_TENSOR && cands.mode != 0) engine = CDB_ENGINE_GRAM;
  if (engine == CDB_ENGINE_GRAM && (max_cands > 512 || kw > 64))  // beyond the Gram kernel's tiles
    engine = cands.mode == 0 ? CDB_ENGINE_TENSOR : CDB_ENGINE_EXACT;
  g_last_engine = engine;
  diag_clear(st);
  if (engine == CDB_ENGINE_EXACT)
    return run_exact(d, ys, f32, p, nullptr, k_max, kw, eps, cands, max_cands, o, di, st);
  if (engine == CDB_ENGINE_TENSOR) return run_tensor(d, ys, f32, p, k_max, kw, eps, cands, o, di, st);
  if (engine == CDB_ENGINE_RESIDENT) {
    if (!resident) return fail(CDB_ERR_ARG, "dictionary too large for the resident engine");
    DevBuf status;
    CDB_CUDA(status.alloc(sizeof(uint32_t) * p, st));
    CDB_CUDA(cudaMemsetAsync(status.ptr, 0, sizeof(uint32_t) * p, st));
    cdb::ResidentArgs r{};
    r.d64 = d->d64;
    r.gram = d->gram;
    r.t = d->t;
    r.n = d->n;
    r.p = p;
    r.k_max = k_max;
    r.k_width = kw;
    r.eps = eps;
    r.cands = cands;
    r.max_cands = max_cands;
    r.out_sel = (int64_t *)o.sel.dev;
    r.out_coef = (double *)o.coef.dev;
    r.out_count = (int64_t *)o.count.dev;
    r.out_rnorm = (double *)o.rnorm.dev;
    r.out_scans = (int64_t *)o.scans.dev;
    r.out_flag = (uint8_t *)o.flag.dev;
    r.status = status.as<uint32_t>();
    r.tag = tag ? (std::string(tag) == "gram_step1" ? "resident_step1" : "resident_step2") : nullptr;
    CDB_CUDA(cdb::launch_resident(r, ys, f32, di.smem_optin, di.sms, st));
    return finish_delegates(d, ys, f32, p, k_max, kw, eps, cands, max_cands, o,
                            status.as<uint32_t>(), di, st);
  }

  DevBuf status;
  CDB_CUDA(status.alloc(sizeof(uint32_t) * p, st));
  CDB_CUDA(cudaMemsetAsync(status.ptr, 0, sizeof(uint32_t) * p, st));
  cdb::GramArgs g{};
  g.d64 = d->d64;
  g.gram = d->gram;
  g.t = d->t;
  g.n = d->n;
  g.ys_stride = d->n;
  g.k_max = k_max;
  g.k_width = kw;
  g.eps = eps;
  g.cands = cands;
  g.max_cands = max_cands;
  g.out_sel = (int64_t *)o.sel.dev;
  g.out_coef = (double *)o.coef.dev;
  g.out_count = (int64_t *)o.count.dev;
  g.out_rnorm = (double *)o.rnorm.dev;
  g.out_scans = (int64_t *)o.scans.dev;
  g.out_flag = (uint8_t *)o.flag.dev;
  g.status = status.as<uint32_t>();
  g.tag = tag;
  g.alpha0_in = alpha0;
  g.prefetch_runner = getenv("CDB_GRAM_PF") ? atoi(getenv("CDB_GRAM_PF")) : 0;
  DevBuf hwork;
  if (!h_smem) {  // streamed H: one L2-resident slot per persistent warp
    const cdb::GramStreamPlan pl = cdb::gram_stream_plan(max_cands, kw, d->n, alpha0 == nullptr,
                                                         di.smem_optin, di.sms);
    if (!pl.ok) return fail(CDB_ERR_ARG, "Gram engine: no shared-memory plan for this H");
    CDB_CUDA(hwork.alloc((size_t)(8 * pl.warps * (pl.slot_doubles > 0 ? pl.slot_doubles : 1)), st));
    g.hwork = hwork.as<double>();
  }
  g.p_offset = 0;
  g.p = p;
  CDB_CUDA(cdb::launch_gram(g, ys, f32, di.smem_optin, di.sms, st));
  return finish_delegates(d, ys, f32, p, k_max, kw, eps, cands, max_cands, o,
                          status.as<uint32_t>(), di, st);
}


// ---------------------------------------------------------------- host-buffer pipelining
// Row-major per-signal arrays crossing the host boundary: the batch is coded
// in chunks; chunk i+1's inputs go H2D on one copy stream and chunk i-1's
// outputs D2H on another (PCIe is full duplex) while chunk i computes on the
// caller's stream.  Two device buffer sets; events order every reuse, and
// nothing waits on the host until the end, so the GPU never idles between
// chunks.  Chunk sizes ramp up and down (small first and last chunks) to
// shrink the copies that cannot overlap compute.  Requires pinned host
// memory for the copies to be asynchronous; pageable memory still works.
struct RowArr {
  void *host;        // host base pointer (or device, then passed through)
  size_t row_bytes;  // bytes per signal
  bool out;          // output (D2H) or input (H2D)
};

cudaStream_t copy_stream(int which) {
  static thread_local cudaStream_t cs[2] = {nullptr, nullptr};
  static thread_local int dev = -1;
  int cur = 0;
  cudaGetDevice(&cur);
  if (!cs[0] || dev != cur) {
    cudaStreamCreateWithFlags(&cs[0], cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&cs[1], cudaStreamNonBlocking);
    dev = cur;
  }
  return cs[which];
}

// Chunk boundaries: a small first chunk (its H2D cannot overlap compute) and
// a small last chunk (its D2H cannot), and the rest in as few chunks as
// possible -- each call carries ~0.1-0.3 ms of fixed cost (launch gaps,
// partial waves), so many small chunks lose more than they hide.
// kind 0: zero-tree calls; kind 1: OMP batches (the tensor engine's 16-
// iteration chunks carry more fixed cost, so fewer, larger chunks).
std::vector<int64_t> chunk_bounds(int64_t p, int kind) {
  if (const char *sched = getenv("CDB_PIPE_SCHEDULE")) {  // "w1,w2,...": relative chunk sizes
    std::vector<double> w;
    double tot = 0.0;
    for (const char *c = sched; *c;) {
      const double v = atof(c);
      if (v > 0) {
        w.push_back(v);
        tot += v;
      }
      while (*c && *c != ',') c++;
      if (*c == ',') c++;
    }
    if (!w.empty()) {
      std::vector<int64_t> b = {0};
      double acc = 0.0;
      for (double x : w) {
        acc += x;
        const int64_t e = (int64_t)(p * acc / tot);
        if (e > b.back()) b.push_back(e);
      }
      b.back() = p;
      return b;
    }
  }
  if (p >= 50000 && !getenv("CDB_PIPE_CHUNK") && !getenv("CDB_PIPE_EDGE")) {
    // measured best for 100k: zero-tree ~9.5% first chunk (its H2D is
    // exposed), two middle chunks, ~10% last (5.85 vs 6.0 ms for [20k, 60k,
    // 20k]); full OMP 15% / 85% (8.96 vs 9.20 ms for [20k, 60k, 20k], 10.6 ms
    // with the zero-tree ramp)
    static const double wz[4] = {0.0947, 0.4262, 0.3789, 0.1002};
    static const double wo[2] = {0.15, 0.85};
    const double *w = kind == 0 ? wz : wo;
    const int nw = kind == 0 ? 4 : 2;
    std::vector<int64_t> b = {0};
    double acc = 0.0;
    for (int i = 0; i < nw; i++) {
      acc += w[i];
      b.push_back((int64_t)(p * acc));
    }
    b.back() = p;
    return b;
  }
  static const int64_t mid_max = getenv("CDB_PIPE_CHUNK") ? atoll(getenv("CDB_PIPE_CHUNK")) : 90000;
  static const int64_t edge_max = getenv("CDB_PIPE_EDGE") ? atoll(getenv("CDB_PIPE_EDGE")) : 20000;
  int64_t edge = p / 5;
  if (edge > edge_max) edge = edge_max;
  std::vector<int64_t> b = {0};
  if (edge < 2048 || p < 4 * edge) {  // too small to bother: two halves
    b.push_back(p / 2);
    b.push_back(p);
    return b;
  }
  b.push_back(edge);
  const int64_t mid = p - 2 * edge;
  const int64_t nm = (mid + mid_max - 1) / mid_max;
  for (int64_t i = 1; i < nm; i++) b.push_back(edge + mid * i / nm);
  b.push_back(p - edge);
  b.push_back(p);
  return b;
}

// A dictionary is usable only on the device it was staged on.
cdb_status check_device(const cdb_dictionary *d) {
  int dev = -1;
  cudaGetDevice(&dev);
  if (d && d->device != dev)
    return fail(CDB_ERR_ARG, "dictionary was staged on device " + std::to_string(d->device) +
                                 ", current device is " + std::to_string(dev));
  return CDB_OK;
}

// The pipeline copies every array with explicit H2D / D2H kinds, so it is
// taken only when every array given is host memory (mixed host / device
// argument sets go through the per-array staging of OutArr instead).
bool all_host(const std::vector<RowArr> &arrs) {
  for (const RowArr &a : arrs)
    if (a.host && is_device_ptr(a.host)) return false;
  return true;
}

template <typename Core>
cdb_status run_pipelined(int64_t p, std::vector<RowArr> &arrs, cudaStream_t st, Core core,
                          int kind = 0) {
  const std::vector<int64_t> bd = chunk_bounds(p, kind);
  const int64_t nch = (int64_t)bd.size() - 1;
  int64_t chunk = 0;
  for (int64_t i = 0; i < nch; i++) chunk = std::max(chunk, bd[i + 1] - bd[i]);
  cudaStream_t cin = copy_stream(0), cout = copy_stream(1);
  const size_t na = arrs.size();
  std::vector<DevBuf> bufs(2 * na);
  for (int b = 0; b < 2; b++)
    for (size_t a = 0; a < na; a++)
      CDB_CUDA(bufs[b * na + a].alloc(arrs[a].row_bytes * chunk, st));
  cudaEvent_t ready, in_ready[2], done[2], out_done[2];
  CDB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  for (int b = 0; b < 2; b++) {
    CDB_CUDA(cudaEventCreateWithFlags(&in_ready[b], cudaEventDisableTiming));
    CDB_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    CDB_CUDA(cudaEventCreateWithFlags(&out_done[b], cudaEventDisableTiming));
  }
  CDB_CUDA(cudaEventRecord(ready, st));  // buffers allocated (stream-ordered)
  CDB_CUDA(cudaStreamWaitEvent(cin, ready, 0));
  CDB_CUDA(cudaStreamWaitEvent(cout, ready, 0));
  bool out_pending[2] = {false, false};
  auto h2d = [&](int64_t i) -> cudaError_t {
    const int b = (int)(i & 1);
    const int64_t off = bd[i], len = bd[i + 1] - bd[i];
    cudaError_t e;
    if (out_pending[b] && (e = cudaStreamWaitEvent(cin, out_done[b], 0)) != cudaSuccess) return e;
    for (size_t a = 0; a < na; a++) {
      if (arrs[a].out || !arrs[a].host) continue;
      e = cudaMemcpyAsync(bufs[b * na + a].ptr,
                          (const uint8_t *)arrs[a].host + off * arrs[a].row_bytes,
                          len * arrs[a].row_bytes, cudaMemcpyHostToDevice, cin);
      if (e != cudaSuccess) return e;
    }
    return cudaEventRecord(in_ready[b], cin);
  };
  static const bool trace = getenv("CDB_PIPE_TRACE") != nullptr;
  auto now_us = [] {
    return (double)std::chrono::duration_cast<std::chrono::microseconds>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t_start = now_us();
  // trace: GPU timestamps of h2d start/end, compute start/end, d2h start/end
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t s_) {
    if (!trace) return -1;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s_);
    tev.push_back(e);
    return (int)tev.size() - 1;
  };
  const int t0ev = tmark(st);
  cdb_status result = CDB_OK;
  cudaError_t ce = h2d(0);
  for (int64_t i = 0; i < nch && ce == cudaSuccess && result == CDB_OK; i++) {
    const int b = (int)(i & 1);
    const int64_t off = bd[i], len = bd[i + 1] - bd[i];
    if (i + 1 < nch && (ce = h2d(i + 1)) != cudaSuccess) break;
    if ((ce = cudaStreamWaitEvent(st, in_ready[b], 0)) != cudaSuccess) break;
    tmark(st);
    std::vector<void *> dev(na);
    for (size_t a = 0; a < na; a++) dev[a] = bufs[b * na + a].ptr;
    result = core(off, len, dev, st);
    if (result != CDB_OK) break;
    if ((ce = cudaEventRecord(done[b], st)) != cudaSuccess) break;
    tmark(st);
    if ((ce = cudaStreamWaitEvent(cout, done[b], 0)) != cudaSuccess) break;
    for (size_t a = 0; a < na && ce == cudaSuccess; a++) {
      if (!arrs[a].out || !arrs[a].host) continue;
      ce = cudaMemcpyAsync((uint8_t *)arrs[a].host + off * arrs[a].row_bytes, dev[a],
                           len * arrs[a].row_bytes, cudaMemcpyDeviceToHost, cout);
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(out_done[b], cout);
    tmark(cout);
    out_pending[b] = true;
    if (trace) fprintf(stderr, "[pipe] chunk %lld len %lld issued at %.0f us\n", (long long)i,
                       (long long)len, now_us() - t_start);
  }
  cudaError_t e1 = cudaStreamSynchronize(cin), e2 = cudaStreamSynchronize(cout);
  cudaError_t e3 = cudaStreamSynchronize(st);
  if (trace) {
    fprintf(stderr, "[pipe] all done at %.0f us; GPU (compute start, compute end, d2h end) ms:",
            now_us() - t_start);
    for (size_t k = 1; k < tev.size(); k++) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, tev[t0ev], tev[k]);
      fprintf(stderr, " %.3f", ms);
    }
    fprintf(stderr, "\n");
    for (auto e : tev) cudaEventDestroy(e);
  }
  cudaEventDestroy(ready);
  for (int b = 0; b < 2; b++) {
    cudaEventDestroy(in_ready[b]);
    cudaEventDestroy(done[b]);
    cudaEventDestroy(out_done[b]);
  }
  if (result != CDB_OK) return result;
  for (cudaError_t e : {ce, e1, e2, e3})
    if (e != cudaSuccess) return fail(CDB_ERR_CUDA, cudaGetErrorString(e));
  return CDB_OK;
}

// ---------------------------------------------------------------- column batches
// The reference hands its batch over as N x P columns (zero_tree_many_arrays'
// and omp_many_arrays' `ys`) and transposes it to rows on the host
// (pursuit.py:433) before the numba kernel.  run_pipelined_cols keeps that
// layout across the boundary: host threads gather slabs of whole columns
// (for each of the N coordinates one contiguous run of the slab's signals)
// into page-locked staging -- as fp32 when every value is fp32-exact, which
// halves the copy and lets the engines read fp32 rows -- a 2-D copy puts the
// slab into the chunk's N x len device block, and the device transposes the
// block into rows (cols_to_rows_kernel) right before the chunk's compute.
// While chunk c computes, the host stages chunk c+1; chunk sizes grow
// geometrically from a small first chunk (the only staging nothing hides).
constexpr int kSlabs = 3;
constexpr size_t kSlabBytes = size_t(64) << 20;

struct PinnedSlabs {  // process-wide, allocated once
  void *base = nullptr;
  cudaError_t get(void **out) {
    if (!base) {
      cudaError_t e = cudaHostAlloc(&base, kSlabs * kSlabBytes, cudaHostAllocPortable);
      if (e != cudaSuccess) {
        base = nullptr;
        return e;
      }
    }
    *out = base;
    return cudaSuccess;
  }
};
PinnedSlabs g_slabs;
std::mutex g_slabs_mu;  // one column pipeline at a time uses the staging

int stage_threads() {
  static const int t = [] {
    if (const char *v = getenv("CDB_STAGE_THREADS")) return std::max(1, atoi(v));
    return (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
  }();
  return t;
}

// Columns [a, a + s) of an n-row column batch (row stride ld elements) into
// dst as an n x s block.  to_f32 (fp64 source only): converted to fp32;
// returns false when some value is not fp32-exact (dst is then garbage).
bool stage_cols(const void *src, bool src_f32, int64_t n, int64_t ld, int64_t a, int64_t s,
                void *dst, bool to_f32) {
  int threads = stage_threads();
  if (threads > n) threads = (int)n;
  std::atomic<bool> exact{true};
  auto work = [&](int tid) {
    const int64_t i0 = n * tid / threads, i1 = n * (tid + 1) / threads;
    unsigned bad = 0;
    for (int64_t i = i0; i < i1; i++) {
      if (src_f32) {
        memcpy((float *)dst + i * s, (const float *)src + i * ld + a, sizeof(float) * s);
      } else if (!to_f32) {
        memcpy((double *)dst + i * s, (const double *)src + i * ld + a, sizeof(double) * s);
      } else {
        const double *r = (const double *)src + i * ld + a;
        float *o = (float *)dst + i * s;
        for (int64_t j = 0; j < s; j++) {
          const float f = (float)r[j];
          o[j] = f;
          bad |= (unsigned)((double)f != r[j]);  // NaN / out of range: inexact
        }
      }
    }
    if (bad) exact.store(false, std::memory_order_relaxed);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; t++) pool.emplace_back(work, t);
  work(0);
  for (auto &t : pool) t.join();
  return exact.load();
}

// Chunk boundaries of a column pipeline: first chunk `first` signals, each
// next one `grow` times larger up to `cap` (the host stages chunk c+1 while
// chunk c computes, so a chunk may only be as much larger as the GPU is
// slower than the staging: configs[4] on the GPU box, 16 threads stage
// ~1.5 us per signal, the solve takes ~2 us); a short tail joins the
// previous chunk.
std::vector<int64_t> cols_bounds(int64_t p) {
  static const int64_t first = getenv("CDB_COLS_FIRST") ? atoll(getenv("CDB_COLS_FIRST")) : 8192;
  static const double grow = getenv("CDB_COLS_GROW") ? atof(getenv("CDB_COLS_GROW")) : 2.0;
  static const int64_t cap = getenv("CDB_COLS_MAX") ? atoll(getenv("CDB_COLS_MAX")) : 131072;
  std::vector<int64_t> b = {0};
  double len = (double)std::max<int64_t>(1, first);
  while (b.back() < p) {
    int64_t l = std::min<int64_t>((int64_t)len, std::max<int64_t>(1, cap));
    if (p - b.back() - l < l / 2) l = p - b.back();  // short tail: merge
    b.push_back(b.back() + l);
    len *= grow > 1.0 ? grow : 1.0;
  }
  return b;
}

// core(off, len, rows_dev, rows_f32, dv, stream): compute one chunk from the
// device rows.  `arrs` are the other per-signal arrays (host memory), as in
// run_pipelined.  *as_f32 in: try fp32 staging (fp64 source); out: the mode
// used.  Returns CDB_ERR_FORMAT internally only for "retry in fp64" (a later
// slab was not fp32-exact); the caller then re-runs with *as_f32 = false.
constexpr cdb_status kRetryF64 = CDB_ERR_FORMAT;

template <typename Core>
cdb_status run_pipelined_cols(int64_t p, int64_t n, const void *cols, bool src_f32, int64_t ld,
                              std::vector<RowArr> &arrs, cudaStream_t st, Core core,
                              bool *as_f32) {
  std::lock_guard<std::mutex> lock(g_slabs_mu);
  void *slab_base = nullptr;
  CDB_CUDA(g_slabs.get(&slab_base));
  bool f32 = src_f32 || *as_f32;
  const std::vector<int64_t> bd = cols_bounds(p);
  const int64_t nch = (int64_t)bd.size() - 1;
  int64_t chunk = 0;
  for (int64_t i = 0; i < nch; i++) chunk = std::max(chunk, bd[i + 1] - bd[i]);
  cudaStream_t cin = copy_stream(0), cout = copy_stream(1);
  const size_t na = arrs.size();
  // slab width: whole slabs of at most kSlabBytes at the fp64 staging size
  const int64_t slab_sig = std::max<int64_t>(1, (int64_t)(kSlabBytes / (8 * (size_t)n)));
  std::vector<DevBuf> bufs(2 * na);
  DevBuf colbuf[2], rows;
  const size_t es_max = 8;
  for (int b = 0; b < 2; b++) {
    CDB_CUDA(colbuf[b].alloc(es_max * n * chunk, st));
    for (size_t a = 0; a < na; a++) CDB_CUDA(bufs[b * na + a].alloc(arrs[a].row_bytes * chunk, st));
  }
  CDB_CUDA(rows.alloc(es_max * n * chunk, st));
  cudaEvent_t ready, slab_ev[kSlabs], in_ready[2], tdone[2], done[2], out_done[2];
  CDB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  for (int r = 0; r < kSlabs; r++) CDB_CUDA(cudaEventCreateWithFlags(&slab_ev[r], cudaEventDisableTiming));
  for (int b = 0; b < 2; b++) {
    CDB_CUDA(cudaEventCreateWithFlags(&in_ready[b], cudaEventDisableTiming));
    CDB_CUDA(cudaEventCreateWithFlags(&tdone[b], cudaEventDisableTiming));
    CDB_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    CDB_CUDA(cudaEventCreateWithFlags(&out_done[b], cudaEventDisableTiming));
  }
  CDB_CUDA(cudaEventRecord(ready, st));  // buffers allocated (stream-ordered)
  CDB_CUDA(cudaStreamWaitEvent(cin, ready, 0));
  CDB_CUDA(cudaStreamWaitEvent(cout, ready, 0));
  static const bool trace = getenv("CDB_PIPE_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto ms_since = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start)
        .count();
  };
  bool slab_used[kSlabs] = {false, false, false};
  int64_t slab_no = 0;
  cdb_status result = CDB_OK;
  cudaError_t ce = cudaSuccess;
  for (int64_t c = 0; c < nch && ce == cudaSuccess && result == CDB_OK; c++) {
    const int b = (int)(c & 1);
    const int64_t off = bd[c], len = bd[c + 1] - bd[c];
    const size_t es = f32 ? 4 : 8;
    if (c >= 2) {
      // colbuf[b] was consumed by chunk c-2's transpose; the input buffers of
      // set b by its compute, whose outputs must have left before reuse
      if ((ce = cudaStreamWaitEvent(cin, tdone[b], 0)) != cudaSuccess) break;
      if ((ce = cudaStreamWaitEvent(cin, out_done[b], 0)) != cudaSuccess) break;
    }
    for (int64_t a0 = 0; a0 < len && ce == cudaSuccess; a0 += slab_sig) {
      const int64_t s = std::min(slab_sig, len - a0);
      const int r = (int)(slab_no++ % kSlabs);
      if (slab_used[r] && (ce = cudaEventSynchronize(slab_ev[r])) != cudaSuccess) break;
      void *slab = (uint8_t *)slab_base + r * kSlabBytes;
      bool exact = stage_cols(cols, src_f32, n, ld, off + a0, s, slab, f32 && !src_f32);
      if (f32 && !src_f32 && !exact) {
        if (c == 0 && a0 == 0) {  // first slab: decide fp64 for the whole call
          f32 = false;
          stage_cols(cols, false, n, ld, off + a0, s, slab, false);
        } else {
          result = kRetryF64;
          break;
        }
      }
      const size_t ess = f32 ? 4 : 8;
      ce = cudaMemcpy2DAsync((uint8_t *)colbuf[b].ptr + a0 * ess, len * ess, slab, s * ess,
                             s * ess, n, cudaMemcpyHostToDevice, cin);
      if (ce == cudaSuccess) ce = cudaEventRecord(slab_ev[r], cin);
      slab_used[r] = true;
    }
    if (ce != cudaSuccess || result != CDB_OK) break;
    for (size_t a = 0; a < na && ce == cudaSuccess; a++) {
      if (arrs[a].out || !arrs[a].host) continue;
      ce = cudaMemcpyAsync(bufs[b * na + a].ptr, (const uint8_t *)arrs[a].host + off * arrs[a].row_bytes,
                           len * arrs[a].row_bytes, cudaMemcpyHostToDevice, cin);
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(in_ready[b], cin);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(st, in_ready[b], 0);
    if (ce == cudaSuccess) ce = cdb::launch_cols_to_rows(colbuf[b].ptr, f32, n, len, rows.ptr, st);
    if (ce == cudaSuccess) ce = cudaEventRecord(tdone[b], st);
    if (ce != cudaSuccess) break;
    (void)es;
    std::vector<void *> dev(na);
    for (size_t a = 0; a < na; a++) dev[a] = bufs[b * na + a].ptr;
    result = core(off, len, rows.ptr, f32, dev, st);
    if (result != CDB_OK) break;
    if ((ce = cudaEventRecord(done[b], st)) != cudaSuccess) break;
    if ((ce = cudaStreamWaitEvent(cout, done[b], 0)) != cudaSuccess) break;
    for (size_t a = 0; a < na && ce == cudaSuccess; a++) {
      if (!arrs[a].out || !arrs[a].host) continue;
      ce = cudaMemcpyAsync((uint8_t *)arrs[a].host + off * arrs[a].row_bytes, dev[a],
                           len * arrs[a].row_bytes, cudaMemcpyDeviceToHost, cout);
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(out_done[b], cout);
    if (trace)
      fprintf(stderr, "[cols] chunk %lld len %lld (%s) staged+issued at %.1f ms\n", (long long)c,
              (long long)len, f32 ? "f32" : "f64", ms_since());
  }
  cudaError_t e1 = cudaStreamSynchronize(cin), e2 = cudaStreamSynchronize(cout);
  cudaError_t e3 = cudaStreamSynchronize(st);
  if (trace) fprintf(stderr, "[cols] all done at %.1f ms\n", ms_since());
  cudaEventDestroy(ready);
  for (int r = 0; r < kSlabs; r++) cudaEventDestroy(slab_ev[r]);
  for (int b = 0; b < 2; b++) {
    cudaEventDestroy(in_ready[b]);
    cudaEventDestroy(tdone[b]);
    cudaEventDestroy(done[b]);
    cudaEventDestroy(out_done[b]);
  }
  *as_f32 = f32;
  if (result != CDB_OK) return result;
  for (cudaError_t e : {ce, e1, e2, e3})
    if (e != cudaSuccess) return fail(CDB_ERR_CUDA, cudaGetErrorString(e));
  return CDB_OK;
}

void dev_outs(Outs &o, void *sel, void *coef, void *count, void *rnorm, void *scans,
              void *flag) {
  o.sel.dev = sel;
  o.coef.dev = coef;
  o.count.dev = count;
  o.rnorm.dev = rnorm;
  o.scans.dev = scans;
  o.flag.dev = flag;
}

constexpr int64_t kPipeMin = 32768;  // pipeline host-buffer calls from this many signals

}  // namespace

namespace {
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
std::atomic<bool> g_prof_on{false};
std::vector<ProfRec> g_prof_open;   // begun, not ended
std::vector<ProfRec> g_prof_done;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

namespace cdb {
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

bool prof_active() { return g_prof_on.load(std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("CDB_PDL");
    return v ? atoi(v) != 0 : true;
  }();
  return on;
}

void prof_begin(const char *name, cudaStream_t stream) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  ProfRec r{name, prof_event(), prof_event()};
  cudaEventRecord(r.a, stream);
  g_prof_open.push_back(r);
}

void prof_end(const char *name, cudaStream_t stream) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  for (size_t i = g_prof_open.size(); i-- > 0;) {
    if (g_prof_open[i].name == name) {
      cudaEventRecord(g_prof_open[i].b, stream);
      g_prof_done.push_back(g_prof_open[i]);
      g_prof_open.erase(g_prof_open.begin() + (long)i);
      return;
    }
  }
}
}  // namespace cdb

extern "C" {

const char *cdb_last_error(void) { return g_last_error.c_str(); }

void cdb_profile_enable(int on) {
  g_prof_on.store(on != 0);
  for (auto &r : g_prof_done) {
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_done.clear();
}

int cdb_profile_read(int max_entries, char *names, int name_len, double *ms, int64_t *launches) {
  // aggregate by name (synchronises on the recorded events)
  std::vector<std::string> keys;
  std::vector<double> tot;
  std::vector<int64_t> cnt;
  for (auto &r : g_prof_done) {
    float t = 0.0f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&t, r.a, r.b);
    size_t k = 0;
    while (k < keys.size() && keys[k] != r.name) k++;
    if (k == keys.size()) {
      keys.push_back(r.name);
      tot.push_back(0.0);
      cnt.push_back(0);
    }
    tot[k] += t;
    cnt[k] += 1;
  }
  const int n = (int)keys.size() < max_entries ? (int)keys.size() : max_entries;
  for (int i = 0; i < n; i++) {
    if (names) {
      std::strncpy(names + (size_t)i * name_len, keys[i].c_str(), (size_t)name_len - 1);
      names[(size_t)i * name_len + name_len - 1] = 0;
    }
    if (ms) ms[i] = tot[i];
    if (launches) launches[i] = cnt[i];
  }
  return (int)keys.size();
}

int64_t cdb_launch_count(void) { return g_launches.load(); }

static cdb_status patch_geometry(int rank, const int64_t *sig, const int64_t *pat,
                                 const int64_t *str, int64_t &n, int64_t &p, int64_t &cells) {
  if (rank < 1 || rank > 4 || !sig || !pat || !str) return fail(CDB_ERR_ARG, "bad patch geometry");
  n = p = cells = 1;
  for (int d = 0; d < rank; d++) {
    if (pat[d] < 1 || str[d] < 1 || sig[d] < 1 || pat[d] > sig[d])
      return fail(CDB_ERR_ARG, "bad patch geometry");
    n *= pat[d];
    p *= (sig[d] - pat[d]) / str[d] + 1;
    cells *= sig[d];
  }
  return CDB_OK;
}

cdb_status cdb_extract_patches(const void *signal, int is_f32, int rank,
                               const int64_t *signal_shape, const int64_t *patch_shape,
                               const int64_t *stride, int remove_dc, double *rows_out,
                               double *dc_out, void *stream) {
  int64_t n, p, cells;
  cdb_status s = patch_geometry(rank, signal_shape, patch_shape, stride, n, p, cells);
  if (s != CDB_OK) return s;
  if (!signal || !rows_out || (remove_dc && !dc_out)) return fail(CDB_ERR_ARG, "null patch buffer");
  DevInfo di;
  if ((s = device_info(di)) != CDB_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  InArr sig;
  OutArr rows, dc;
  CDB_CUDA(sig.bind(signal, (is_f32 ? 4 : 8) * cells, st));
  CDB_CUDA(rows.bind(rows_out, sizeof(double) * p * n, st));
  if (remove_dc) CDB_CUDA(dc.bind(dc_out, sizeof(double) * p, st));
  CDB_CUDA(cdb::launch_extract_patches(sig.dev, is_f32 != 0, rank, signal_shape, patch_shape,
                                       stride, remove_dc, (double *)rows.dev,
                                       remove_dc ? (double *)dc.dev : nullptr, di.sms, st));
  CDB_CUDA(rows.finish(st));
  if (remove_dc) CDB_CUDA(dc.finish(st));
  CDB_CUDA(cudaStreamSynchronize(st));
  return CDB_OK;
}

cdb_status cdb_reconstruct_aggregate(const cdb_dictionary *dict, const int64_t *sel,
                                     const double *coef, int64_t k_width, int64_t p,
                                     const double *dc, int rank, const int64_t *signal_shape,
                                     const int64_t *patch_shape, const int64_t *stride,
                                     double *out, int64_t *uncovered, void *stream) {
  int64_t n, pp, cells;
  cdb_status s = patch_geometry(rank, signal_shape, patch_shape, stride, n, pp, cells);
  if (s != CDB_OK) return s;
  if (!dict || !out || p != pp || n != dict->n || k_width < 0 || (k_width > 0 && (!sel || !coef)))
    return fail(CDB_ERR_ARG, "bad reconstruct arguments");
  DevInfo di;
  if ((s = device_info(di)) != CDB_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  InArr sel_in, coef_in, dc_in;
  OutArr out_o;
  CDB_CUDA(sel_in.bind(sel, sizeof(int64_t) * p * k_width, st));
  CDB_CUDA(coef_in.bind(coef, sizeof(double) * p * k_width, st));
  if (dc) CDB_CUDA(dc_in.bind(dc, sizeof(double) * p, st));
  CDB_CUDA(out_o.bind(out, sizeof(double) * cells, st));
  DevBuf est, unc;
  CDB_CUDA(est.alloc(sizeof(double) * p * n, st));
  CDB_CUDA(unc.alloc(sizeof(unsigned long long), st));
  CDB_CUDA(cudaMemsetAsync(unc.ptr, 0, sizeof(unsigned long long), st));
  CDB_CUDA(cdb::launch_reconstruct_aggregate(
      dict->d64, n, (const int64_t *)sel_in.dev, (const double *)coef_in.dev, k_width, p,
      dc ? (const double *)dc_in.dev : nullptr, rank, signal_shape, patch_shape, stride,
      est.as<double>(), (double *)out_o.dev, (unsigned long long *)unc.ptr, di.sms, st));
  CDB_CUDA(out_o.finish(st));
  unsigned long long h_unc = 0;
  CDB_CUDA(cudaMemcpyAsync(&h_unc, unc.ptr, sizeof(h_unc), cudaMemcpyDeviceToHost, st));
  CDB_CUDA(cudaStreamSynchronize(st));
  if (uncovered) *uncovered = (int64_t)h_unc;
  return CDB_OK;
}

cdb_status cdb_aggregate_patches(const double *rows, const double *dc, int rank,
                                 const int64_t *signal_shape, const int64_t *patch_shape,
                                 const int64_t *stride, double *out, int64_t *uncovered,
                                 void *stream) {
  int64_t n, p, cells;
  cdb_status s = patch_geometry(rank, signal_shape, patch_shape, stride, n, p, cells);
  if (s != CDB_OK) return s;
  if (!rows || !out) return fail(CDB_ERR_ARG, "null patch buffer");
  DevInfo di;
  if ((s = device_info(di)) != CDB_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  InArr rows_in, dc_in;
  OutArr out_o;
  CDB_CUDA(rows_in.bind(rows, sizeof(double) * p * n, st));
  if (dc) CDB_CUDA(dc_in.bind(dc, sizeof(double) * p, st));
  CDB_CUDA(out_o.bind(out, sizeof(double) * cells, st));
  DevBuf unc;
  CDB_CUDA(unc.alloc(sizeof(unsigned long long), st));
  CDB_CUDA(cudaMemsetAsync(unc.ptr, 0, sizeof(unsigned long long), st));
  CDB_CUDA(cdb::launch_aggregate((const double *)rows_in.dev, dc ? (const double *)dc_in.dev : nullptr,
                                 rank, signal_shape, patch_shape, stride, (double *)out_o.dev,
                                 (unsigned long long *)unc.ptr, st));
  CDB_CUDA(out_o.finish(st));
  unsigned long long h_unc = 0;
  CDB_CUDA(cudaMemcpyAsync(&h_unc, unc.ptr, sizeof(h_unc), cudaMemcpyDeviceToHost, st));
  CDB_CUDA(cudaStreamSynchronize(st));
  if (uncovered) *uncovered = (int64_t)h_unc;
  return CDB_OK;
}

// ---------------------------------------------------------------- .csd files
static uint32_t crc32_zlib(const uint8_t *data, size_t len) {
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; i++) {
      uint32_t c = i;
      for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < len; i++) c = table[(c ^ data[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

static std::string py_tuple(const int64_t *v, int r) {  // Python's tuple repr
  std::string s = "(";
  for (int i = 0; i < r; i++) {
    if (i) s += ", ";
    s += std::to_string(v[i]);
  }
  return s + (r == 1 ? ",)" : ")");
}

namespace {
// Parse one in-memory .csd image.  atoms_t[s] (when given) receives scale s's
// T x N rows; capacity[s] (doubles, when given) must cover them.
cdb_status csd_parse(const uint8_t *raw_data, size_t raw_size, const std::string &P,
                     int32_t *scale_count, cdb_csd_scale *scales, double *const *atoms_t,
                     const int64_t *capacity) {
  struct {
    const uint8_t *p;
    size_t n;
    const uint8_t *data() const { return p; }
    size_t size() const { return n; }
  } raw{raw_data, raw_size};
  if (raw.size() < 16) return fail(CDB_ERR_FORMAT, P + ": too short for a model file");
  uint32_t stored;
  memcpy(&stored, raw.data() + raw.size() - 4, 4);
  const size_t body = raw.size() - 4;
  if (crc32_zlib(raw.data(), body) != stored)
    return fail(CDB_ERR_CHECKSUM, P + ": CRC-32 mismatch, refusing to load");
  if (memcmp(raw.data(), "CSDM", 4) != 0)
    return fail(CDB_ERR_FORMAT, P + ": not a .csd file (bad magic)");
  size_t pos = 4;
  auto take = [&](uint32_t &v) -> bool {
    if (pos + 4 > body) return false;
    memcpy(&v, raw.data() + pos, 4);
    pos += 4;
    return true;
  };
  uint32_t version, count;
  if (!take(version)) return fail(CDB_ERR_FORMAT, P + ": truncated file");
  if (version != 1)
    return fail(CDB_ERR_FORMAT, P + ": unsupported version " + std::to_string(version));
  if (!take(count)) return fail(CDB_ERR_FORMAT, P + ": truncated file");
  if (count != 1 && count != 2)
    return fail(CDB_ERR_FORMAT, P + ": scale count " + std::to_string(count) + " not in (1, 2)");
  for (uint32_t sidx = 0; sidx < count; sidx++) {
    cdb_csd_scale &sc = scales[sidx];
    uint32_t rank;
    if (!take(rank)) return fail(CDB_ERR_FORMAT, P + ": truncated file");
    if (rank < 1 || rank > 4)
      return fail(CDB_ERR_FORMAT, P + ": patch rank " + std::to_string(rank) + " outside 1..4");
    sc.rank = (int32_t)rank;
    int64_t prod = 1;
    for (uint32_t d = 0; d < 4; d++) sc.extents[d] = 0;
    if (pos + 4 * rank > body) return fail(CDB_ERR_FORMAT, P + ": truncated file");
    for (uint32_t d = 0; d < rank; d++) {
      uint32_t e;
      take(e);
      sc.extents[d] = e;
      if (__builtin_mul_overflow(prod, (int64_t)e, &prod))
        return fail(CDB_ERR_FORMAT, P + ": patch shape overflows");
    }
    uint32_t nn, tt, kk, qq;
    if (pos + 16 > body) return fail(CDB_ERR_FORMAT, P + ": truncated file");
    take(nn);
    take(tt);
    take(kk);
    take(qq);
    if ((int64_t)nn != prod)
      return fail(CDB_ERR_FORMAT, P + ": N=" + std::to_string(nn) +
                                      " inconsistent with patch shape " +
                                      py_tuple(sc.extents, (int)rank));
    sc.n = nn;
    sc.t = tt;
    sc.k = kk;
    sc.q = qq;
    uint64_t elems, bytes;
    if (__builtin_mul_overflow((uint64_t)nn, (uint64_t)tt, &elems) ||
        __builtin_mul_overflow(elems, (uint64_t)8, &bytes) || bytes > body - pos)
      return fail(CDB_ERR_FORMAT, P + ": truncated atom data");
    if (atoms_t && atoms_t[sidx]) {
      if (capacity && (capacity[sidx] < 0 || (uint64_t)capacity[sidx] < elems))
        return fail(CDB_ERR_ARG, P + ": atom buffer too small for scale " + std::to_string(sidx));
      memcpy(atoms_t[sidx], raw.data() + pos, bytes);
    }
    pos += bytes;
  }
  *scale_count = (int32_t)count;
  if (count == 2) {
    const cdb_csd_scale &lo = scales[0], &hi = scales[1];
    if (hi.q != 0)
      return fail(CDB_ERR_FORMAT,
                  P + ": finest scale must have Q=0, got " + std::to_string(hi.q));
    if (hi.t != lo.q * lo.t)
      return fail(CDB_ERR_FORMAT, P + ": T_high=" + std::to_string(hi.t) +
                                      " != Q*T_low=" + std::to_string(lo.q * lo.t));
    bool bad = lo.rank != hi.rank;
    for (int d = 0; d < hi.rank && !bad; d++) bad = hi.extents[d] % lo.extents[d] != 0;
    if (bad)
      return fail(CDB_ERR_FORMAT, P + ": fine shape " + py_tuple(hi.extents, hi.rank) +
                                      " not divisible by coarse " +
                                      py_tuple(lo.extents, lo.rank));
  }
  return CDB_OK;
}
}  // namespace

cdb_status cdb_csd_read(const char *path, int32_t *scale_count, cdb_csd_scale *scales,
                        double *const *atoms_t) {
  if (!path || !scale_count || !scales) return fail(CDB_ERR_ARG, "bad csd arguments");
  const std::string P(path);
  FILE *f = fopen(path, "rb");
  if (!f) return fail(CDB_ERR_ARG, P + ": cannot open");
  std::vector<uint8_t> raw;
  uint8_t chunk[1 << 16];
  size_t got;
  while ((got = fread(chunk, 1, sizeof(chunk), f)) > 0) raw.insert(raw.end(), chunk, chunk + got);
  fclose(f);
  return csd_parse(raw.data(), raw.size(), P, scale_count, scales, atoms_t, nullptr);
}

cdb_status cdb_csd_parse(const uint8_t *data, int64_t size, const char *name,
                         int32_t *scale_count, cdb_csd_scale *scales, double *const *atoms_t,
                         const int64_t *capacity) {
  if (!data || size < 0 || !scale_count || !scales) return fail(CDB_ERR_ARG, "bad csd arguments");
  return csd_parse(data, (size_t)size, name ? std::string(name) : std::string("<memory>"),
                   scale_count, scales, atoms_t, capacity);
}

cdb_status cdb_rows_from_cols(const void *cols, int64_t n, int64_t p, int elem_size, void *rows,
                              int threads) {
  if (!cols || !rows || n < 0 || p < 0 || (elem_size != 4 && elem_size != 8))
    return fail(CDB_ERR_ARG, "bad rows_from_cols arguments");
  if (n == 0 || p == 0) return CDB_OK;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t B = 64;  // 64 x 64 tiles: both sides touch whole cache lines
  const int64_t tiles_p = (p + B - 1) / B;
  if (threads > tiles_p) threads = (int)tiles_p;
  auto work = [&](int tid) {
    for (int64_t tp = tid; tp < tiles_p; tp += threads) {
      const int64_t j0 = tp * B, j1 = std::min(p, j0 + B);
      for (int64_t i0 = 0; i0 < n; i0 += B) {
        const int64_t i1 = std::min(n, i0 + B);
        if (elem_size == 4) {
          const float *src = (const float *)cols;
          float *dst = (float *)rows;
          for (int64_t j = j0; j < j1; j++)
            for (int64_t i = i0; i < i1; i++) dst[j * n + i] = src[i * p + j];
        } else {
          const double *src = (const double *)cols;
          double *dst = (double *)rows;
          for (int64_t j = j0; j < j1; j++)
            for (int64_t i = i0; i < i1; i++) dst[j * n + i] = src[i * p + j];
        }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; t++) pool.emplace_back(work, t);
  work(0);
  for (auto &t : pool) t.join();
  return CDB_OK;
}

int cdb_host_equal(const void *a, const void *b, int64_t nbytes, int threads) {
  if (nbytes <= 0 || a == b) return 1;
  if (!a || !b) return 0;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t piece = int64_t(1) << 20;  // threads stop at the first differing 1 MiB piece
  const int64_t pieces = (nbytes + piece - 1) / piece;
  if (threads > pieces) threads = (int)pieces;
  std::atomic<int> differ{0};
  auto work = [&](int tid) {
    for (int64_t i = tid; i < pieces && !differ.load(std::memory_order_relaxed); i += threads) {
      const int64_t o = i * piece, len = std::min(piece, nbytes - o);
      if (memcmp((const uint8_t *)a + o, (const uint8_t *)b + o, (size_t)len) != 0)
        differ.store(1, std::memory_order_relaxed);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; t++) pool.emplace_back(work, t);
  work(0);
  for (auto &t : pool) t.join();
  return differ.load() ? 0 : 1;
}

void cdb_last_run_info(int *engine, int *delegated, int *rescans) {
  if (engine) *engine = g_last_engine;
  int h[2] = {0, 0};
  int *diag = g_diag ? diag_dev() : nullptr;
  if (diag && cudaDeviceSynchronize() == cudaSuccess)
    cudaMemcpy(h, diag, sizeof(h), cudaMemcpyDeviceToHost);
  if (delegated) *delegated = h[0];
  if (rescans) *rescans = h[1];
}

cdb_status cdb_device_info(int *sm_count, int *cc_major, int *cc_minor) {
  DevInfo di;
  int dev = 0;
  CDB_CUDA(cudaGetDevice(&dev));
  CDB_CUDA(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
  CDB_CUDA(cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, dev));
  CDB_CUDA(cudaDeviceGetAttribute(&di.minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (sm_count) *sm_count = di.sms;
  if (cc_major) *cc_major = di.major;
  if (cc_minor) *cc_minor = di.minor;
  return CDB_OK;
}

cdb_status cdb_dictionary_create(const double *atoms_t, int64_t t, int64_t n,
                                 int64_t gram_budget_bytes, void *stream, cdb_dictionary **out) {
  if (!atoms_t || t < 1 || n < 1 || !out) return fail(CDB_ERR_ARG, "bad dictionary arguments");
  DevInfo di;
  cdb_status s0 = device_info(di);
  if (s0 != CDB_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  auto *d = new cdb_dictionary();
  cudaGetDevice(&d->device);
  d->t = t;
  d->n = n;
  d->n_pad = (n + 63) / 64 * 64;
  auto cleanup = [&](cdb_status s, const std::string &m) {
    cdb_dictionary_destroy(d);
    return fail(s, m);
  };
  const size_t b64 = sizeof(double) * t * n;
  if (cudaMalloc(&d->d64, b64) != cudaSuccess) return cleanup(CDB_ERR_NOMEM, "d64 alloc");
  if (cudaMemcpyAsync(d->d64, atoms_t, b64, cudaMemcpyDefault, st) != cudaSuccess)
    return cleanup(CDB_ERR_CUDA, "d64 copy");
  d->bytes += b64;
  const size_t b16 = 2 * t * d->n_pad;
  if (cudaMalloc(&d->d16, b16) != cudaSuccess) return cleanup(CDB_ERR_NOMEM, "d16 alloc");
  d->bytes += b16;
  if (cudaMalloc(&d->d32, 4 * t * n) != cudaSuccess) return cleanup(CDB_ERR_NOMEM, "d32 alloc");
  d->bytes += 4 * t * n;
  if (cdb::launch_to_f32(d->d64, t * n, d->d32, st) != cudaSuccess)
    return cleanup(CDB_ERR_CUDA, "f32 conversion");
  {
    double *dm = nullptr;
    if (cudaMallocAsync((void **)&dm, sizeof(double), st) != cudaSuccess)
      return cleanup(CDB_ERR_NOMEM, "dmax alloc");
    if (cdb::launch_row_norm_max(d->d64, t, n, dm, st) != cudaSuccess ||
        cudaMemcpyAsync(&d->dmax, dm, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return cleanup(CDB_ERR_CUDA, "dmax kernel");
    if (cudaStreamSynchronize(st) != cudaSuccess) return cleanup(CDB_ERR_CUDA, "dmax sync");
    // the fp16 operand carries dscale * d: largest atom norm in [2^8, 2^9)
    d->dscale = 1.0;
    if (d->dmax > 0x1p-900 && d->dmax < 0x1p900) d->dscale = std::ldexp(1.0, 8 - std::ilogb(d->dmax));
    if (cdb::launch_to_f16(d->d64, t, n, d->n_pad, d->dscale, d->d16, st) != cudaSuccess)
      return cleanup(CDB_ERR_CUDA, "fp16 conversion");
    if (cdb::launch_quant_err_max(d->d64, d->d16, t, n, d->n_pad, d->dscale, dm, st) !=
            cudaSuccess ||
        cudaMemcpyAsync(&d->emax, dm, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return cleanup(CDB_ERR_CUDA, "quantisation-error kernel");
    cudaFreeAsync(dm, st);
  }
  const double gb = 8.0 * (double)t * (double)t;
  if (gb <= (double)gram_budget_bytes) {
    if (cudaMalloc(&d->gram, (size_t)gb) != cudaSuccess) return cleanup(CDB_ERR_NOMEM, "gram alloc");
    d->bytes += (int64_t)gb;
    if (cdb::launch_gram_matrix(d->d64, t, n, d->gram, st) != cudaSuccess)
      return cleanup(CDB_ERR_CUDA, "gram kernel");
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return cleanup(CDB_ERR_CUDA, "dictionary sync");
  *out = d;
  return CDB_OK;
}

cdb_status cdb_dictionary_destroy(cdb_dictionary *d) {
  if (!d) return CDB_OK;
  if (d->d64) cudaFree(d->d64);
  if (d->gram) cudaFree(d->gram);
  if (d->d16) cudaFree(d->d16);
  if (d->d32) cudaFree(d->d32);
  delete d;
  return CDB_OK;
}

int64_t cdb_dictionary_bytes(const cdb_dictionary *d) { return d ? d->bytes : 0; }

cdb_status cdb_debug_corr_topk(const cdb_dictionary *d, const float *rows, int64_t p,
                               int *cand_idx, float *cand_val, float *cand_drop, int grid_cap,
                               void *stream) {
  if (!d || !rows || p < 1) return fail(CDB_ERR_ARG, "bad debug_corr_topk arguments");
  cudaStream_t st = (cudaStream_t)stream;
  CDB_CUDA(cdb::debug_corr_topk(d->d16, d->dscale, d->t, d->n, rows, p, cand_idx, cand_val,
                                cand_drop, grid_cap, st));
  CDB_CUDA(cudaStreamSynchronize(st));
  return CDB_OK;
}

// nb != NULL (mode 2): per-signal block counts, budget min(k_max, nb*q, N)
// per signal (the reference's per-group k_max rule, pursuit.py:423).
static cdb_status omp_common(const cdb_dictionary *dict, const void *ys, int ys_is_f32, int64_t p,
                             int64_t k_max, const double *eps, const int64_t *ids, int64_t stride,
                             int mode, int64_t q, int64_t *out_sel, double *out_coef,
                             int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                             uint8_t *out_flag, int engine, void *stream,
                             const int64_t *nb = nullptr) {
  if (!dict || p < 0 || k_max < 0 || (p > 0 && (!ys || !eps)))
    return fail(CDB_ERR_ARG, "bad omp arguments");
  if (p == 0) return CDB_OK;
  DevInfo di;
  cdb_status s0 = device_info(di);
  if (s0 != CDB_OK) return s0;
  if ((s0 = check_device(dict)) != CDB_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  const bool f32 = ys_is_f32 != 0;
  const int64_t n = dict->n;
  const int64_t max_c0 = mode == 0 ? dict->t : (mode == 1 ? stride : stride * q);
  const bool host_io = !is_device_ptr(ys) || !is_device_ptr(out_sel) || !is_device_ptr(out_coef);
  if (host_io && p >= kPipeMin && !is_device_ptr(ys) && !is_device_ptr(eps)) {
    std::vector<RowArr> arrs = {
        {(void *)ys, (size_t)(f32 ? 4 : 8) * n, false}, {(void *)eps, sizeof(double), false},
        {(void *)ids, sizeof(int64_t) * (mode ? stride : 0) + (mode ? 0 : 8), false},
        {out_sel, sizeof(int64_t) * k_max, true}, {out_coef, sizeof(double) * k_max, true},
        {out_count, sizeof(int64_t), true}, {out_rnorm, sizeof(double), true},
        {out_scans, sizeof(int64_t), true}, {out_flag, sizeof(uint8_t), true},
        {(void *)nb, sizeof(int64_t), false}};
    if (!mode) arrs[2].host = nullptr;
    if (all_host(arrs))
    return run_pipelined(p, arrs, st, [&](int64_t, int64_t len, std::vector<void *> &dv,
                                          cudaStream_t s2) -> cdb_status {
      cdb::Cands c{};
      c.mode = mode;
      c.t = dict->t;
      c.ids = (const int64_t *)dv[2];
      c.stride = stride;
      c.q = q;
      c.nb_fixed = stride;
      c.nb = nb ? (const int64_t *)dv[9] : nullptr;
      c.clip = nb ? 1 : 0;
      Outs o;
      dev_outs(o, dv[3], dv[4], dv[5], dv[6], dv[7], dv[8]);
      return run_omp(dict, dv[0], f32, len, k_max, k_max, (const double *)dv[1], c, max_c0, o,
                     engine, di, s2);
    }, 1);
  }
  InArr y_in, e_in, id_in, nb_in;
  CDB_CUDA(y_in.bind(ys, (f32 ? 4 : 8) * p * n, st));
  CDB_CUDA(e_in.bind(eps, sizeof(double) * p, st));
  if (mode != 0) CDB_CUDA(id_in.bind(ids, sizeof(int64_t) * p * stride, st));
  if (nb) CDB_CUDA(nb_in.bind(nb, sizeof(int64_t) * p, st));
  Outs o;
  CDB_CUDA(o.bind(p, k_max, out_sel, out_coef, out_count, out_rnorm, out_scans, out_flag, st));
  cdb::Cands c{};
  c.mode = mode;
  c.t = dict->t;
  c.ids = (const int64_t *)id_in.dev;
  c.stride = stride;
  c.q = q;
  c.nb = nb ? (const int64_t *)nb_in.dev : nullptr;
  c.nb_fixed = stride;
  c.clip = nb ? 1 : 0;
  const int64_t max_c = mode == 0 ? dict->t : (mode == 1 ? stride : stride * q);
  cdb_status s = run_omp(dict, y_in.dev, f32, p, k_max, k_max, (const double *)e_in.dev, c, max_c,
                         o, engine, di, st);
  if (s != CDB_OK) return s;
  CDB_CUDA(o.finish(st));
  CDB_CUDA(cudaStreamSynchronize(st));
  return CDB_OK;
}

cdb_status cdb_omp_batch(const cdb_dictionary *dict, const void *ys, int ys_is_f32, int64_t p,
                         int64_t k_max, const double *eps, const int64_t *allowed,
                         int64_t s_allowed, int restricted, int64_t *out_sel, double *out_coef,
                         int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                         uint8_t *out_flag, int engine, void *stream) {
  if (restricted && (!allowed || s_allowed < 1) && p > 0)
    return fail(CDB_ERR_ARG, "restricted call without allowed ids");
  return omp_common(dict, ys, ys_is_f32, p, k_max, eps, allowed, s_allowed, restricted ? 1 : 0, 1,
                    out_sel, out_coef, out_count, out_rnorm, out_scans, out_flag, engine, stream);
}

cdb_status cdb_omp_batch_cols(const cdb_dictionary *dict, const void *ys_cols, int ys_is_f32,
                              int64_t ld, int64_t p, int64_t k_max, const double *eps,
                              double rel_tol, int64_t *out_sel, double *out_coef,
                              int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                              uint8_t *out_flag, int engine, void *stream) {
  if (!dict || p < 0 || k_max < 0 || ld < p) return fail(CDB_ERR_ARG, "bad omp arguments");
  if (p == 0) return CDB_OK;
  if (!ys_cols || is_device_ptr(ys_cols)) return fail(CDB_ERR_ARG, "ys_cols must be host memory");
  if (eps && is_device_ptr(eps)) return fail(CDB_ERR_ARG, "eps must be host memory");
  DevInfo di;
  cdb_status s0 = device_info(di);
  if (s0 != CDB_OK) return s0;
  if ((s0 = check_device(dict)) != CDB_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = dict->n;
  std::vector<RowArr> arrs = {
      {out_sel, sizeof(int64_t) * k_max, true}, {out_coef, sizeof(double) * k_max, true},
      {out_count, sizeof(int64_t), true}, {out_rnorm, sizeof(double), true},
      {out_scans, sizeof(int64_t), true}, {out_flag, sizeof(uint8_t), true},
      {(void *)eps, sizeof(double), false}};
  for (size_t a = 0; a < 6; a++)
    if (!arrs[a].host) return fail(CDB_ERR_ARG, "null output");
  if (!all_host(arrs)) return fail(CDB_ERR_ARG, "outputs must be host memory");
  auto run = [&](bool try_f32) -> cdb_status {
    bool f32 = try_f32;
    return run_pipelined_cols(
        p, n, ys_cols, ys_is_f32 != 0, ld, arrs, st,
        [&](int64_t, int64_t len, const void *rows, bool rows_f32, std::vector<void *> &dv,
            cudaStream_t s2) -> cdb_status {
          DevBuf etmp;
          const double *e_dev = (const double *)dv[6];
          if (!eps) {  // rel_tol * |y| per signal, on the device
            CDB_CUDA(etmp.alloc(sizeof(double) * len, s2));
            CDB_CUDA(cdb::launch_row_tol(rows, rows_f32, len, n, rel_tol, etmp.as<double>(), s2));
            e_dev = etmp.as<double>();
          }
          cdb::Cands c{};
          c.mode = 0;
          c.t = dict->t;
          Outs o;
          dev_outs(o, dv[0], dv[1], dv[2], dv[3], dv[4], dv[5]);
          return run_omp(dict, rows, rows_f32, len, k_max, k_max, e_dev, c, dict->t, o, engine, di,
                         s2);
        },
        &f32);
  };
  cdb_status s = run(ys_is_f32 == 0);
  if (s == kRetryF64) s = run(false);
  return s;
}

cdb_status cdb_omp_batch_coded(const cdb_dictionary *dict, const double *ys, int64_t m_stride,
                               const int32_t *rows, int64_t fan, int sum_order,
                               const int64_t *m, int64_t p,
                               int64_t k_max, const double *eps, const int64_t *blocks,
                               int64_t nb_max, const int64_t *nb, int64_t q, int64_t *out_sel,
                               double *out_coef, int64_t *out_count, double *out_rnorm,
                               int64_t *out_scans, uint8_t *out_flag, void *stream) {
  if (!dict || p < 0 || k_max < 0 || fan < 1 || fan > 1024 || sum_order < 0 ||
      sum_order > 1 || (sum_order == 1 && fan > 128) ||
      (p > 0 && (!ys || !rows || !m || !eps || m_stride < 1 || m_stride > dict->n)))
    return fail(CDB_ERR_ARG, "bad coded omp arguments");
  if (blocks && (nb_max < 1 || q < 1 || nb_max * q > dict->t))
    return fail(CDB_ERR_ARG, "bad block arguments");
  if (p == 0) return CDB_OK;
  DevInfo di;
  cdb_status s0 = device_info(di);
  if (s0 != CDB_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  InArr y_in, r_in, m_in, e_in, b_in, nb_in;
  CDB_CUDA(y_in.bind(ys, sizeof(double) * p * m_stride, st));
  CDB_CUDA(r_in.bind(rows, sizeof(int32_t) * p * m_stride * fan, st));
  CDB_CUDA(m_in.bind(m, sizeof(int64_t) * p, st));
  CDB_CUDA(e_in.bind(eps, sizeof(double) * p, st));
  Outs o;
  CDB_CUDA(o.bind(p, k_max, out_sel, out_coef, out_count, out_rnorm, out_scans, out_flag, st));
  cdb::Cands c{};
  c.t = dict->t;
  c.clip = 1;  // budget min(k_max, candidates, m_p) per signal
  int64_t max_cands = dict->t;
  if (blocks) {
    CDB_CUDA(b_in.bind(blocks, sizeof(int64_t) * p * nb_max, st));
    if (nb) CDB_CUDA(nb_in.bind(nb, sizeof(int64_t) * p, st));
    c.mode = 2;
    c.ids = (const int64_t *)b_in.dev;
    c.stride = nb_max;
    c.q = q;
    c.nb = nb ? (const int64_t *)nb_in.dev : nullptr;
    c.nb_fixed = nb_max;
    max_cands = nb_max * q;
  } else {
    c.mode = 0;
  }
  g_last_engine = CDB_ENGINE_EXACT;
  diag_clear(st);
  cdb_status s = run_exact(dict, y_in.dev, false, p, nullptr, k_max, k_max,
                           (const double *)e_in.dev, c, max_cands, o, di, st, nullptr,
                           (const int32_t *)r_in.dev, (const int64_t *)m_in.dev, (int)fan,
                           m_stride, sum_order);
  if (s != CDB_OK) return s;
  CDB_CUDA(o.finish(st));
  CDB_CUDA(cudaStreamSynchronize(st));
  return CDB_OK;
}

cdb_status cdb_omp_batch_masked(const cdb_dictionary *dict, const double *ys,
                                const int32_t *rows, const int64_t *m, int64_t p, int64_t k_max,
                                const double *eps, int64_t *out_sel, double *out_coef,
                                int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                                uint8_t *out_flag, void *stream) {
  if (!dict) return fail(CDB_ERR_ARG, "bad masked omp arguments");
  return cdb_omp_batch_coded(dict, ys, dict->n, rows, 1, 0, m, p, k_max, eps, nullptr, 0, nullptr,
                             0, out_sel, out_coef, out_count, out_rnorm, out_scans, out_flag,
                             stream);
}

cdb_status cdb_omp_batch_blocked_ragged(const cdb_dictionary *dict, const void *ys, int ys_is_f32,
                                        int64_t p, int64_t k_max, const double *eps,
                                        const int64_t *blocks, int64_t nb_max, const int64_t *nb,
                                        int64_t q, int64_t *out_sel, double *out_coef,
                                        int64_t *out_count, double *out_rnorm, int64_t *out_scans,
                                        uint8_t *out_flag, int engine, void *stream) {
  if (p > 0 && (!blocks || !nb || nb_max < 1 || q < 1)) return fail(CDB_ERR_ARG, "bad block arguments");
  return omp_common(dict, ys, ys_is_f32, p, k_max, eps, blocks, nb_max, 2, q, out_sel, out_coef,
                    out_count, out_rnorm, out_scans, out_flag, engine, stream, nb);
}

cdb_status cdb_omp_batch_blocked(const cdb_dictionary *dict, const void *ys, int ys_is_f32,
                                 int64_t p, int64_t k_max, const double *eps,
                                 const int64_t *blocks, int64_t nb, int64_t q, int64_t *out_sel,
                                 double *out_coef, int64_t *out_count, double *out_rnorm,
                                 int64_t *out_scans, uint8_t *out_flag, int engine, void *stream) {
  if (p > 0 && (!blocks || nb < 1 || q < 1)) return fail(CDB_ERR_ARG, "bad block arguments");
  return omp_common(dict, ys, ys_is_f32, p, k_max, eps, blocks, nb, 2, q, out_sel, out_coef,
                    out_count, out_rnorm, out_scans, out_flag, engine, stream);
}

// Per-step device times of zero-tree calls: events recorded per (chunk) call,
// read once after the caller's final synchronisation -- no mid-call waits.
struct StepTimer {
  std::vector<std::array<cudaEvent_t, 3>> ev;
  cudaError_t open(cudaStream_t st) {
    std::array<cudaEvent_t, 3> e{};
    for (auto &x : e) {
      cudaError_t r = cudaEventCreate(&x);
      if (r != cudaSuccess) return r;
    }
    ev.push_back(e);
    return cudaEventRecord(e[0], st);
  }
  cudaError_t mark(int i, cudaStream_t st) { return cudaEventRecord(ev.back()[i], st); }
  void finish(float *step_ms) {  // after the stream was synchronised
    for (auto &e : ev) {
      float a = 0.0f, b = 0.0f;
      if (step_ms && cudaEventElapsedTime(&a, e[0], e[1]) == cudaSuccess &&
          cudaEventElapsedTime(&b, e[1], e[2]) == cudaSuccess) {
        step_ms[0] += a;
        step_ms[1] += b;
      }
      for (auto &x : e) cudaEventDestroy(x);
    }
    ev.clear();
  }
  ~StepTimer() { finish(nullptr); }
};

static cdb_status zero_tree_core(const cdb_dictionary *low, const cdb_dictionary *high,
                                 const int64_t *fine_shape, const int64_t *factors, int rank,
                                 const void *ydev, bool f32, int64_t p, int64_t k1,
                                 int64_t k_high, double rel_tol, int phi_mode, Outs &lo, Outs &hi,
                                 int engine, StepTimer *tm, const DevInfo &di, cudaStream_t st) {
  const int64_t n = high->n, q = high->t / low->t;
  if (tm) CDB_CUDA(tm->open(st));

  // ---- step 1: W y (identity) or y (Phi), tolerance relative to it
  DevBuf ylow, eps1, eps2, blocks;
  const void *y1 = ydev;
  bool y1_f32 = f32;
  if (!phi_mode) {
    int64_t n_low = 1;
    for (int d = 0; d < rank; d++) n_low *= fine_shape[d] / factors[d];
    if (n_low != low->n) return fail(CDB_ERR_ARG, "coarse size != low dictionary dim");
    CDB_CUDA(ylow.alloc(sizeof(double) * p * n_low, st));
    CDB_CUDA(eps1.alloc(sizeof(double) * p, st));
    CDB_CUDA(eps2.alloc(sizeof(double) * p, st));
    // downsample + both stopping tolerances in one pass over y
    CDB_CUDA(cdb::launch_downsample(ydev, f32, p, n, fine_shape, factors, rank,
                                    ylow.as<double>(), n_low, st, rel_tol, eps1.as<double>(),
                                    eps2.as<double>()));
    y1 = ylow.ptr;
    y1_f32 = false;
  } else {
    CDB_CUDA(eps1.alloc(sizeof(double) * p, st));
    CDB_CUDA(cdb::launch_row_tol(y1, y1_f32, p, low->n, rel_tol, eps1.as<double>(), st));
  }
  cdb::Cands c1{};
  c1.mode = 0;
  c1.t = low->t;
  cdb_status s = run_omp(low, y1, y1_f32, p, k1, k1, eps1.as<double>(), c1, low->t, lo, engine, di,
                         st, "gram_step1");
  if (s != CDB_OK) return s;
  if (tm) CDB_CUDA(tm->mark(1, st));

  // ---- step 2: restricted to the children of the sorted coarse support
  CDB_CUDA(blocks.alloc(sizeof(int64_t) * p * k1, st));
  CDB_CUDA(cdb::launch_sort_blocks((const int64_t *)lo.sel.dev, (const int64_t *)lo.count.dev, p,
                                   k1, blocks.as<int64_t>(), st));
  if (phi_mode) {  // Phi: step-1 input is y itself, eps2 == eps1 in value
    CDB_CUDA(eps2.alloc(sizeof(double) * p, st));
    CDB_CUDA(cdb::launch_row_tol(ydev, f32, p, n, rel_tol, eps2.as<double>(), st));
  }
  cdb::Cands c2{};
  c2.mode = 2;
  c2.t = high->t;
  c2.ids = blocks.as<int64_t>();
  c2.stride = k1;
  c2.q = q;
  c2.nb = (const int64_t *)lo.count.dev;
  c2.clip = 1;
  // the Gram engine gets its alpha0 = <d_C, y> from the parent-routed kernel
  DevBuf alpha0, rwork;
  const bool high_resident =
      cdb::resident_fits(high->n, high->t, k_high, k1 * q, di.smem_optin) &&
      (engine == CDB_ENGINE_RESIDENT ||
       (engine == CDB_ENGINE_AUTO && !gram_preferred(high, k1 * q, k_high)));
  const bool use_route = high->gram && !high_resident && engine != CDB_ENGINE_EXACT &&
                         high->t / q == low->t &&
                         (8 * q * n <= 192 * 1024 || cdb::route_alpha0_dmma(q, n)) && k1 < 65536 &&
                         (q == 1 || q == 2 || q == 4 || q == 8 || q == 16);
  if (use_route) {
    CDB_CUDA(alpha0.alloc(sizeof(double) * p * k1 * q, st));
    CDB_CUDA(rwork.alloc((size_t)cdb::route_work_bytes(low->t, p, k1, n, f32), st));
    CDB_CUDA(cdb::launch_route_alpha0(high->d64, low->t, n, q, ydev, f32, blocks.as<int64_t>(),
                                      (const int64_t *)lo.count.dev, p, k1, k1 * q,
                                      alpha0.as<double>(), rwork.ptr, st));
  }
  s = run_omp(high, ydev, f32, p, k_high, k_high, eps2.as<double>(), c2, k1 * q, hi, engine, di,
              st, "gram_step2", use_route ? alpha0.as<double>() : nullptr);
  if (s != CDB_OK) return s;
  if (tm) CDB_CUDA(tm->mark(2, st));
  return CDB_OK;
}

cdb_status cdb_zero_tree_batch(const cdb_dictionary *low, const cdb_dictionary *high,
                               const int64_t *fine_shape, const int64_t *factors, int rank,
                               const void *ys, int ys_is_f32, int64_t p, int64_t k1,
                               int64_t k_high, double rel_tol, int phi_mode, int64_t *low_sel,
                               double *low_coef, int64_t *low_count, double *low_rnorm,
                               int64_t *low_scans, uint8_t *low_flag, int64_t *high_sel,
                               double *high_coef, int64_t *high_count, double *high_rnorm,
                               int64_t *high_scans, uint8_t *high_flag, int engine,
                               float *step_ms, void *stream) {
  if (!low || !high || p < 0 || k1 < 1 || k_high < 1 || high->t % low->t)
    return fail(CDB_ERR_ARG, "bad zero-tree arguments");
  if (!phi_mode && (!fine_shape || !factors || rank < 1 || rank > 4))
    return fail(CDB_ERR_ARG, "bad scale spec");
  if (phi_mode && low->n != high->n) return fail(CDB_ERR_ARG, "Phi mode needs equal M");
  if (p == 0) return CDB_OK;
  DevInfo di;
  cdb_status s0 = device_info(di);
  if (s0 != CDB_OK) return s0;
  if ((s0 = check_device(low)) != CDB_OK || (s0 = check_device(high)) != CDB_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  const bool f32 = ys_is_f32 != 0;
  const int64_t n = high->n;
  if (step_ms) step_ms[0] = step_ms[1] = 0.0f;
  const bool host_io = !is_device_ptr(ys) || !is_device_ptr(high_sel) || !is_device_ptr(low_sel);
  if (host_io && p >= kPipeMin && !is_device_ptr(ys)) {
    std::vector<RowArr> arrs = {
        {(void *)ys, (size_t)(f32 ? 4 : 8) * n, false},
        {low_sel, sizeof(int64_t) * k1, true}, {low_coef, sizeof(double) * k1, true},
        {low_count, sizeof(int64_t), true}, {low_rnorm, sizeof(double), true},
        {low_scans, sizeof(int64_t), true}, {low_flag, sizeof(uint8_t), true},
        {high_sel, sizeof(int64_t) * k_high, true}, {high_coef, sizeof(double) * k_high, true},
        {high_count, sizeof(int64_t), true}, {high_rnorm, sizeof(double), true},
        {high_scans, sizeof(int64_t), true}, {high_flag, sizeof(uint8_t), true}};
    if (all_host(arrs)) {
      StepTimer tm;
      cdb_status s = run_pipelined(p, arrs, st, [&](int64_t, int64_t len, std::vector<void *> &dv,
                                                    cudaStream_t s2) -> cdb_status {
        Outs lo, hi;
        dev_outs(lo, dv[1], dv[2], dv[3], dv[4], dv[5], dv[6]);
        dev_outs(hi, dv[7], dv[8], dv[9], dv[10], dv[11], dv[12]);
        return zero_tree_core(low, high, fine_shape, factors, rank, dv[0], f32, len, k1, k_high,
                              rel_tol, phi_mode, lo, hi, engine, step_ms ? &tm : nullptr, di, s2);
      });
      tm.finish(step_ms);
      return s;
    }
  }
  InArr y_in;
  CDB_CUDA(y_in.bind(ys, (f32 ? 4 : 8) * p * n, st));
  Outs lo, hi;
  CDB_CUDA(lo.bind(p, k1, low_sel, low_coef, low_count, low_rnorm, low_scans, low_flag, st));
  CDB_CUDA(hi.bind(p, k_high, high_sel, high_coef, high_count, high_rnorm, high_scans, high_flag, st));
  StepTimer tm;
  cdb_status s = zero_tree_core(low, high, fine_shape, factors, rank, y_in.dev, f32, p, k1, k_high,
                                rel_tol, phi_mode, lo, hi, engine, step_ms ? &tm : nullptr, di, st);
  if (s != CDB_OK) return s;
  CDB_CUDA(lo.finish(st));
  CDB_CUDA(hi.finish(st));
  CDB_CUDA(cudaStreamSynchronize(st));
  tm.finish(step_ms);
  return CDB_OK;
}

cdb_status cdb_zero_tree_batch_cols(const cdb_dictionary *low, const cdb_dictionary *high,
                                    const int64_t *fine_shape, const int64_t *factors, int rank,
                                    const void *ys_cols, int ys_is_f32, int64_t ld, int64_t p,
                                    int64_t k1, int64_t k_high, double rel_tol, int phi_mode,
                                    int64_t *low_sel, double *low_coef, int64_t *low_count,
                                    double *low_rnorm, int64_t *low_scans, uint8_t *low_flag,
                                    int64_t *high_sel, double *high_coef, int64_t *high_count,
                                    double *high_rnorm, int64_t *high_scans, uint8_t *high_flag,
                                    int engine, float *step_ms, void *stream) {
  if (!low || !high || p < 0 || k1 < 1 || k_high < 1 || high->t % low->t || ld < p)
    return fail(CDB_ERR_ARG, "bad zero-tree arguments");
  if (!phi_mode && (!fine_shape || !factors || rank < 1 || rank > 4))
    return fail(CDB_ERR_ARG, "bad scale spec");
  if (phi_mode && low->n != high->n) return fail(CDB_ERR_ARG, "Phi mode needs equal M");
  if (p == 0) return CDB_OK;
  if (!ys_cols || is_device_ptr(ys_cols)) return fail(CDB_ERR_ARG, "ys_cols must be host memory");
  DevInfo di;
  cdb_status s0 = device_info(di);
  if (s0 != CDB_OK) return s0;
  if ((s0 = check_device(low)) != CDB_OK || (s0 = check_device(high)) != CDB_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  const bool src_f32 = ys_is_f32 != 0;
  const int64_t n = high->n;
  if (step_ms) step_ms[0] = step_ms[1] = 0.0f;
  std::vector<RowArr> arrs = {
      {low_sel, sizeof(int64_t) * k1, true}, {low_coef, sizeof(double) * k1, true},
      {low_count, sizeof(int64_t), true}, {low_rnorm, sizeof(double), true},
      {low_scans, sizeof(int64_t), true}, {low_flag, sizeof(uint8_t), true},
      {high_sel, sizeof(int64_t) * k_high, true}, {high_coef, sizeof(double) * k_high, true},
      {high_count, sizeof(int64_t), true}, {high_rnorm, sizeof(double), true},
      {high_scans, sizeof(int64_t), true}, {high_flag, sizeof(uint8_t), true}};
  for (const RowArr &a : arrs)
    if (!a.host) return fail(CDB_ERR_ARG, "null output");
  if (!all_host(arrs)) {
    // device outputs: the whole column batch in one 2-D copy, transposed on
    // the device, then the device-resident solve
    const size_t es = src_f32 ? 4 : 8;
    DevBuf cb, rb;
    CDB_CUDA(cb.alloc(es * n * p, st));
    CDB_CUDA(rb.alloc(es * n * p, st));
    CDB_CUDA(cudaMemcpy2DAsync(cb.ptr, p * es, ys_cols, ld * es, p * es, n, cudaMemcpyHostToDevice,
                               st));
    CDB_CUDA(cdb::launch_cols_to_rows(cb.ptr, src_f32, n, p, rb.ptr, st));
    Outs lo, hi;
    CDB_CUDA(lo.bind(p, k1, low_sel, low_coef, low_count, low_rnorm, low_scans, low_flag, st));
    CDB_CUDA(hi.bind(p, k_high, high_sel, high_coef, high_count, high_rnorm, high_scans, high_flag,
                     st));
    StepTimer tm;
    cdb_status s = zero_tree_core(low, high, fine_shape, factors, rank, rb.ptr, src_f32, p, k1,
                                  k_high, rel_tol, phi_mode, lo, hi, engine,
                                  step_ms ? &tm : nullptr, di, st);
    if (s != CDB_OK) return s;
    CDB_CUDA(lo.finish(st));
    CDB_CUDA(hi.finish(st));
    CDB_CUDA(cudaStreamSynchronize(st));
    tm.finish(step_ms);
    return CDB_OK;
  }
  auto run = [&](bool try_f32) -> cdb_status {
    bool f32 = try_f32;
    StepTimer tm;
    cdb_status s = run_pipelined_cols(
        p, n, ys_cols, src_f32, ld, arrs, st,
        [&](int64_t, int64_t len, const void *rows, bool rows_f32, std::vector<void *> &dv,
            cudaStream_t s2) -> cdb_status {
          Outs lo, hi;
          dev_outs(lo, dv[0], dv[1], dv[2], dv[3], dv[4], dv[5]);
          dev_outs(hi, dv[6], dv[7], dv[8], dv[9], dv[10], dv[11]);
          return zero_tree_core(low, high, fine_shape, factors, rank, rows, rows_f32, len, k1,
                                k_high, rel_tol, phi_mode, lo, hi, engine,
                                step_ms ? &tm : nullptr, di, s2);
        },
        &f32);
    if (step_ms) step_ms[0] = step_ms[1] = 0.0f;
    tm.finish(step_ms);
    return s;
  };
  cdb_status s = run(!src_f32);
  if (s == kRetryF64) s = run(false);  // a later slab was not fp32-exact
  return s;
}

cdb_status cdb_ksvd_update(int64_t n, int64_t m, int64_t t, const double *y_rows, double *e_rows,
                           double *d_rows, const int64_t *atom_ptr, const int64_t *atom_sig,
                           double *vals, int64_t nnz, int64_t max_users, int64_t threshold,
                           int64_t *replaced, void *stream) {
  if (n < 1 || m < 1 || t < 1 || nnz < 0 || max_users < 0 || max_users > m || !y_rows ||
      !e_rows || !d_rows || !atom_ptr || (nnz > 0 && (!atom_sig || !vals)) || !replaced)
    return fail(CDB_ERR_ARG, "bad K-SVD update arguments");
  DevInfo di;
  cdb_status s0 = device_info(di);
  if (s0 != CDB_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  InArr y_in, p_in, s_in;
  IoArr e_io, d_io, v_io;
  OutArr r_out;
  CDB_CUDA(y_in.bind(y_rows, sizeof(double) * m * n, st));
  CDB_CUDA(p_in.bind(atom_ptr, sizeof(int64_t) * (t + 1), st));
  CDB_CUDA(s_in.bind(atom_sig, sizeof(int64_t) * (nnz > 0 ? nnz : 1), st));
  CDB_CUDA(e_io.bind(e_rows, sizeof(double) * m * n, st));
  CDB_CUDA(d_io.bind(d_rows, sizeof(double) * t * n, st));
  CDB_CUDA(v_io.bind(vals, sizeof(double) * (nnz > 0 ? nnz : 1), st));
  CDB_CUDA(r_out.bind(replaced, sizeof(int64_t), st));
  const int64_t budget = (200 * 1024) / 8 - 4 * n - 32 - 33 * n;  // see ksvd_update_smem
  if (budget < 64) return fail(CDB_ERR_ARG, "signal dimension too large for the update kernel");
  const int64_t smem_b = n * n <= budget ? n * n : budget;
  DevBuf ej, bg, taken;
  CDB_CUDA(ej.alloc(sizeof(double) * (max_users > 0 ? max_users : 1) * n, st));
  CDB_CUDA(bg.alloc(n * n > smem_b ? sizeof(double) * n * n : 16, st));
  CDB_CUDA(taken.alloc(sizeof(uint32_t) * ((m + 31) / 32), st));
  CDB_CUDA(cudaMemsetAsync(taken.ptr, 0, sizeof(uint32_t) * ((m + 31) / 32), st));
  cdb::KsvdArgs a{};
  a.y = (const double *)y_in.dev;
  a.e = (double *)e_io.dev;
  a.d = (double *)d_io.dev;
  a.ptr = (const int64_t *)p_in.dev;
  a.sig = (const int64_t *)s_in.dev;
  a.val = (double *)v_io.dev;
  a.n = n;
  a.m = m;
  a.t = t;
  a.threshold = threshold;
  a.smem_b = smem_b;
  a.ej = ej.as<double>();
  a.bglob = bg.as<double>();
  a.taken = taken.as<uint32_t>();
  a.replaced = (int64_t *)r_out.dev;
  DevBuf prof;
  const bool kprof = getenv("CDB_KSVD_PROF") != nullptr;
  if (kprof) {
    CDB_CUDA(prof.alloc(16 * sizeof(long long), st));
    CDB_CUDA(cudaMemsetAsync(prof.ptr, 0, 16 * sizeof(long long), st));
    a.prof = (long long *)prof.ptr;
  }
  CDB_CUDA(cdb::launch_ksvd_update(a, cdb::ksvd_update_smem(n, smem_b), st));
  if (kprof) {
    long long hp[16];
    CDB_CUDA(cudaMemcpyAsync(hp, prof.ptr, sizeof(hp), cudaMemcpyDeviceToHost, st));
    CDB_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "ksvd phases (k cycles):");
    for (int i = 0; i < 13; i++) fprintf(stderr, " %d:%.0f", i, hp[i] * 1e-3);
    fprintf(stderr, "\n");
  }
  CDB_CUDA(e_io.finish(st));
  CDB_CUDA(d_io.finish(st));
  CDB_CUDA(v_io.finish(st));
  CDB_CUDA(r_out.finish(st));
  CDB_CUDA(cudaStreamSynchronize(st));
  return CDB_OK;
}

}  // extern "C"
