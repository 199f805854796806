// Candidate-set addressing shared by all engines.
//
// The reference scans either all T atoms or, when `restricted`, the row
// allowed[p, :] of ascending 0-based ids (_kernels.py:70,97,107).  The
// blocked form allowed = blocks * Q + arange(Q) (pursuit.py:421-422) is kept
// implicit here so the P x (nb*Q) expansion is never materialised.
#pragma once
#include <cstdint>

namespace cdb {

struct Cands {
  int mode;               // 0: all T atoms, 1: explicit id list, 2: blocks
  int64_t t;              // dictionary size
  const int64_t *ids;     // mode 1: P x stride ids; mode 2: P x stride block ids
  int64_t stride;         // row stride of ids
  int64_t q;              // mode 2: block size Q
  const int64_t *nb;      // mode 2: per-signal block count (NULL -> nb_fixed)
  int64_t nb_fixed;       // mode 2: block count when nb == NULL
  int clip;               // clip the budget to min(k_max, count, N) per signal

  __device__ __forceinline__ int64_t count(int64_t p) const {
    if (mode == 0) return t;
    if (mode == 1) return stride;
    return (nb ? nb[p] : nb_fixed) * q;
  }
  __device__ __forceinline__ int64_t id(int64_t p, int64_t jl) const {
    if (mode == 0) return jl;
    if (mode == 1) return ids[p * stride + jl];
    return ids[p * stride + jl / q] * q + jl % q;
  }
  __device__ __forceinline__ int64_t budget(int64_t p, int64_t k_max, int64_t n) const {
    if (!clip) return k_max;
    int64_t c = count(p);
    int64_t k = k_max < c ? k_max : c;
    return k < n ? k : n;
  }
};

}  // namespace cdb
