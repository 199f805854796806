"""Golden outputs of the REFERENCE's K-SVD coding stage (crossdict
learn._code_stage, learn.py:240-262) for SURVEY §8 row f1:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_learn.py

Three modes on seeded data: no restriction (omp_many), ragged block hints
(grouped blocked omp_many), explicit allowed sets (per-column omp).  Stored
per sample: selected atoms in pick order (1-based, -1 padded), the code's
support / values, residual norm, iterations, scan count.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from crossdict.learn import _code_stage  # noqa: E402


def pack(results, k):
    m = len(results)
    sel = np.full((m, k), -1, np.int64)
    sup = np.full((m, k), -1, np.int64)
    val = np.zeros((m, k))
    rn, it, sc = np.zeros(m), np.zeros(m, np.int64), np.zeros(m, np.int64)
    for p, r in enumerate(results):
        sel[p, :len(r.selected)] = r.selected
        s = np.asarray(r.code.support, dtype=np.int64)
        sup[p, :len(s)] = s
        val[p, :len(s)] = np.asarray(r.code.coefficients)
        rn[p], it[p], sc[p] = r.residual_norm, r.iterations, r.atom_scan_count
    return dict(sel=sel, support=sup, values=val, rnorm=rn, iterations=it, scans=sc)


def main():
    rng = np.random.default_rng(240)
    n, t, q, k = 16, 48, 4, 5
    d = rng.standard_normal((n, t))
    d /= np.linalg.norm(d, axis=0)
    y = rng.standard_normal((n, 300))
    out = {"d": d, "y": y, "k": k, "q": q}
    for key, v in pack(_code_stage(d, y, k, None, None), k).items():
        out[f"plain_{key}"] = v
    blocks_list = [sorted(rng.choice(t // q, size=rng.integers(1, 6), replace=False).tolist())
                   for _ in range(y.shape[1])]
    allowed = [set(b2 * q + c + 1 for b2 in b for c in range(q)) for b in blocks_list]  # 1-based
    res = _code_stage(d, y, k, allowed, (blocks_list, q))
    for key, v in pack(res, k).items():
        out[f"blocks_{key}"] = v
    nbm = max(len(b) for b in blocks_list)
    bl = np.full((len(blocks_list), nbm), -1, np.int64)
    for p, b in enumerate(blocks_list):
        bl[p, :len(b)] = b
    out["blocks_list"] = bl
    y2 = y[:, :24]
    sets = [sorted((rng.choice(t, size=rng.integers(3, 12), replace=False) + 1).tolist())
            for _ in range(24)]  # 1-based atom ids
    res = _code_stage(d, y2, k, [set(s) for s in sets], None)
    for key, v in pack(res, k).items():
        out[f"sets_{key}"] = v
    sl = np.full((24, 12), -1, np.int64)
    for p, s_ in enumerate(sets):
        sl[p, :len(s_)] = s_
    out["sets_list"] = sl
    np.savez_compressed(os.path.join(HERE, "learn_code_stage.npz"), **out)
    print("wrote learn_code_stage.npz")


if __name__ == "__main__":
    main()
