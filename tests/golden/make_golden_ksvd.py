"""Golden outputs of the REFERENCE's K-SVD update stage (SURVEY §8 row f1
follow-on): crossdict.learn._update_stage (learn.py:169-199) on seeded
problems from oracle/ksvd_oracle.problem -- atoms with many users (E_j E_j^T
side), few users (E_j^T E_j side), dead atoms re-seeded.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_ksvd.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from crossdict.learn import _update_stage  # noqa: E402
from ksvd_oracle import problem  # noqa: E402

CASES = {  # name: (n, t, m, k, seed, dead atoms, threshold)
    "left": (16, 24, 400, 3, 11, (), 1),
    "right": (64, 96, 300, 3, 12, (), 1),
    "dead": (32, 40, 200, 4, 13, (5, 6, 17, 30), 2),
}


def main():
    for name, (n, t, m, k, seed, dead, thr) in CASES.items():
        y, d, x = problem(n, t, m, k, seed, dead)
        d1, x1 = d.copy(), x.copy()
        replaced, e = _update_stage(y, d1, x1, thr)
        np.savez_compressed(os.path.join(HERE, f"ksvd_{name}.npz"), y=y, d=d, x=x, threshold=thr,
                            d_out=d1, x_out=x1, e_out=e, replaced=replaced)
    print("wrote ksvd goldens")


if __name__ == "__main__":
    main()
