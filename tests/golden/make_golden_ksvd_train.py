"""Golden outputs of the REFERENCE's K-SVD training:
crossdict.learn.ksvd and ksvd_constrained with a block hint (learn.py:265-331)
on seeded data -- objective traces, replaced-atom counts, the final
dictionary and codes.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_ksvd_train.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import crossdict.pursuit as cpursuit  # noqa: E402
from crossdict.learn import TrainConfig, ksvd, ksvd_constrained, train_cross_scale  # noqa: E402
from crossdict.scaling import ScaleSpec  # noqa: E402


def data(n, t, m, k, seed):
    rng = np.random.default_rng(seed)
    dt = rng.standard_normal((n, t))
    dt /= np.linalg.norm(dt, axis=0)
    x = np.zeros((t, m))
    for p in range(m):
        sup = rng.choice(t, size=k, replace=False)
        x[sup, p] = rng.standard_normal(k)
    return dt @ x + 0.02 * rng.standard_normal((n, m))


def save(name, y, d, codes, rep, **extra):
    t = d.atom_dim and d.num_atoms
    x = np.zeros((t, y.shape[1]))
    for p, c in enumerate(codes):
        for i, v in c.entries:
            x[i - 1, p] = v
    np.savez_compressed(os.path.join(HERE, f"ksvd_train_{name}.npz"), y=y, d=d.atoms, x=x,
                        pre=np.array(rep.objective_pre_update),
                        post=np.array(rep.objective_per_iteration),
                        replaced=rep.replaced_atoms, **extra)


def main():
    cpursuit.REL_RESIDUAL_TOL = 1e-6
    y = data(16, 24, 300, 3, 5)
    cfg = TrainConfig(24, 3, iterations=4, seed=1)
    d, codes, rep = ksvd(y, cfg)
    save("plain", y, d, codes, rep, t=24, k=3, iterations=4, seed=1, threshold=1)
    y2 = data(12, 30, 240, 2, 6)
    cfg2 = TrainConfig(30, 2, iterations=3, seed=2, dead_atom_threshold=2)
    d2, codes2, rep2 = ksvd(y2, cfg2)
    save("dead", y2, d2, codes2, rep2, t=30, k=2, iterations=3, seed=2, threshold=2)
    # block-restricted (the two-scale trainer's step 2): 10 blocks of q = 3
    rng = np.random.default_rng(9)
    y3 = data(16, 30, 200, 3, 7)
    blocks = [sorted(rng.choice(10, size=3, replace=False).tolist()) for _ in range(200)]
    sets = [frozenset(int(b) * 3 + c + 1 for b in bl for c in range(3)) for bl in blocks]
    cfg3 = TrainConfig(30, 3, iterations=3, seed=3)
    d3, codes3, rep3 = ksvd_constrained(y3, sets, cfg3, block_hint=(blocks, 3))
    save("blocked", y3, d3, codes3, rep3, t=30, k=3, iterations=3, seed=3, threshold=1,
         blocks=np.array(blocks), q=3)
    # two-scale training (learn.py:334-379): 4 x 4 patches, 2 x 2 blocks
    y4 = data(16, 32, 260, 3, 8)
    model, (rl, rh) = train_cross_scale(y4, ScaleSpec((4, 4), (2, 2)), 8, 32, 2, 4,
                                        iterations=3, seed=4)
    np.savez_compressed(os.path.join(HERE, "train_cross_scale.npz"), y=y4, d_low=model.d_low.atoms,
                        d_high=model.d_high.atoms, pre_low=np.array(rl.objective_pre_update),
                        post_low=np.array(rl.objective_per_iteration),
                        pre_high=np.array(rh.objective_pre_update),
                        post_high=np.array(rh.objective_per_iteration))
    print("wrote ksvd training goldens")


if __name__ == "__main__":
    main()
