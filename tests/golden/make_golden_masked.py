"""Golden outputs of the REFERENCE's masked recovery:
crossdict.pipelines.recover with a mask operator (pipelines.py:175-197,
_recover_operator 256-322, sensing.patch_problem mask branch).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_masked.py
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import crossdict.pursuit as cpursuit  # noqa: E402
from crossdict.pipelines import PipelineConfig, recover  # noqa: E402
from crossdict.sensing import make_mask  # noqa: E402
from crossdict.tensor import normalize_atoms  # noqa: E402


def case(name, shape, patch, stride, k, frac, hole, rng):
    sig = np.cumsum(rng.standard_normal(shape), axis=-1) / 4.0
    known = rng.random(shape) < frac
    if hole is not None:
        known[hole] = False
    n = int(np.prod(patch))
    d = normalize_atoms(rng.standard_normal((n, 3 * n)))
    phi = make_mask(int(np.prod(shape)), (np.flatnonzero(known.ravel()) + 1).tolist())
    meas = np.where(known, sig, 0.0)
    cfg = PipelineConfig("omp-single", d, patch_shape=patch, stride=stride, sparsity=k)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        est, metrics = recover(meas, phi, cfg, signal_shape=shape)
    np.savez_compressed(os.path.join(HERE, f"masked_{name}.npz"), meas=meas, known=known,
                        atoms=d.atoms, patch=np.array(patch), stride=np.array(stride), k=k,
                        estimate=np.asarray(est), flagged=metrics.flagged_patches,
                        resid=np.asarray(metrics.residual_norms),
                        scans=metrics.scan_count_step1)


def main():
    cpursuit.REL_RESIDUAL_TOL = 1e-6
    rng = np.random.default_rng(322)
    case("2d", (24, 22), (4, 4), (2, 2), 4, 0.6, (slice(4, 9), slice(4, 9)), rng)
    case("2d_s1", (16, 15), (4, 4), (1, 1), 3, 0.5, None, rng)
    case("1d", (61,), (8,), (3,), 3, 0.7, slice(20, 29), rng)
    print("wrote masked goldens")


if __name__ == "__main__":
    main()
