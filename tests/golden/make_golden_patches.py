"""Golden vectors for the patch pipeline ends, produced by
running the REFERENCE (crossdict) in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_patches.py

* ``patch_extract_*.npz``: signal, geometry, remove_dc -> the reference's
  extract_patches columns, origins and dc (patchwork.py:58-89).
* ``patch_aggregate_*.npz``: columns + geometry (+ dc) -> aggregate_patches
  output (patchwork.py:92-122), including a stride that leaves cells uncovered.
* ``patch_recover_*.npz``: the identity recovery chain exactly as
  pipelines.py:206-248 composes it -- extract_patches(remove_dc=True) ->
  omp_many_arrays (or zero_tree_many_arrays) -> dictionary.atoms @
  coefficient_matrix() -> aggregate_patches(add_dc=True).
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
from crossdict.crossscale import CrossScaleModel, zero_tree_many_arrays  # noqa: E402
from crossdict.patchwork import aggregate_patches, extract_patches  # noqa: E402
from crossdict.pursuit import PursuitConfig, omp_many_arrays  # noqa: E402
from crossdict.scaling import ScaleSpec  # noqa: E402
from crossdict.tensor import normalize_atoms  # noqa: E402

EXTRACT = [  # name, signal shape, patch, stride, remove_dc
    ("1d", (37,), (5,), (2,), False),
    ("2d_dc", (20, 17), (5, 4), (2, 3), True),
    ("2d_s1", (12, 11), (4, 4), (1, 1), False),
    ("3d_dc", (10, 9, 6), (4, 4, 2), (1, 2, 2), True),
    ("4d", (6, 5, 4, 4), (2, 2, 2, 2), (2, 1, 2, 1), True),
]
AGGREGATE = [  # name, signal shape, patch, stride, add_dc
    ("2d", (20, 17), (5, 4), (2, 3), False),
    ("2d_dc", (16, 16), (4, 4), (1, 1), True),
    ("uncovered", (11, 9), (3, 2), (4, 3), False),
    ("3d_dc", (10, 9, 6), (4, 4, 2), (1, 2, 2), True),
]


def main():
    rng = np.random.default_rng(20261020)
    for name, shape, pat, st, dc in EXTRACT:
        sig = rng.standard_normal(shape)
        cols, grid = extract_patches(sig, pat, st, remove_dc=dc)
        np.savez_compressed(os.path.join(HERE, f"patch_extract_{name}.npz"), signal=sig,
                            patch=np.array(pat), stride=np.array(st), remove_dc=dc, cols=cols,
                            origins=grid.origins,
                            dc=grid.dc_values if dc else np.zeros(0))
    for name, shape, pat, st, add in AGGREGATE:
        sig = rng.standard_normal(shape)
        _, grid = extract_patches(sig, pat, st, remove_dc=add)
        cols = rng.standard_normal((grid.patch_size, grid.patch_count))
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            out = np.asarray(aggregate_patches(cols, grid, add_dc=add))
        np.savez_compressed(os.path.join(HERE, f"patch_aggregate_{name}.npz"), signal_shape=np.array(shape),
                            patch=np.array(pat), stride=np.array(st), add_dc=add, cols=cols,
                            dc=grid.dc_values if add else np.zeros(0), out=out,
                            warned=len(w) > 0)
    # identity recovery chain (pipelines.py:206-248), default REL_RESIDUAL_TOL
    cpursuit.REL_RESIDUAL_TOL = 1e-6
    img = np.clip(np.cumsum(rng.standard_normal((24, 22)), axis=1) / 6.0, -2, 2)
    noisy = img + 0.05 * rng.standard_normal(img.shape)
    d = normalize_atoms(rng.standard_normal((16, 48)))
    cols, grid = extract_patches(noisy, (4, 4), (1, 1), remove_dc=True)
    solve = omp_many_arrays(d, cols, PursuitConfig(5))
    est = np.asarray(aggregate_patches(d.atoms @ solve.coefficient_matrix(), grid, add_dc=True))
    np.savez_compressed(os.path.join(HERE, "patch_recover_omp.npz"), signal=noisy,
                        atoms=d.atoms, patch=np.array((4, 4)), stride=np.array((1, 1)), k=5,
                        sel=solve.sel, alpha=solve.alpha, counts=solve.counts, estimate=est)
    # zero-tree variant on a planted cross-scale model
    spec = ScaleSpec((4, 4), (2, 2))
    d_low = normalize_atoms(rng.standard_normal((4, 12)))
    child = []
    for j in range(12):
        base = np.repeat(np.repeat(d_low.atoms[:, j].reshape(2, 2), 2, axis=0), 2, axis=1).ravel()
        for c in range(3):
            child.append(base + 0.3 * rng.standard_normal(16))
    d_high = normalize_atoms(np.stack(child, axis=1))
    model = CrossScaleModel(d_low, d_high, spec, 3, 5)
    cols, grid = extract_patches(noisy, (4, 4), (2, 1), remove_dc=True)
    low, high, _ = zero_tree_many_arrays(model, cols)
    est = np.asarray(aggregate_patches(d_high.atoms @ high.coefficient_matrix(), grid,
                                       add_dc=True))
    np.savez_compressed(os.path.join(HERE, "patch_recover_zt.npz"), signal=noisy,
                        low_atoms=d_low.atoms, high_atoms=d_high.atoms, patch=np.array((4, 4)),
                        stride=np.array((2, 1)), factors=np.array((2, 2)), k_low=3, k_high=5,
                        low_sel=low.sel, sel=high.sel, alpha=high.alpha, estimate=est)
    print("wrote patch goldens")


if __name__ == "__main__":
    main()
