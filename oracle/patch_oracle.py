"""CPU restatement of crossdict's patch pipeline ends --
TEST INFRASTRUCTURE ONLY (imported by tests/ to check the device kernels;
never by the product path).

* extract_patches   patchwork.py:58-89: sliding windows at stride positions,
  row-major patch cells as columns; remove_dc subtracts each column's mean
  (numpy's axis-0 reduction: sequential sum over the cells, then / N).
* aggregate_patches patchwork.py:92-122: for p ascending, acc[window] +=
  column p, weight[window] += 1; uncovered cells -> 0; acc / weight.
* reconstruct       pipelines.py:246: est = atoms @ coef, written as the sum
  over each patch's picks (the dense product adds exact zeros elsewhere).

Pinned bit-exact against the reference's own outputs in
tests/golden/patch_*.npz (tests/golden/make_golden_patches.py).
"""

from __future__ import annotations

import numpy as np


def extract_patches(signal, patch, stride, remove_dc=False):
    arr = np.asarray(signal, dtype=np.float64)
    grid = [(e - q) // s + 1 for e, q, s in zip(arr.shape, patch, stride)]
    origins = np.stack([m.ravel() for m in np.meshgrid(
        *[np.arange(g) * s for g, s in zip(grid, stride)], indexing="ij")], axis=1)
    n = int(np.prod(patch))
    cols = np.empty((n, len(origins)))
    for p, o in enumerate(origins):
        cols[:, p] = arr[tuple(slice(a, a + q) for a, q in zip(o, patch))].ravel()
    dc = None
    if remove_dc:
        dc = np.zeros(cols.shape[1])
        for i in range(n):  # sequential over cells, as numpy's axis-0 reduce
            dc = dc + cols[i]
        dc = dc / n
        cols = cols - dc[None, :]
    return cols, origins.astype(np.int64), dc


def aggregate_patches(cols, origins, signal_shape, patch, dc=None):
    cols = np.asarray(cols, dtype=np.float64)
    if dc is not None:
        cols = cols + dc[None, :]
    acc = np.zeros(signal_shape)
    w = np.zeros(signal_shape)
    for p, o in enumerate(origins):
        win = tuple(slice(a, a + q) for a, q in zip(o, patch))
        acc[win] += cols[:, p].reshape(patch)
        w[win] += 1.0
    unc = w == 0
    w[unc] = 1.0
    return acc / w, int(unc.sum())


def reconstruct(atoms, sel, alpha):
    """Columns atoms @ coef from (sel, alpha) rows (sel -1 padded)."""
    n = atoms.shape[0]
    est = np.zeros((n, sel.shape[0]))
    for p in range(sel.shape[0]):
        for l in range(sel.shape[1]):
            if sel[p, l] < 0:
                break
            est[:, p] += alpha[p, l] * atoms[:, sel[p, l]]
    return est
