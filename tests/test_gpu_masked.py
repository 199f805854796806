"""Masked (inpainting) recovery on the device against the
reference's own recover() with a mask operator: per-patch residual norms,
scan counts, flagged patches and the estimate."""

import glob
import os

import numpy as np
import pytest

from paper_1511_05174_b200.pipelines import recover_masked

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "masked_*.npz"))))
def test_masked_recovery_matches_reference(path):
    g = np.load(path)
    est, solve, flagged = recover_masked(g["meas"], g["known"], tuple(g["patch"]),
                                         tuple(g["stride"]), dictionary=g["atoms"],
                                         sparsity=int(g["k"]))
    assert flagged == int(g["flagged"])
    live = solve.counts > 0
    # exact engine on the compacted effective dictionaries: bit-identical residuals
    assert np.array_equal(solve.rnorm[live], g["resid"][live])
    assert int(solve.scans.sum()) == int(g["scans"])
    # reconstruction sums picks in pick order (the reference: sorted support, BLAS)
    np.testing.assert_allclose(np.asarray(est), g["estimate"], rtol=0, atol=1e-12)


def test_mask_shape_mismatch():
    from paper_1511_05174_b200.errors import DimensionError
    with pytest.raises(DimensionError):
        recover_masked(np.zeros((8, 8)), np.ones((8, 7), bool), (4, 4), 2,
                       dictionary=np.eye(16), sparsity=2)
