"""The K-SVD update-stage oracle (oracle/ksvd_oracle.py) reproduces the
reference's _update_stage bit for bit on its goldens (CPU only)."""

import glob
import os

import numpy as np
import pytest

import ksvd_oracle as KO

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("path", sorted(p for p in glob.glob(os.path.join(GOLD, "ksvd_*.npz"))
                                         if "ksvd_train_" not in p),
                         ids=lambda p: os.path.basename(p)[5:-4])
def test_update_stage_oracle_matches_reference(path):
    g = np.load(path)
    d, x = g["d"].copy(), g["x"].copy()
    replaced, e = KO.update_stage(g["y"], d, x, int(g["threshold"]))
    assert replaced == int(g["replaced"])
    assert np.array_equal(d, g["d_out"])
    assert np.array_equal(x, g["x_out"])
    assert np.array_equal(e, g["e_out"])


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "ksvd_train_*.npz"))),
                         ids=lambda p: os.path.basename(p)[11:-4])
def test_training_oracle_matches_reference(path):
    """The oracle's restated training loop (C coding kernel + numpy update)
    reproduces the reference's K-SVD runs."""
    g = np.load(path)
    kw = {}
    if "blocks" in g:
        kw = dict(blocks=np.sort(g["blocks"], axis=1), q=int(g["q"]))
    d, x, pre, post, rep = KO.train(g["y"], int(g["t"]), int(g["k"]), int(g["iterations"]),
                                    seed=int(g["seed"]), threshold=int(g["threshold"]), **kw)
    assert rep == int(g["replaced"])
    np.testing.assert_allclose(pre, g["pre"], rtol=1e-12)
    np.testing.assert_allclose(post, g["post"], rtol=1e-12)
    np.testing.assert_allclose(d, g["d"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(x, g["x"], rtol=0, atol=1e-12)
