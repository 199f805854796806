"""The K-SVD update-stage oracle (oracle/ksvd_oracle.py) reproduces the
reference's _update_stage bit for bit on its goldens (CPU only)."""

import glob
import os

import numpy as np
import pytest

import ksvd_oracle as KO

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "ksvd_*.npz"))),
                         ids=lambda p: os.path.basename(p)[5:-4])
def test_update_stage_oracle_matches_reference(path):
    g = np.load(path)
    d, x = g["d"].copy(), g["x"].copy()
    replaced, e = KO.update_stage(g["y"], d, x, int(g["threshold"]))
    assert replaced == int(g["replaced"])
    assert np.array_equal(d, g["d_out"])
    assert np.array_equal(x, g["x_out"])
    assert np.array_equal(e, g["e_out"])
