"""The patch-pipeline oracle (oracle/patch_oracle.py) pinned against the
reference's own outputs (tests/golden/patch_*.npz): extraction and
aggregation bit-exact, reconstruction to fp64 rounding."""

import glob
import os

import numpy as np
import pytest

import patch_oracle as PO

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "patch_extract_*.npz"))))
def test_extract_matches_reference(path):
    g = np.load(path)
    cols, origins, dc = PO.extract_patches(g["signal"], tuple(g["patch"]), tuple(g["stride"]),
                                           bool(g["remove_dc"]))
    assert np.array_equal(origins, g["origins"])
    assert np.array_equal(cols, g["cols"])
    if bool(g["remove_dc"]):
        assert np.array_equal(dc, g["dc"])


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "patch_aggregate_*.npz"))))
def test_aggregate_matches_reference(path):
    g = np.load(path)
    shape, patch, stride = tuple(g["signal_shape"]), tuple(g["patch"]), tuple(g["stride"])
    _, origins, _ = PO.extract_patches(np.zeros(shape), patch, stride)
    out, unc = PO.aggregate_patches(g["cols"], origins, shape, patch,
                                    g["dc"] if bool(g["add_dc"]) else None)
    assert np.array_equal(out, g["out"])
    assert (unc > 0) == bool(g["warned"])


def test_recover_chain_matches_reference():
    g = np.load(os.path.join(GOLD, "patch_recover_omp.npz"))
    patch, stride = tuple(g["patch"]), tuple(g["stride"])
    cols, origins, dc = PO.extract_patches(g["signal"], patch, stride, True)
    est = PO.reconstruct(g["atoms"], g["sel"], g["alpha"])
    out, _ = PO.aggregate_patches(est, origins, g["signal"].shape, patch, dc)
    np.testing.assert_allclose(out, g["estimate"], rtol=0, atol=1e-12)
