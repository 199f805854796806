"""Patch pipeline ends on the device against the
reference's goldens and the patch oracle: extraction and aggregation
bit-exact, reconstruction to fp64 rounding, the device-resident recovery
chain with the parity contract of the pursuit."""

import glob
import os
import warnings

import numpy as np
import pytest
import torch

import patch_oracle as PO
from paper_1511_05174_b200 import device as D
from paper_1511_05174_b200 import patchwork as PW
from paper_1511_05174_b200.crossscale import CrossScaleModel
from paper_1511_05174_b200.pipelines import denoise
from paper_1511_05174_b200.scaling import ScaleSpec
from paper_1511_05174_b200.tensor import Dictionary

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "patch_extract_*.npz"))))
def test_extract_bit_exact(path):
    g = np.load(path)
    cols, grid = PW.extract_patches(g["signal"], tuple(g["patch"]), tuple(g["stride"]),
                                    remove_dc=bool(g["remove_dc"]))
    assert np.array_equal(cols, g["cols"])
    assert np.array_equal(grid.origins, g["origins"])
    if bool(g["remove_dc"]):
        assert np.array_equal(grid.dc_values, g["dc"])
    else:
        assert grid.dc_values is None


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "patch_aggregate_*.npz"))))
def test_aggregate_bit_exact(path):
    g = np.load(path)
    shape, patch, stride = tuple(g["signal_shape"]), tuple(g["patch"]), tuple(g["stride"])
    _, grid = PW.extract_patches(np.zeros(shape), patch, stride, remove_dc=bool(g["add_dc"]))
    if bool(g["add_dc"]):
        grid = PW.PatchGrid(grid.signal_shape, grid.patch_shape, grid.stride, grid.origins, g["dc"])
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        out = np.asarray(PW.aggregate_patches(g["cols"], grid, add_dc=bool(g["add_dc"])))
    assert np.array_equal(out, g["out"])
    assert (len(w) > 0) == bool(g["warned"])


def test_aggregate_shape_errors():
    _, grid = PW.extract_patches(np.zeros((8, 8)), (4, 4), 2)
    from paper_1511_05174_b200.errors import DimensionError
    with pytest.raises(DimensionError):
        PW.aggregate_patches(np.zeros((16, grid.patch_count + 1)), grid)
    with pytest.raises(DimensionError):
        PW.aggregate_patches(np.zeros((16, grid.patch_count)), grid, add_dc=True)
    with pytest.raises(DimensionError):
        PW.extract_patches(np.zeros((8, 8)), (9, 2))


def test_reconstruct_aggregate_matches_reference_chain():
    g = np.load(os.path.join(GOLD, "patch_recover_omp.npz"))
    _, grid = PW.extract_patches(g["signal"], tuple(g["patch"]), tuple(g["stride"]), True)

    class S:  # the solve fields reconstruct_aggregate reads
        sel, alpha = g["sel"], g["alpha"]
    out = np.asarray(PW.reconstruct_aggregate(np.ascontiguousarray(g["atoms"].T), S, grid, True))
    np.testing.assert_allclose(out, g["estimate"], rtol=0, atol=1e-12)


def test_denoise_omp_matches_reference_chain():
    g = np.load(os.path.join(GOLD, "patch_recover_omp.npz"))
    est, solve, _ = denoise(g["signal"], tuple(g["patch"]), tuple(g["stride"]),
                            dictionary=g["atoms"], sparsity=int(g["k"]))
    assert np.array_equal(solve.sel, g["sel"])
    np.testing.assert_allclose(solve.alpha, g["alpha"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.asarray(est), g["estimate"], rtol=0, atol=1e-10)


def test_denoise_zero_tree_matches_reference_chain():
    g = np.load(os.path.join(GOLD, "patch_recover_zt.npz"))
    model = CrossScaleModel(Dictionary(g["low_atoms"]), Dictionary(g["high_atoms"]),
                            ScaleSpec(tuple(g["patch"]), tuple(g["factors"])), int(g["k_low"]),
                            int(g["k_high"]))
    est, (low, high), _ = denoise(g["signal"], tuple(g["patch"]), tuple(g["stride"]), model=model)
    assert np.array_equal(low.sel, g["low_sel"])
    assert np.array_equal(high.sel, g["sel"])
    np.testing.assert_allclose(np.asarray(est), g["estimate"], rtol=0, atol=1e-10)


@pytest.mark.parametrize("shape,patch,stride", [((256, 256), (8, 8), (1, 1)),
                                                ((64, 48, 12), (8, 8, 4), (2, 2, 1))])
def test_large_extract_aggregate_vs_oracle(shape, patch, stride):
    rng = np.random.default_rng(sum(shape))
    sig = rng.standard_normal(shape).astype(np.float32)  # fp32 input, fp64 rows
    rows, grid = PW.extract_rows(sig, patch, stride, remove_dc=True)
    cols, origins, dc = PO.extract_patches(sig.astype(np.float64), patch, stride, True)
    assert np.array_equal(rows, cols.T) and np.array_equal(grid.dc_values, dc)
    vals = rng.standard_normal(cols.shape)
    out = np.asarray(PW.aggregate_patches(vals, grid, add_dc=True))
    ref, unc = PO.aggregate_patches(vals, origins, shape, patch, dc)
    assert unc == 0 and np.array_equal(out, ref)


def test_device_tensor_signal_keeps_rows_on_device():
    sig = torch.randn(40, 33, dtype=torch.float64, device="cuda")
    rows = torch.empty(((40 - 5) // 1 + 1) * ((33 - 5) // 2 + 1), 25, dtype=torch.float64,
                       device="cuda")
    dc = torch.empty(rows.shape[0], dtype=torch.float64, device="cuda")
    D.extract_patches_raw(sig, (5, 5), (1, 2), True, rows, dc)
    cols, _, dcr = PO.extract_patches(sig.cpu().numpy(), (5, 5), (1, 2), True)
    assert np.array_equal(rows.cpu().numpy(), cols.T) and np.array_equal(dc.cpu().numpy(), dcr)
