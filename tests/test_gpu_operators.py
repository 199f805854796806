"""Operator recovery on the device (masks, channel
mosaics, temporal codes, angular sampling; single-scale OMP and zero-tree)
against the reference's own recover() outputs, and seeded random problems
against the oracle (oracle/operator_oracle.py)."""

import glob
import os

import numpy as np
import pytest

import operator_oracle as OO
from test_operator_oracle import make_op

from paper_1511_05174_b200 import sensing as S
from paper_1511_05174_b200.crossscale import CrossScaleModel
from paper_1511_05174_b200.pipelines import recover_operator
from paper_1511_05174_b200.scaling import ScaleSpec
from paper_1511_05174_b200.tensor import Dictionary

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _run(g, rel=1e-6):
    from paper_1511_05174_b200 import pursuit
    old = pursuit.REL_RESIDUAL_TOL
    pursuit.REL_RESIDUAL_TOL = rel
    try:
        op = make_op(g)
        sig = tuple(int(e) for e in g["sig_shape"])
        patch = tuple(int(e) for e in g["patch"])
        stride = tuple(int(e) for e in g["stride"])
        if str(g["method"]) == "zerotree":
            fac = tuple(int(f) for f in g["factors"])
            model = CrossScaleModel(Dictionary(g["d_low"]), Dictionary(g["d_high"]),
                                    ScaleSpec(patch, fac), int(g["k_low"]), int(g["k_high"]))
            return recover_operator(g["meas"], op, patch, stride, model=model, signal_shape=sig)
        return recover_operator(g["meas"], op, patch, stride, dictionary=g["atoms"],
                                sparsity=int(g["k"]), signal_shape=sig)
    finally:
        pursuit.REL_RESIDUAL_TOL = old


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "operator_*.npz"))),
                         ids=lambda p: os.path.basename(p)[9:-4])
def test_operator_recovery_matches_reference(path):
    g = np.load(path)
    est, met, _ = _run(g)
    assert met.flagged_patches == int(g["flagged"])
    assert met.scan_count_step1 == int(g["scans1"])
    assert met.scan_count_step2 == int(g["scans2"])
    # exact engine on the coded effective dictionaries: bit-identical residuals
    assert np.array_equal(met.residual_norms, g["resid"])
    if float(g["nesting"]) >= 0:
        assert met.nesting_ok_fraction == float(g["nesting"])
    np.testing.assert_allclose(np.asarray(est), g["estimate"], rtol=0, atol=1e-12)


def _rand_case(kind, method, seed):
    rng = np.random.default_rng(seed)
    if kind == "temporal-code":
        spatial, f = (11, 9), 8
        ns = int(np.prod(spatial))
        code = (rng.random((ns, f)) < 0.6).astype(float)
        code[code.sum(1) == 0, 3] = 1.0
        g = dict(kind=kind, code=code, frames=f, sig_shape=np.array(spatial + (f,)),
                 patch=np.array((4, 4, f)), stride=np.array((3, 2, 1)),
                 meas=rng.standard_normal(spatial))
    else:
        spatial, c = (13, 10), 4
        a = rng.integers(1, c + 1, int(np.prod(spatial)))
        g = dict(kind=kind, assignment=a, channels=c, sig_shape=np.array(spatial + (c,)),
                 patch=np.array((4, 4, c)), stride=np.array((3, 2, 1)),
                 meas=rng.standard_normal(spatial))
    n = int(np.prod(g["patch"]))
    if method == "zerotree":
        fac = (2, 2, 2) if kind == "temporal-code" else (2, 2, 1)
        coarse = n // int(np.prod(fac))
        dl = rng.standard_normal((coarse, 9))
        dh = rng.standard_normal((n, 9 * 4))
        g.update(method="zerotree", d_low=dl / np.linalg.norm(dl, axis=0),
                 d_high=dh / np.linalg.norm(dh, axis=0), factors=np.array(fac), k_low=4, k_high=7)
    else:
        d = rng.standard_normal((n, 3 * n // 2))
        g.update(method="omp-single", atoms=d / np.linalg.norm(d, axis=0), k=6)
    return g


@pytest.mark.parametrize("kind", ["temporal-code", "channel-mosaic"])
@pytest.mark.parametrize("method", ["omp-single", "zerotree"])
def test_operator_recovery_random_vs_oracle(kind, method):
    g = _rand_case(kind, method, 7 if method == "zerotree" else 8)
    ref = OO.recover(g, rel=1e-3)
    est, met, _ = _run(g, rel=1e-3)
    assert met.flagged_patches == ref["flagged"]
    assert (met.scan_count_step1, met.scan_count_step2) == (ref["scans1"], ref["scans2"])
    assert np.array_equal(met.residual_norms, ref["resid"])
    np.testing.assert_allclose(np.asarray(est), ref["estimate"], rtol=0, atol=1e-10)


def test_dc_removal_refused_for_non_mask():
    from paper_1511_05174_b200.errors import ConfigError
    op = S.make_channel_mosaic(16, 2, np.ones(16, int))
    with pytest.raises(ConfigError):
        recover_operator(np.zeros((4, 4)), op, (2, 2, 2), dictionary=np.eye(8), sparsity=2,
                         remove_dc=True)


def test_recover_operator_stage_fills_reference_metrics():
    """The install() drop-in for pipelines._recover_operator, called the way
    the reference's recover() calls it (pipelines.py:196-197)."""
    from types import SimpleNamespace

    from paper_1511_05174_b200.pipelines import RecoveryMetrics, recover_operator_stage
    g = np.load(os.path.join(GOLD, "operator_temporal_zt8.npz"))
    from paper_1511_05174_b200 import pursuit
    old = pursuit.REL_RESIDUAL_TOL
    pursuit.REL_RESIDUAL_TOL = 1e-6
    try:
        patch = tuple(int(e) for e in g["patch"])
        fac = tuple(int(f) for f in g["factors"])
        model = CrossScaleModel(Dictionary(g["d_low"]), Dictionary(g["d_high"]),
                                ScaleSpec(patch, fac), int(g["k_low"]), int(g["k_high"]))
        cfg = SimpleNamespace(method="zerotree", model=model, remove_dc=None)
        met = RecoveryMetrics("zerotree")
        est, met = recover_operator_stage(g["meas"], make_op(g), tuple(g["sig_shape"]), patch,
                                          tuple(int(e) for e in g["stride"]), cfg, met)
    finally:
        pursuit.REL_RESIDUAL_TOL = old
    assert (met.scan_count_step1, met.scan_count_step2) == (int(g["scans1"]), int(g["scans2"]))
    assert np.array_equal(met.residual_norms, g["resid"])
    assert met.flagged_patches == int(g["flagged"]) and met.patch_count == g["resid"].size
    np.testing.assert_allclose(np.asarray(est), g["estimate"], rtol=0, atol=1e-12)


def test_angular_zero_tree_vs_oracle():
    """Angular sampling with zero-tree coding (the view axes coarsened by 1)."""
    rng = np.random.default_rng(21)
    spatial, grid, kept = (7, 6), (2, 2), np.array([1, 4])
    patch = (4, 4, 2, 2)
    n = int(np.prod(patch))
    fac = (2, 2, 1, 1)
    dl = rng.standard_normal((n // 4, 10))
    dh = rng.standard_normal((n, 30))
    g = dict(kind="angular-sample", view_grid=np.array(grid), kept=kept,
             sig_shape=np.array(spatial + grid), patch=np.array(patch),
             stride=np.array((3, 2, 1, 1)), meas=rng.standard_normal(spatial + (kept.size,)),
             method="zerotree", d_low=dl / np.linalg.norm(dl, axis=0),
             d_high=dh / np.linalg.norm(dh, axis=0), factors=np.array(fac), k_low=3, k_high=5)
    ref = OO.recover(g, rel=1e-3)
    est, met, _ = _run(g, rel=1e-3)
    assert met.flagged_patches == ref["flagged"]
    assert (met.scan_count_step1, met.scan_count_step2) == (ref["scans1"], ref["scans2"])
    assert np.array_equal(met.residual_norms, ref["resid"])
    np.testing.assert_allclose(np.asarray(est), ref["estimate"], rtol=0, atol=1e-10)
