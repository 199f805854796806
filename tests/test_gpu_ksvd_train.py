"""K-SVD training with both stages on the device:
learn.ksvd / ksvd_constrained against the reference's own runs
(tests/golden/ksvd_train_*.npz): objective traces before and after every
update, replaced-atom counts, the final dictionary and codes.  Atoms (and
their code rows) are compared after aligning each atom's sign -- the
reference's LAPACK SVD fixes it arbitrarily; nothing else depends on it.
Tolerance 1e-8 (relative on objectives, absolute on unit atoms)."""

import glob
import os

import numpy as np
import pytest

from paper_1511_05174_b200 import learn as L
from paper_1511_05174_b200 import pursuit

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "ksvd_train_*.npz"))),
                         ids=lambda p: os.path.basename(p)[11:-4])
def test_ksvd_training_matches_reference(path):
    g = np.load(path)
    old = pursuit.REL_RESIDUAL_TOL
    pursuit.REL_RESIDUAL_TOL = 1e-6
    try:
        cfg = L.TrainConfig(int(g["t"]), int(g["k"]), iterations=int(g["iterations"]),
                            seed=int(g["seed"]), dead_atom_threshold=int(g["threshold"]))
        if "blocks" in g:
            blocks = [list(map(int, b)) for b in g["blocks"]]
            q = int(g["q"])
            sets = [frozenset(b * q + c + 1 for b in bl for c in range(q)) for bl in blocks]
            d, codes, rep = L.ksvd_constrained(g["y"], sets, cfg, block_hint=(blocks, q))
        else:
            d, codes, rep = L.ksvd(g["y"], cfg)
    finally:
        pursuit.REL_RESIDUAL_TOL = old
    np.testing.assert_allclose(rep.objective_pre_update, g["pre"], rtol=1e-8)
    np.testing.assert_allclose(rep.objective_per_iteration, g["post"], rtol=1e-8)
    assert rep.replaced_atoms == int(g["replaced"])
    sgn = np.sign(np.sum(d.atoms * g["d"], axis=0))
    assert np.abs(d.atoms - g["d"] * sgn).max() <= 1e-8
    x = np.zeros_like(g["x"])
    for p, c in enumerate(codes):
        for i, v in c.entries:
            x[i - 1, p] = v
    assert np.abs(x - g["x"] * sgn[:, None]).max() <= 1e-8 * max(1.0, np.abs(g["x"]).max())


def test_train_cross_scale_matches_reference():
    """Two-scale training (learn.py:334-379) on the device loop vs the
    reference's run: both objective traces and both dictionaries."""
    from paper_1511_05174_b200.scaling import ScaleSpec
    g = np.load(os.path.join(GOLD, "train_cross_scale.npz"))
    old = pursuit.REL_RESIDUAL_TOL
    pursuit.REL_RESIDUAL_TOL = 1e-6
    try:
        model, (rl, rh) = L.train_cross_scale(g["y"], ScaleSpec((4, 4), (2, 2)), 8, 32, 2, 4,
                                              iterations=3, seed=4)
    finally:
        pursuit.REL_RESIDUAL_TOL = old
    for got, key in ((rl.objective_pre_update, "pre_low"), (rl.objective_per_iteration, "post_low"),
                     (rh.objective_pre_update, "pre_high"),
                     (rh.objective_per_iteration, "post_high")):
        np.testing.assert_allclose(got, g[key], rtol=1e-8)
    for d, ref in ((model.d_low.atoms, g["d_low"]), (model.d_high.atoms, g["d_high"])):
        sgn = np.sign(np.sum(d * ref, axis=0))
        assert np.abs(d - ref * sgn).max() <= 1e-8
