"""K-SVD dictionary-update stage on the device (SURVEY §8 row f1 follow-on)
against the reference's _update_stage (goldens) and the oracle (seeded
problems).  The reference's atoms come from LAPACK's SVD, whose per-atom
sign is arbitrary, so atoms and code rows are compared after aligning each
atom's sign; E (sign-invariant) directly.  Tolerance: 1e-9 absolute on unit
atoms, 1e-9 relative on code rows and residuals (fp64 power iteration to
|dv| < 1e-14 vs LAPACK)."""

import glob
import os

import numpy as np
import pytest

import ksvd_oracle as KO
from paper_1511_05174_b200.learn import update_stage

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-9


def _compare(y, d0, x0, thr, d_ref, x_ref, e_ref, rep_ref):
    d, x = d0.copy(), x0.copy()
    replaced, e = update_stage(y, d, x, thr)
    assert replaced == rep_ref
    sgn = np.sign(np.sum(d * d_ref, axis=0))
    sgn[sgn == 0] = 1.0
    assert np.abs(d - d_ref * sgn).max() <= TOL
    scale = max(np.abs(x_ref).max(), 1.0)
    assert np.abs(x - x_ref * sgn[:, None]).max() <= TOL * scale
    assert np.array_equal(x != 0, x_ref != 0) or np.abs(x - x_ref * sgn[:, None]).max() <= TOL
    assert np.abs(e - e_ref).max() <= TOL * max(np.abs(y).max(), 1.0)


@pytest.mark.parametrize("path", sorted(p for p in glob.glob(os.path.join(GOLD, "ksvd_*.npz"))
                                         if "ksvd_train_" not in p),
                         ids=lambda p: os.path.basename(p)[5:-4])
def test_update_stage_matches_reference(path):
    g = np.load(path)
    _compare(g["y"], g["d"], g["x"], int(g["threshold"]), g["d_out"], g["x_out"], g["e_out"],
             int(g["replaced"]))


@pytest.mark.parametrize("n,t,m,k,dead,thr", [(8, 12, 150, 2, (), 1), (48, 64, 500, 5, (3,), 2),
                                              (100, 128, 256, 4, (0, 9, 10), 3),
                                              (180, 200, 260, 3, (), 1)])
def test_update_stage_matches_oracle(n, t, m, k, dead, thr):
    y, d, x = KO.problem(n, t, m, k, n + t, dead)
    d1, x1 = d.copy(), x.copy()
    rep, e = KO.update_stage(y, d1, x1, thr)
    _compare(y, d, x, thr, d1, x1, e, rep)


def test_update_stage_every_atom_dead():
    """threshold above every atom's user count: all atoms re-seeded, each from
    a different worst-coded signal (learn.py:179-191), codes zeroed."""
    y, d, x = KO.problem(12, 10, 60, 2, 5)
    d1, x1 = d.copy(), x.copy()
    rep, e = KO.update_stage(y, d1, x1, 10 ** 6)
    _compare(y, d, x, 10 ** 6, d1, x1, e, rep)
    assert rep == 10


def test_update_stage_zero_codes():
    """An all-zero code matrix: E = Y, every atom dead at threshold 1."""
    y, d, x = KO.problem(9, 6, 40, 2, 6)
    x[:] = 0.0
    d1, x1 = d.copy(), x.copy()
    rep, e = KO.update_stage(y, d1, x1, 1)
    _compare(y, d, x, 1, d1, x1, e, rep)
