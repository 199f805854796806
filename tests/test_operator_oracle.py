"""The operator-recovery oracle (oracle/operator_oracle.py) against the
reference's own outputs (tests/golden/operator_*.npz), and the host-side
all-patches slicing (sensing.coded_problems) against the oracle's per-patch
patch_problem / apply_matrix restatement -- CPU only."""

import glob
import os

import numpy as np
import pytest

import operator_oracle as OO
from paper_1511_05174_b200 import sensing as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(glob.glob(os.path.join(GOLD, "operator_*.npz")))


def make_op(g):
    """The golden's operator, rebuilt with this package's constructors."""
    kind = str(g["kind"])
    sig = tuple(int(e) for e in g["sig_shape"])
    if kind == "mask":
        return S.mask_from_tensor(g["known"])
    if kind == "channel-mosaic":
        return S.make_channel_mosaic(g["assignment"].size, int(g["channels"]), g["assignment"])
    if kind == "temporal-code":
        f = int(g["frames"])
        return S.make_temporal_code(int(np.prod(sig[:-1])), f, g["code"])
    if kind == "angular-sample":
        return S.make_angular_sample(int(np.prod(sig[:-2])), tuple(g["view_grid"]), g["kept"])
    raise ValueError(kind)


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[9:-4])
def test_oracle_matches_reference(path):
    g = np.load(path)
    r = OO.recover(g)
    assert r["flagged"] == int(g["flagged"])
    assert r["scans1"] == int(g["scans1"]) and r["scans2"] == int(g["scans2"])
    assert np.array_equal(r["resid"], g["resid"])
    np.testing.assert_allclose(r["estimate"], g["estimate"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[9:-4])
def test_coded_problems_match_patch_problem(path):
    g = np.load(path)
    op = make_op(g)
    sig = tuple(int(e) for e in g["sig_shape"])
    patch = tuple(int(e) for e in g["patch"])
    stride = tuple(int(e) for e in g["stride"])
    ys, rows, m = S.coded_problems(op, g["meas"], sig, patch, stride)
    _, origins, _ = OO.PO.extract_patches(np.zeros(sig), patch, stride)
    assert ys.shape[0] == len(origins) == m.size
    n = int(np.prod(patch))
    atoms = np.random.default_rng(0).standard_normal((n, 7))
    opd = {k: g[k] for k in ("known", "assignment", "channels", "code", "frames", "view_grid",
                             "kept") if k in g}
    for p, o in enumerate(origins):
        gather, code, y = OO._local_ops(str(g["kind"]), opd, sig, patch, o, g["meas"])
        if y is None:
            assert m[p] == 0
            continue
        assert m[p] == y.size and np.array_equal(ys[p, :m[p]], y)
        want = OO._apply(gather, code, atoms)
        got = np.zeros((m[p], atoms.shape[1]))
        for i in range(m[p]):  # eff_at: ordered sum of the listed sources
            src = rows[p, i][rows[p, i] >= 0]
            acc = atoms[src[0]].copy()
            for s in src[1:]:
                acc = acc + atoms[s]
            got[i] = acc
        assert np.array_equal(got, want)


def test_operator_constructors_reject_bad_input():
    from paper_1511_05174_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        S.make_temporal_code(2, 2, [[0, 0], [1, 0]])
    with pytest.raises(ConfigError):
        S.make_channel_mosaic(2, 3, [1, 4])
    with pytest.raises(ConfigError):
        S.make_angular_sample(2, (2, 2), [5])
    with pytest.raises(ConfigError):
        S.make_mask(4, [])
    with pytest.raises(ConfigError):
        S.coded_problems(S.make_dense(np.eye(4)), np.zeros(4), (4,), (2,), (1,))


def _np_pairwise(v):
    """numpy's pairwise_sum for n <= 128 (what eff_at ord 1 restates)."""
    n = len(v)
    if n < 8:
        r = 0.0
        for x in v:
            r = r + x
        return r
    r = list(v[:8])
    i = 8
    while i < n - (n % 8):
        for j in range(8):
            r[j] = r[j] + v[i + j]
        i += 8
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    for x in v[i:]:
        res = res + x
    return res


@pytest.mark.parametrize("frames", [3, 8, 9, 16, 21])
def test_slot_rows_pairwise_match_step2_layout(frames):
    """Slot rows summed in numpy's pairwise order equal phi.apply_matrix on the
    F-layout step-2 columns d_high.atoms_t[allowed0].T (crossscale.py:215)."""
    rng = np.random.default_rng(frames)
    spatial = (6, 5)
    ns = int(np.prod(spatial))
    code = (rng.random((ns, frames)) < 0.6).astype(float)
    code[code.sum(1) == 0, 0] = 1.0
    op = S.make_temporal_code(ns, frames, code)
    sig, patch, stride = spatial + (frames,), (3, 3, frames), (2, 1, 1)
    meas = rng.standard_normal(spatial)
    ys, rows, m = S.coded_problems(op, meas, sig, patch, stride, slots=True)
    n = int(np.prod(patch))
    atoms_t = rng.standard_normal((11, n))
    allowed0 = np.array([1, 2, 5, 6, 9])
    cols = atoms_t[allowed0].T  # F layout, as the reference's step 2
    _, origins, _ = OO.PO.extract_patches(np.zeros(sig), patch, stride)
    for p, o in enumerate(origins):
        gather, lc, _ = OO._local_ops("temporal-code", {"code": code, "frames": frames}, sig,
                                      patch, o, meas)
        want = OO._apply(gather, lc, cols)
        for i in range(m[p]):
            v = [[atoms_t[a, s] if s >= 0 else 0.0 for s in rows[p, i]] for a in allowed0]
            got = np.array([_np_pairwise(x) for x in v])
            assert np.array_equal(got, want[i])
