"""Seeded random zero-tree problems (ranks 1-3, odd extents, factors 1-3, Q
from 1 to 8, budgets up to the model limits, fp32 and fp64 signals, the Phi
path on random effective dictionaries) on the device against the oracle:
step 1 with the parity contract; step 2 on the signals whose step 1 support
matched (its candidate set then equals the oracle's), also with the contract
plus the nesting invariant (crossscale.py:224)."""

import numpy as np
import pytest

from parity import check_zero_tree

import oracle as O
from paper_1511_05174_b200 import _native as N
from paper_1511_05174_b200 import device as D

pytestmark = pytest.mark.gpu

CASES = [  # fine_shape, factors, T_low, Q, k_low, k_high, P
    ((12,), (2,), 9, 3, 3, 5, 64),
    ((6, 4), (2, 2), 10, 2, 4, 6, 64),
    ((9, 6), (3, 2), 13, 4, 5, 9, 48),
    ((8, 8), (2, 2), 64, 4, 8, 8, 96),
    ((6, 6, 2), (3, 3, 2), 7, 5, 2, 7, 48),
    ((8, 8, 4), (2, 2, 2), 256, 8, 16, 16, 128),
    ((10, 10), (5, 2), 31, 1, 6, 6, 40),
]


def _model(fine, fac, t_low, q, seed):
    rng = np.random.default_rng(seed)
    coarse = tuple(e // f for e, f in zip(fine, fac))
    n_low, n = int(np.prod(coarse)), int(np.prod(fine))
    d_low = rng.standard_normal((t_low, n_low))
    d_low /= np.linalg.norm(d_low, axis=1, keepdims=True)
    up = d_low.reshape((t_low,) + coarse)
    for ax, f in enumerate(fac):
        up = np.repeat(up, f, axis=ax + 1)
    up = up.reshape(t_low, n)
    d_high = np.repeat(up, q, axis=0) + 0.3 * rng.standard_normal((t_low * q, n))
    d_high /= np.linalg.norm(d_high, axis=1, keepdims=True)
    return d_low, d_high


def _signals(d_high, q, k, p, seed):
    rng = np.random.default_rng(seed + 1)
    t_low = d_high.shape[0] // q
    ys = np.zeros((p, d_high.shape[1]))
    for i in range(p):
        par = rng.choice(t_low, size=min(k, t_low), replace=False)
        ch = par * q + rng.integers(0, q, size=par.size)
        ys[i] = rng.standard_normal(ch.size) @ d_high[ch]
    ys += 0.01 * rng.standard_normal(ys.shape)
    ys[0] = 0.0
    return ys


def _check_zt(d_low_t, d_high_t, q, ys, low, high, rl, rh, k1, yl=None):
    check_zero_tree(d_low_t, d_high_t, q, ys, low, high, rl, rh, yl)


def _dev_outs(o):
    o = dict(o)
    o["flag"] = np.asarray(o["flag"]).astype(bool)
    return o


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("f32", [True, False])
def test_random_zero_tree(case, f32):
    fine, fac, t_low, q, k1, k2, p = case
    d_low, d_high = _model(fine, fac, t_low, q, t_low * q + len(fine))
    ys = _signals(d_high, q, k1, p, t_low)
    if f32:
        ys = ys.astype(np.float32).astype(np.float64)
    rl, rh = O.zero_tree_many_arrays(d_low, d_high, fine, fac, k1, k2, ys, rel_tol=1e-3)
    lo, hi, ms = D.zero_tree_raw(D.DeviceDictionary(d_low), D.DeviceDictionary(d_high), fine, fac,
                                 ys.astype(np.float32) if f32 else ys, p, k1, k2, 1e-3, False,
                                 "auto")
    yl = O.downsample_rows(ys, fine, fac)
    _check_zt(d_low, d_high, q, ys, _dev_outs(lo), _dev_outs(hi), rl, rh, k1, yl)


@pytest.mark.parametrize("m,t_low,q,k1,k2", [(24, 9, 2, 4, 6), (40, 20, 4, 6, 10),
                                             (64, 64, 4, 8, 12)])
def test_random_zero_tree_phi(m, t_low, q, k1, k2):
    rng = np.random.default_rng(m + t_low)
    e_low = rng.standard_normal((t_low, m))
    e_high = np.repeat(e_low, q, axis=0) + 0.3 * rng.standard_normal((t_low * q, m))
    ys = _signals(e_high, q, k1, 48, m)
    rl, rh = O.zero_tree_phi_many(e_low, e_high, k1, k2, ys, rel_tol=1e-3)
    kb = min(k1, m, t_low)
    lo, hi, ms = D.zero_tree_raw(D.DeviceDictionary(e_low), D.DeviceDictionary(e_high), None, None,
                                 ys, ys.shape[0], kb, k2, 1e-3, True, "auto")
    _check_zt(e_low, e_high, q, ys, _dev_outs(lo), _dev_outs(hi), rl, rh, kb)


# Q and N that select each routed-alpha0 kernel (the Gram engine for step 2
# forced, so alpha0 always comes from the routing): the DMMA tiles with the
# children in registers (Q = 8, N <= 256), from L1 (Q = 8 above N = 256,
# Q = 16), and the FFMA warp kernel (Q = 4).
ROUTED = [  # fine_shape, factors, T_low, Q, k_low, k_high, P
    ((8, 16), (2, 2), 20, 8, 4, 8, 64),
    ((8, 8, 8), (2, 2, 2), 24, 8, 4, 8, 64),
    ((16, 16), (2, 2), 12, 16, 4, 8, 64),
    ((8, 8), (2, 2), 16, 4, 4, 6, 64),
]


@pytest.mark.parametrize("case", ROUTED)
@pytest.mark.parametrize("f32", [True, False])
def test_routed_alpha0_kernels(case, f32):
    fine, fac, t_low, q, k1, k2, p = case
    d_low, d_high = _model(fine, fac, t_low, q, 7 * t_low + q)
    ys = _signals(d_high, q, k1, p, t_low + 1)
    if f32:
        ys = ys.astype(np.float32).astype(np.float64)
    rl, rh = O.zero_tree_many_arrays(d_low, d_high, fine, fac, k1, k2, ys, rel_tol=1e-3)
    N.profile_enable(True)
    lo, hi, ms = D.zero_tree_raw(D.DeviceDictionary(d_low), D.DeviceDictionary(d_high), fine, fac,
                                 ys.astype(np.float32) if f32 else ys, p, k1, k2, 1e-3, False,
                                 "gram")
    prof = N.profile_read()
    N.profile_enable(False)
    assert "route_alpha0" in prof, sorted(prof)
    yl = O.downsample_rows(ys, fine, fac)
    _check_zt(d_low, d_high, q, ys, _dev_outs(lo), _dev_outs(hi), rl, rh, k1, yl)
