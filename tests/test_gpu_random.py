"""Seeded random problems across shapes the goldens do not pin: N not a
multiple of 4 / 32 / 64, T not a multiple of 32, K from 1 to N, fp32 and
fp64 signals, near-duplicate atoms (delegation to the exact engine), full
and block-restricted candidates, every engine -- each against the oracle
(oracle/omp_oracle.c) with the parity contract (tests/parity.py); the exact
engine bit-identically."""

import numpy as np
import pytest

from parity import compare

import oracle as O
from paper_1511_05174_b200 import device as D

pytestmark = pytest.mark.gpu

SHAPES = [  # (N, T, K, P)
    (5, 11, 3, 40), (17, 40, 6, 64), (31, 97, 9, 80), (33, 64, 12, 64),
    (64, 256, 8, 96), (70, 300, 10, 64), (129, 513, 16, 48), (256, 1000, 20, 32),
]
ENGINES = ["exact", "gram", "tensor", "resident", "auto"]


def _problem(n, t, k, p, seed, dup):
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((t, n))
    if dup:  # a few near-duplicate atoms: rank trouble for the fast engines
        d[1] = d[0] + 1e-7 * rng.standard_normal(n)
        d[t // 2] = d[2] * 0.5 + d[3] * 0.5
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    x = np.zeros((p, t))
    for i in range(p):
        sup = rng.choice(t, size=min(k, t), replace=False)
        x[i, sup] = rng.standard_normal(sup.size)
    ys = x @ d + 0.01 * rng.standard_normal((p, n))
    ys[0] = 0.0  # zero signal: immediate exit
    return d, ys


def _oracle(d, ys, k, eps, allowed=None):
    sel, coef, count, rnorm, scans, flag = O.omp_batch(d, ys, k, eps, allowed)
    return dict(sel=sel, alpha=coef, counts=count, rnorm=rnorm, scans=scans,
                flag=np.asarray(flag, bool))


def _check(ref, got, d, ys, eps, engine, allowed=None):
    got["flag"] = got["flag"].astype(bool)
    if engine == "exact":
        keep = ~ref["flag"]
        for key in ("counts", "sel", "scans", "flag"):
            assert np.array_equal(got[key], ref[key]), key
        assert np.array_equal(got["alpha"][keep], ref["alpha"][keep])
        assert np.array_equal(got["rnorm"][keep], ref["rnorm"][keep])
        return
    rep = compare(ref, got, d, ys, eps, allowed)
    assert not rep["bad"], rep["bad"][:3]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("engine", ENGINES)
def test_random_full(shape, engine):
    n, t, k, p = shape
    k = min(k, n, t)
    for seed, dup, f32 in ((n * t, False, True), (n * t + 1, True, False)):
        d, ys = _problem(n, t, k, p, seed, dup)
        if f32:
            ys = ys.astype(np.float32).astype(np.float64)
        eps = 1e-3 * np.linalg.norm(ys, axis=1)
        ref = _oracle(d, ys, k, eps)
        dd = D.DeviceDictionary(d)
        got = D.omp_batch_raw(dd, ys.astype(np.float32) if f32 else ys, p, k, eps, None, engine)
        _check(ref, got, d, ys, eps, engine)


@pytest.mark.parametrize("shape", SHAPES[1:6])
@pytest.mark.parametrize("engine", ["exact", "gram", "resident", "auto"])
def test_random_blocked(shape, engine):
    n, t, k, p = shape
    q = 4
    t = (t // q) * q
    nb = 3
    d, ys = _problem(n, t, k, p, n + t, False)
    rng = np.random.default_rng(t)
    blocks = np.sort(np.stack([rng.choice(t // q, size=nb, replace=False) for _ in range(p)]), 1)
    allowed = (blocks[:, :, None] * q + np.arange(q)[None, None, :]).reshape(p, -1)
    k_max = min(k, nb * q, n)
    eps = 1e-3 * np.linalg.norm(ys, axis=1)
    ref = _oracle(d, ys, k_max, eps, allowed)
    dd = D.DeviceDictionary(d)
    got = D.omp_batch_blocked_raw(dd, ys, p, k_max, eps, np.ascontiguousarray(blocks), q, engine)
    _check(ref, got, d, ys, eps, engine, allowed)


def _clustered(n, t, k, p, seed, nc=12, spread=3e-4):
    """Five clusters of `nc` atoms within `spread` of one direction: whenever a
    cluster leads the scan more than 8 candidates sit inside the certification
    window of the fp16 scan, so the pick cannot be certified from the top-8 list."""
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((t, n))
    heads = np.arange(0, 5 * nc, nc)
    for c in heads:
        d[c + 1:c + nc] = d[c] + spread * np.linalg.norm(d[c]) / np.sqrt(n) * \
            rng.standard_normal((nc - 1, n))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    x = np.zeros((p, t))
    for i in range(p):
        sup = rng.choice(np.arange(5 * nc, t), size=min(k, t) - 1, replace=False)
        x[i, sup] = rng.standard_normal(sup.size)
        x[i, rng.choice(heads) + rng.integers(nc)] = 3.0 * (1 if rng.random() < 0.5 else -1)
    ys = x @ d + 0.01 * rng.standard_normal((p, n))
    return d, ys


def test_tiled_rescan_matches_oracle(monkeypatch):
    """The tensor engine's tiled fp64 rescan (the large-dictionary path),
    forced on shapes whose fp16 scans leave picks uncertified (clusters of
    more than 8 nearly parallel atoms) and on noisy near-tie problems."""
    from paper_1511_05174_b200 import _native as N
    monkeypatch.setenv("CDB_RESCAN", "tile")
    rescans = 0
    for n, t, k, p in ((129, 513, 16, 160), (256, 1000, 20, 200), (70, 300, 10, 130)):
        d, ys = _clustered(n, t, k, p, n + t + 5)
        eps = 1e-4 * np.linalg.norm(ys, axis=1)
        ref = _oracle(d, ys, k, eps)
        got = D.omp_batch_raw(D.DeviceDictionary(d), ys, p, k, eps, None, "tensor")
        rescans += N.last_run_info()[2]
        _check(ref, got, d, ys, eps, "tensor")
        d, ys = _problem(n, t, k, p, n + t + 5, True)
        ys += 0.2 * np.random.default_rng(n).standard_normal(ys.shape)  # noisy: near ties
        eps = 1e-4 * np.linalg.norm(ys, axis=1)
        ref = _oracle(d, ys, k, eps)
        got = D.omp_batch_raw(D.DeviceDictionary(d), ys, p, k, eps, None, "tensor")
        _check(ref, got, d, ys, eps, "tensor")
    assert rescans > 0


def test_grouped_rescan_matches_oracle(monkeypatch):
    """The grouped exact rescan (small dictionaries) on the clustered problems."""
    from paper_1511_05174_b200 import _native as N
    monkeypatch.setenv("CDB_RESCAN", "group")
    rescans = 0
    for n, t, k, p in ((64, 256, 8, 150), (129, 513, 16, 100)):
        d, ys = _clustered(n, t, k, p, n + t + 9)
        eps = 1e-4 * np.linalg.norm(ys, axis=1)
        ref = _oracle(d, ys, k, eps)
        got = D.omp_batch_raw(D.DeviceDictionary(d), ys, p, k, eps, None, "tensor")
        rescans += N.last_run_info()[2]
        _check(ref, got, d, ys, eps, "tensor")
    assert rescans > 0


def test_split_residual_matches_oracle(monkeypatch):
    """The tensor engine's split-mode scan operand (resid_split_kernel, the
    large-N path), forced on shapes below its default threshold."""
    monkeypatch.setenv("CDB_LS_SPLIT", "1")
    for n, t, k, p in ((129, 513, 16, 96), (256, 1000, 20, 64), (33, 64, 12, 64)):
        d, ys = _problem(n, t, k, p, n * t + 3, False)
        eps = 1e-3 * np.linalg.norm(ys, axis=1)
        ref = _oracle(d, ys, k, eps)
        got = D.omp_batch_raw(D.DeviceDictionary(d), ys, p, k, eps, None, "tensor")
        _check(ref, got, d, ys, eps, "tensor")


@pytest.mark.parametrize("nb,q,k", [(15, 12, 14), (28, 12, 20), (9, 20, 12)])
def test_gram_candidate_widths(nb, q, k):
    """Block-restricted sets whose width lands on the Gram engine's U = 6 and
    U = 12 H layouts (S in (128, 192] and (256, 384]) and U = 8 (S = 180)."""
    n, p = 64, 40
    t = 40 * q
    d, ys = _problem(n, t, k, p, nb * q + k, False)
    rng = np.random.default_rng(nb)
    blocks = np.sort(np.stack([rng.choice(t // q, size=nb, replace=False) for _ in range(p)]), 1)
    allowed = (blocks[:, :, None] * q + np.arange(q)[None, None, :]).reshape(p, -1)
    k_max = min(k, nb * q, n)
    eps = 1e-3 * np.linalg.norm(ys, axis=1)
    ref = _oracle(d, ys, k_max, eps, allowed)
    got = D.omp_batch_blocked_raw(D.DeviceDictionary(d), ys, p, k_max, eps,
                                  np.ascontiguousarray(blocks), q, "gram")
    _check(ref, got, d, ys, eps, "gram", allowed)


@pytest.mark.parametrize("n,k", [(320, 7), (1024, 12), (2048, 24), (1000, 32)])
def test_short_supports_on_long_rows(n, k):
    """N > 256 with K <= 32: the warp-per-signal least-squares kernel with one
    support entry per lane (ls_wide_kernel, KR = 1) and the separate scan-operand
    kernels (fp32 N = 1024, bulk-copy ring N = 2048, generic otherwise)."""
    t, p = 300, 80
    d, ys = _problem(n, t, k, p, 11 * n + k, n == 320)
    eps = 1e-3 * np.linalg.norm(ys, axis=1)
    ref = _oracle(d, ys, k, eps)
    dd = D.DeviceDictionary(d)
    got = D.omp_batch_raw(dd, ys, p, k, eps, None, "tensor")
    _check(ref, got, d, ys, eps, "tensor")


@pytest.mark.parametrize("n,f32", [(2048, True), (3072, False), (4096, True), (4096, False)])
def test_long_row_scan_operand(n, f32):
    """Tensor engine on long rows (N = 1024 J up to 4096): the next scan's
    operand r~ = y - D32_S x comes from the bulk-copy ring kernel
    (resid_bulk_kernel, J = 2, 3, 4; fp32 and fp64 signals), supports up to K = 40
    so the producer's ring wraps several times per signal."""
    t, k, p = 384, 40, 96
    d, ys = _problem(n, t, k, p, 7 * n + f32, False)
    ys[1] = d[5] * 2.0  # one-atom signal: stops after a pick or two
    if f32:
        ys = ys.astype(np.float32).astype(np.float64)
    eps = 1e-3 * np.linalg.norm(ys, axis=1)
    ref = _oracle(d, ys, k, eps)
    dd = D.DeviceDictionary(d)
    got = D.omp_batch_raw(dd, ys.astype(np.float32) if f32 else ys, p, k, eps, None, "tensor")
    _check(ref, got, d, ys, eps, "tensor")


def test_bulk_ring_two_kilobyte_rows_hbm_dictionary():
    """N = 2048 takes the bulk-copy ring (J = 2) only when the fp32 dictionary
    is larger than L2 (12,288 atoms: 101 MB)."""
    n, t, k, p = 2048, 12288, 12, 32
    d, ys = _problem(n, t, k, p, 2048, False)
    ys = ys.astype(np.float32).astype(np.float64)
    eps = 1e-3 * np.linalg.norm(ys, axis=1)
    ref = _oracle(d, ys, k, eps)
    dd = D.DeviceDictionary(d)
    got = D.omp_batch_raw(dd, ys.astype(np.float32), p, k, eps, None, "tensor")
    _check(ref, got, d, ys, eps, "tensor")
    dd.close()
