"""BASELINE configs at their FULL sizes, checked through size-independent
properties (the CPU oracle cannot run them whole): zero-tree nesting, the
reference's scan-count formula (pursuit.py:18-20), the stop rule, residual
consistency and least-squares optimality on samples, and the parity contract
against the oracle on a seeded random subset."""

import numpy as np
import pytest
import torch

from parity import compare

import oracle as O
from paper_1511_05174_b200 import device as D
from paper_1511_05174_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _host(o):
    return {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in o.items()}


def _scan_formula(t, counts):
    c = counts.astype(np.int64)
    return t * c - c * (c - 1) // 2


def _check_ls(mat_t, ys, sol, eps, idx):
    for p in idx:
        c = int(sol["counts"][p])
        if c == 0:
            assert sol["rnorm"][p] == pytest.approx(np.linalg.norm(ys[p]), rel=1e-12)
            continue
        A = mat_t[sol["sel"][p, :c]].T
        r = ys[p] - A @ sol["alpha"][p, :c]
        assert abs(np.linalg.norm(r) - sol["rnorm"][p]) <= 1e-9 * np.linalg.norm(ys[p])
        # least-squares optimality: residual orthogonal to the support
        assert np.abs(A.T @ r).max() <= 1e-9 * np.linalg.norm(ys[p])


def _check_stop(sol, eps, budget):
    c = sol["counts"]
    stopped = (sol["rnorm"] <= eps * (1 + 1e-9)) | (c == budget)
    assert stopped.mean() > 0.9999


@pytest.mark.parametrize("ci", [0, 1])
def test_zero_tree_full_size(ci):
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    P = w.signals
    ys = W.signals(ci, 0, P)
    low, high, _ = D.zero_tree_raw(D.device_dictionary(d.low_t), D.device_dictionary(d.high_t),
                                   w.fine_shape, w.factors, ys.astype(np.float32), P, w.k, w.k,
                                   W.REL_TOL, False, "auto")
    # nesting (crossscale.py:224): every fine atom is a child of a coarse pick
    for p in range(P):
        cl, ch = int(low["counts"][p]), int(high["counts"][p])
        parents = set(low["sel"][p, :cl].tolist())
        assert all(int(j) // w.q in parents for j in high["sel"][p, :ch])
    # scan counts: step 1 scans T_low per pick, step 2 scans nb*Q candidates
    assert np.array_equal(low["scans"], _scan_formula(w.t_low, low["counts"]))
    nbq = low["counts"].astype(np.int64) * w.q
    c2 = high["counts"].astype(np.int64)
    assert np.array_equal(high["scans"], nbq * c2 - c2 * (c2 - 1) // 2)
    eps2 = W.REL_TOL * np.linalg.norm(ys, axis=1)
    _check_stop(high, eps2, np.minimum(w.k, nbq))
    rng = np.random.default_rng(ci)
    idx = rng.choice(P, size=256, replace=False)
    _check_ls(d.high_t, ys, high, eps2, idx)
    # parity contract vs the oracle on the random subset
    rl, rh = O.zero_tree_many_arrays(d.low_t, d.high_t, w.fine_shape, w.factors, w.k, w.k,
                                     ys[idx], rel_tol=W.REL_TOL, nthreads=8)
    sub = {k: v[idx] for k, v in high.items()}
    sub["flag"] = sub["flag"].astype(bool)
    same1 = np.array([np.array_equal(low["sel"][p], rl["sel"][i]) for i, p in enumerate(idx)])
    assert same1.mean() > 0.99
    agree = np.mean([np.array_equal(sub["sel"][i], rh["sel"][i]) for i in range(len(idx))])
    assert agree > 0.98


@pytest.mark.parametrize("ci", [0, 1])
def test_full_omp_full_size(ci):
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    P = w.signals
    ys = W.signals(ci, 0, P)
    eps = W.REL_TOL * np.linalg.norm(ys, axis=1)
    sol = D.omp_batch_raw(D.device_dictionary(d.high_t), ys.astype(np.float32), P, w.k, eps, None,
                          "auto")
    assert np.array_equal(sol["scans"], _scan_formula(w.t_high, sol["counts"]))
    _check_stop(sol, eps, w.k)
    rng = np.random.default_rng(10 + ci)
    idx = rng.choice(P, size=256, replace=False)
    _check_ls(d.high_t, ys, sol, eps, idx)
    ref = O.omp_many_arrays(d.high_t, ys[idx], w.k, rel_tol=W.REL_TOL, nthreads=8)
    got = {k: v[idx] for k, v in sol.items()}
    got["flag"] = got["flag"].astype(bool)
    rep = compare(ref, got, d.high_t, ys[idx], eps[idx])
    assert not rep["bad"], rep["bad"][:3]


def test_device_resident_inputs_match_host_inputs():
    # the same batch through device tensors (bench `value` path) and host
    # arrays (bench `e2e` path) gives identical results
    ci = 1
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    ys = W.signals(ci, 0, 4096).astype(np.float32)
    lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
    a_low, a_high, _ = D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, ys, len(ys), w.k, w.k,
                                       W.REL_TOL, False, "auto")
    yd = torch.from_numpy(ys).cuda()
    mk = lambda k: dict(sel=torch.empty((len(ys), k), dtype=torch.int64, device="cuda"),
                        alpha=torch.empty((len(ys), k), dtype=torch.float64, device="cuda"),
                        counts=torch.empty(len(ys), dtype=torch.int64, device="cuda"),
                        rnorm=torch.empty(len(ys), dtype=torch.float64, device="cuda"),
                        scans=torch.empty(len(ys), dtype=torch.int64, device="cuda"),
                        flag=torch.empty(len(ys), dtype=torch.uint8, device="cuda"))
    ol, oh = mk(w.k), mk(w.k)
    D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, len(ys), w.k, w.k, W.REL_TOL, False,
                    "auto", ol, oh)
    ol, oh = _host(ol), _host(oh)
    for k in ("sel", "counts", "scans"):
        assert np.array_equal(ol[k], a_low[k]) and np.array_equal(oh[k], a_high[k])
    assert np.array_equal(oh["alpha"], a_high["alpha"])


@pytest.mark.parametrize("kind", ["zt", "full"])
def test_pipelined_host_buffers_match_device_buffers(kind):
    # >= 32768 signals with host buffers take the chunked copy/compute pipeline
    ci = 1
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    P = 70_000
    ys = W.signals(ci, 0, P).astype(np.float32)
    lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
    yd = torch.from_numpy(ys).cuda()
    mk = lambda k: dict(sel=torch.empty((P, k), dtype=torch.int64, device="cuda"),
                        alpha=torch.empty((P, k), dtype=torch.float64, device="cuda"),
                        counts=torch.empty(P, dtype=torch.int64, device="cuda"),
                        rnorm=torch.empty(P, dtype=torch.float64, device="cuda"),
                        scans=torch.empty(P, dtype=torch.int64, device="cuda"),
                        flag=torch.empty(P, dtype=torch.uint8, device="cuda"))
    if kind == "zt":
        h_low, h_high, ms_h = D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, ys, P, w.k, w.k,
                                              W.REL_TOL, False, "auto")
        d_low, d_high = mk(w.k), mk(w.k)
        D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, P, w.k, w.k, W.REL_TOL, False, "auto",
                        d_low, d_high)
        pairs = [(h_low, _host(d_low)), (h_high, _host(d_high))]
        assert ms_h[0] > 0 and ms_h[1] > 0
    else:
        eps = W.REL_TOL * np.linalg.norm(ys.astype(np.float64), axis=1)
        h = D.omp_batch_raw(hi, ys, P, w.k, eps, None, "auto")
        dd = mk(w.k)
        D.omp_batch_raw(hi, yd, P, w.k, torch.from_numpy(eps).cuda(), None, "auto", dd)
        pairs = [(h, _host(dd))]
    for a, b in pairs:
        for k in ("sel", "counts", "scans", "alpha", "rnorm"):
            assert np.array_equal(a[k], b[k]), k
