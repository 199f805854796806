"""The parity contract of BASELINE.json ``north_star``, as executable checks.

Supports must equal the oracle's (in pick order) except where the oracle's
top-two relative |correlation| gap at that pick is below ``GAP`` (1e-6):
from such a pick on, the rest of that signal is excused.  Coefficients must
match within ``COEF_RTOL`` (1e-4) relative; counts and scan counts must
match except in the stop-test band, where the oracle's final residual norm
is within ``STOP_BAND`` (1e-5) relative of the tolerance.

The gaps are recomputed by replaying the oracle's pick sequence in fp64
(exact least squares at every step) -- test infrastructure, numpy only.
"""

from __future__ import annotations

import numpy as np

GAP = 1e-6
COEF_RTOL = 1e-4
STOP_BAND = 1e-5


def replay_gaps(mat_t, y, sel, count, allowed=None):
    """Relative top-two gap of |<d_j, r>| at each oracle pick (fp64 replay)."""
    t = mat_t.shape[0]
    cand = np.arange(t) if allowed is None else np.asarray(allowed)
    gaps = np.full(int(count), np.inf)
    r = y.copy()
    chosen = []
    for k in range(int(count)):
        live = np.array([c for c in cand if c not in chosen], dtype=np.int64)
        v = np.abs(mat_t[live] @ r)
        if v.size >= 2:
            top = np.sort(v)[-2:]
            gaps[k] = (top[1] - top[0]) / top[1] if top[1] > 0 else 0.0
        chosen.append(int(sel[k]))
        a = mat_t[chosen].T
        coef = np.linalg.lstsq(a, y, rcond=None)[0]
        r = y - a @ coef
    return gaps


def compare(ref, got, mat_t, ys_rows, eps, allowed_rows=None, check_scans=True, coef_rtol=COEF_RTOL):
    """Return a report dict; ``report['bad']`` lists signals violating the contract."""
    p_all = ys_rows.shape[0]
    bad, excused_gap, excused_stop, exact = [], 0, 0, 0
    for p in range(p_all):
        c_ref, c_got = int(ref["counts"][p]), int(got["counts"][p])
        s_ref, s_got = ref["sel"][p, :c_ref], got["sel"][p, :c_got]
        same = c_ref == c_got and np.array_equal(s_ref, s_got)
        if same and bool(ref["flag"][p]):
            # dense minimum-norm mode: the reference calls LAPACK, values are
            # "parity unpinned" -- support, flag, finiteness and a residual no
            # larger than the reference's (to rounding) are required
            ok = (bool(got["flag"][p]) and np.isfinite(got["alpha"][p, :c_got]).all()
                  and got["rnorm"][p] <= ref["rnorm"][p] + 1e-9 * np.linalg.norm(ys_rows[p]))
            if ok:
                exact += 1
            else:
                bad.append((p, "dense-mode", {}))
            continue
        if same:
            a_ref, a_got = ref["alpha"][p, :c_ref], got["alpha"][p, :c_got]
            scale = np.abs(a_ref).max() if c_ref else 0.0
            ok_coef = np.all(np.abs(a_got - a_ref) <= coef_rtol * np.abs(a_ref) + 1e-9 * scale)
            ok_rn = abs(got["rnorm"][p] - ref["rnorm"][p]) <= 1e-6 * max(ref["rnorm"][p], 1e-300) + 1e-12
            ok_scan = (not check_scans) or int(ref["scans"][p]) == int(got["scans"][p])
            ok_flag = bool(ref["flag"][p]) == bool(got["flag"][p])
            if ok_coef and ok_rn and ok_scan and ok_flag:
                exact += 1
                continue
            bad.append((p, "values", dict(coef=ok_coef, rnorm=ok_rn, scans=ok_scan, flag=ok_flag)))
            continue
        # first divergence
        m = min(c_ref, c_got)
        div = next((i for i in range(m) if s_ref[i] != s_got[i]), m)
        allowed = None if allowed_rows is None else allowed_rows[p]
        gaps = replay_gaps(mat_t, ys_rows[p], s_ref, c_ref, allowed)
        if div < c_ref and gaps[div] < GAP:
            excused_gap += 1
            continue
        tol = eps[p]
        if tol > 0 and abs(ref["rnorm"][p] - tol) <= STOP_BAND * tol:
            excused_stop += 1
            continue
        if div == m and tol > 0:
            # one run stopped a pick earlier: stop-test band on the shorter run
            rn_short = got["rnorm"][p] if c_got < c_ref else ref["rnorm"][p]
            if abs(rn_short - tol) <= STOP_BAND * tol:
                excused_stop += 1
                continue
        bad.append((p, "support", dict(div=div, gap=float(gaps[div]) if div < c_ref else None,
                                       ref=s_ref.tolist(), got=s_got.tolist())))
    return dict(bad=bad, exact=exact, excused_gap=excused_gap, excused_stop=excused_stop, n=p_all)


def batch_dict(s):
    """BatchSolve-like object or dict -> dict of arrays with a per-signal flag."""
    if isinstance(s, dict):
        return s
    flag = np.zeros(len(s.counts), bool)
    for i in s.rank_deficient:
        flag[i] = True
    return dict(counts=s.counts, sel=s.sel, alpha=s.alpha, rnorm=s.rnorm, scans=s.scans, flag=flag)


def golden_dict(g, prefix=""):
    p = len(g[prefix + "counts"])
    flag = np.zeros(p, bool)
    flag[g[prefix + "flag"]] = True
    return dict(counts=g[prefix + "counts"], sel=g[prefix + "sel"], alpha=g[prefix + "alpha"],
                rnorm=g[prefix + "rnorm"], scans=g[prefix + "scans"], flag=flag)


def check_zero_tree(d_low_t, d_high_t, q, ys, low, high, rl, rh, yl=None, min_same=0.9):
    """The contract on a zero-tree batch: step 1 against the oracle's step 1
    (eps = 1e-3 |W y|), step 2 on the signals whose step-1 support equals the
    oracle's (their candidate sets are then identical; allowed = the oracle's
    sorted blocks x Q), and the nesting invariant (crossscale.py:224).
    ``low``/``high`` hold the device outputs of exactly these signals."""
    p = ys.shape[0]
    y1 = yl if yl is not None else ys
    eps1 = 1e-3 * np.linalg.norm(y1, axis=1)
    rep1 = compare(rl, low, d_low_t, y1, eps1)
    assert not rep1["bad"], ("step1", rep1["bad"][:3])
    same = np.array([np.array_equal(low["sel"][i], rl["sel"][i]) for i in range(p)])
    assert same.mean() >= min_same, same.mean()  # enough signals for a step-2 check
    idx = np.flatnonzero(same)
    eps2 = 1e-3 * np.linalg.norm(ys, axis=1)
    allowed = []
    for i in idx:
        c = int(rl["counts"][i])
        b = np.sort(rl["sel"][i, :c])
        allowed.append((b[:, None] * q + np.arange(q)[None, :]).ravel())

    def sub(o):
        return {k: np.asarray(v)[idx] for k, v in o.items() if np.ndim(v) >= 1 and len(v) == p}

    rep2 = compare(sub(rh), sub(high), d_high_t, ys[idx], eps2[idx], allowed if idx.size else None)
    assert not rep2["bad"], ("step2", rep2["bad"][:3])
    for i in range(p):
        parents = set(np.asarray(low["sel"][i, :int(low["counts"][i])]).tolist())
        assert all(int(j) // q in parents for j in high["sel"][i, :int(high["counts"][i])])
    return rep1, rep2
