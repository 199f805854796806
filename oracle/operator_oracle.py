"""CPU restatement of crossdict's operator recovery --
TEST INFRASTRUCTURE ONLY (imported by tests/ to check the device path; never
by the product package).

Per patch, as the reference does it:

* patch_problem    sensing.py:205-279: the patch window of the measurement
  and the patch-local operator (mask: kept cells ascending; channel mosaic:
  pixel s reads s*C + a_s - 1; temporal code: pixel s sums the frames coded
  1; angular: spatial s, kept view v -> s*V + v - 1).
* apply_matrix     sensing.py:78-92: gather rows, or the frame-axis sum of
  (cols.reshape(S, F, T) * code), called on the same column layouts as the
  reference (C-contiguous atoms: numpy sums f sequentially; step 2's
  atoms_t[allowed0].T: f is contiguous and numpy sums it pairwise).
* _recover_operator pipelines.py:258-322: DC removal for masks (numpy mean),
  omp(eff, y, min(k, m)) for "omp-single"; for "zerotree" zero_tree_omp's Phi
  branch crossscale.py:194-222 (step 1 on phi U D_low, budget
  min(k_low, m, T_low); step 2 local OMP over phi D_high[:, allowed0],
  budget min(k_high, |allowed0|, m), localised; empty step 1 -> rnorm
  ||y||, flagged), reconstruction atoms @ coef + dc, aggregate_patches.

The OMP itself is the C kernel restatement (oracle.omp_batch).  Pinned
against the reference's own outputs in tests/golden/operator_*.npz
(tests/golden/make_golden_operators.py).
"""

from __future__ import annotations

import numpy as np

import oracle as O
import patch_oracle as PO


def _local_ops(kind, op, sig_shape, patch, origin, meas):
    """(gather or None, code or None, y) of one patch (sensing.py:205-279)."""
    win = tuple(slice(o, o + e) for o, e in zip(origin, patch))
    if kind == "mask":
        local = op["known"][win].ravel()
        kept0 = np.flatnonzero(local)
        if kept0.size == 0:
            return None, None, None
        return kept0, None, meas[win].ravel()[kept0]
    if kind == "channel-mosaic":
        c = int(op["channels"])
        a = op["assignment"].reshape(sig_shape[:-1])[win[:-1]].ravel()
        return np.arange(a.size) * c + (a - 1), None, meas[win[:-1]].ravel().copy()
    if kind == "temporal-code":
        f = int(op["frames"])
        code = op["code"].reshape(sig_shape[:-1] + (f,))[win[:-1]].reshape(-1, f)
        if (code.sum(axis=1) == 1).all():
            g = np.arange(code.shape[0]) * f + np.argmax(code, axis=1)
            return g, None, meas[win[:-1]].ravel().copy()
        return None, code, meas[win[:-1]].ravel().copy()
    if kind == "angular-sample":
        vr, vc = (int(v) for v in op["view_grid"])
        kept = np.asarray(op["kept"])
        ns = int(np.prod(patch[:-2]))
        g = (np.arange(ns)[:, None] * (vr * vc) + (kept - 1)[None, :]).ravel()
        return g, None, meas[win[:-2]].reshape(ns, kept.size).ravel().copy()
    raise ValueError(kind)


def _apply(gather, code, cols):
    if gather is not None:
        return cols[gather]
    s, f = code.shape
    return (cols.reshape(s, f, -1) * code[:, :, None]).sum(axis=1)


def _omp(eff, y, k, rel):
    eps = np.array([rel * float(np.linalg.norm(y))])
    sel, coef, cnt, rn, sc, fl = O.omp_batch(np.ascontiguousarray(eff.T), y[None, :], k, eps)
    c = int(cnt[0])
    return sel[0, :c], coef[0, :c], float(rn[0]), int(sc[0])


def _upsample(d_low, fine, factors):
    coarse = tuple(e // f for e, f in zip(fine, factors))
    t = d_low.shape[1]
    st = d_low.T.reshape((t,) + coarse)
    for ax, f in enumerate(factors):
        if f > 1:
            st = np.repeat(st, f, axis=ax + 1)
    return np.ascontiguousarray(st.reshape(t, -1).T)


def recover(g, rel=1e-6):
    """Restated recover() on one golden case (the npz fields)."""
    kind = str(g["kind"])
    sig_shape = tuple(int(e) for e in g["sig_shape"])
    patch = tuple(int(e) for e in g["patch"])
    stride = tuple(int(e) for e in g["stride"])
    meas = np.asarray(g["meas"], dtype=np.float64)
    op = {k: g[k] for k in ("known", "assignment", "channels", "code", "frames", "view_grid",
                            "kept") if k in g}
    method = str(g["method"])
    _, origins, _ = PO.extract_patches(np.zeros(sig_shape), patch, stride)
    p = len(origins)
    n = int(np.prod(patch))
    remove_dc = kind == "mask"
    if method == "zerotree":
        d_high = np.asarray(g["d_high"])
        ud = _upsample(np.asarray(g["d_low"]), patch, tuple(int(f) for f in g["factors"]))
        k_low, k_high = int(g["k_low"]), int(g["k_high"])
        q = d_high.shape[1] // ud.shape[1]
        atoms = d_high
    else:
        atoms = np.asarray(g["atoms"])
        k = min(int(g["k"]), atoms.shape[1])
    est_cols = np.zeros((n, p))
    resid = np.zeros(p)
    flagged = scans1 = scans2 = 0
    for i, o in enumerate(origins):
        gather, code, y = _local_ops(kind, op, sig_shape, patch, o, meas)
        if y is None or y.size == 0:
            flagged += 1
            continue
        dc = 0.0
        if remove_dc:
            dc = float(y.mean())
            y = y - dc
        m = y.size
        if method == "omp-single":
            sel, coef, rn, sc = _omp(_apply(gather, code, atoms), y, min(k, m), rel)
            scans1 += sc
        else:
            s1, _, rn1, sc1 = _omp(_apply(gather, code, ud), y, min(k_low, m, ud.shape[1]), rel)
            scans1 += sc1
            if s1.size == 0:
                flagged += int(np.linalg.norm(y) > 0)
                resid[i] = float(np.linalg.norm(y))
                est_cols[:, i] = dc
                continue
            allowed0 = (np.sort(s1)[:, None] * q + np.arange(q)[None, :]).ravel()
            cols2 = np.ascontiguousarray(atoms.T)[allowed0].T  # atoms_t[allowed0].T, F layout
            loc, coef, rn, sc = _omp(_apply(gather, code, cols2), y,
                                     min(k_high, allowed0.size, m), rel)
            sel = allowed0[loc]
            scans2 += sc
        resid[i] = rn
        est_cols[:, i] = PO.reconstruct(atoms, sel[None, :], coef[None, :])[:, 0] + dc
    est, _ = PO.aggregate_patches(est_cols, origins, sig_shape, patch)
    return dict(estimate=est, resid=resid, flagged=flagged, scans1=scans1, scans2=scans2)
