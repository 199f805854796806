"""CPU oracle for batched OMP / zero-tree OMP -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker or as the timed CPU baseline.  The product package never
imports it.

Layout: the per-signal kernel is the C restatement in ``omp_oracle.c``
(``_kernels.py:50-168``); this file restates the numpy orchestration around
it, citing the reference line it follows:

* ``omp_many_arrays``   -> ``pursuit.py:388-441`` (+ ``_run_kernel`` 234-250)
* ``downsample_columns``-> ``scaling.py:99-116``
* ``zero_tree_many_arrays`` -> ``crossscale.py:235-283``
* ``zero_tree_phi_many``    -> ``crossscale.py:169-232`` (Phi branch), batched on
  precomputed effective dictionaries as BASELINE.md §2 prescribes.

Parity pin: ``tests/test_oracle.py`` checks these functions against the
golden vectors in ``tests/golden/`` produced by running the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile the C oracle (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        _lib.oracle_omp_batch.argtypes = [p, i64, i64, p, i64, i64, p, p, i64, ctypes.c_int,
                                          p, p, p, p, p, p, ctypes.c_int]
        _lib.oracle_omp_batch.restype = ctypes.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def omp_batch(mat_t, ys_rows, k_max, eps, allowed=None, nthreads=1):
    """The reference kernel call (``pursuit._run_kernel``, ``pursuit.py:234-250``)."""
    mat_t = np.ascontiguousarray(mat_t, dtype=np.float64)
    ys_rows = np.ascontiguousarray(ys_rows, dtype=np.float64)
    eps = np.ascontiguousarray(eps, dtype=np.float64)
    p_all, n = ys_rows.shape
    t = mat_t.shape[0]
    restricted = allowed is not None
    if restricted:
        allowed = np.ascontiguousarray(allowed, dtype=np.int64)
        s = allowed.shape[1]
    else:
        allowed = np.zeros((max(p_all, 1), 1), dtype=np.int64)
        s = 1
    out_sel = np.full((p_all, k_max), -1, dtype=np.int64)
    out_coef = np.zeros((p_all, k_max))
    out_count = np.zeros(p_all, dtype=np.int64)
    out_rnorm = np.zeros(p_all)
    out_scans = np.zeros(p_all, dtype=np.int64)
    out_flag = np.zeros(p_all, dtype=np.uint8)
    if p_all:
        rc = lib().oracle_omp_batch(_ptr(mat_t), t, n, _ptr(ys_rows), p_all, k_max, _ptr(eps),
                                    _ptr(allowed), s, int(restricted), _ptr(out_sel),
                                    _ptr(out_coef), _ptr(out_count), _ptr(out_rnorm),
                                    _ptr(out_scans), _ptr(out_flag), int(nthreads))
        if rc != 0:
            raise MemoryError("oracle workspace allocation failed")
    return out_sel, out_coef, out_count, out_rnorm, out_scans, out_flag.astype(bool)


def omp_many_arrays(mat_t, ys_rows, k, *, rel_tol=1e-6, residual_tolerance=None,
                    allowed_blocks=None, block_q=None, nthreads=1):
    """``pursuit.omp_many_arrays`` (``pursuit.py:388-441``) without validation.

    ``mat_t`` is T x N (atoms as rows), ``ys_rows`` P x N (signals as rows).
    Returns a dict with the BatchSolve arrays.
    """
    t, n = mat_t.shape
    p_all = ys_rows.shape[0]
    allowed = None
    if allowed_blocks is not None:
        blocks = np.asarray(allowed_blocks, dtype=np.int64)
        allowed = (blocks[:, :, None] * block_q
                   + np.arange(block_q, dtype=np.int64)[None, None, :]).reshape(p_all, -1)
        k_max = min(k, allowed.shape[1], n)
    else:
        k_max = k
    if residual_tolerance is not None:
        eps = np.full(p_all, float(residual_tolerance))
    else:
        eps = rel_tol * np.sqrt(np.einsum("pn,pn->p", ys_rows, ys_rows))
    sel, coef, count, rnorm, scans, flag = omp_batch(mat_t, ys_rows, k_max, eps, allowed, nthreads)
    return dict(counts=count, sel=sel, alpha=coef, rnorm=rnorm, scans=scans, flag=flag, dim=t)


def downsample_rows(ys_rows, fine_shape, factors):
    """Block mean of row-major fine patches (``scaling.py:99-116``).

    Signals are rows here, but the reduction is evaluated on the reference's
    own column layout and view (``cols.T.reshape(...).mean(...)``) so that the
    summation order -- hence every bit -- matches."""
    cols = np.ascontiguousarray(np.asarray(ys_rows, dtype=np.float64).T)
    p = cols.shape[1]
    coarse = tuple(e // f for e, f in zip(fine_shape, factors))
    stacked = cols.T.reshape((p,) + tuple(fine_shape))
    inter = [p]
    for c, f in zip(coarse, factors):
        inter.extend((c, f))
    view = stacked.reshape(inter)
    red = view.mean(axis=tuple(range(2, 2 * len(factors) + 1, 2)))
    return np.ascontiguousarray(red.reshape(p, -1))


def _zero_tree_step2(high_t, ys_rows, low, k_high, q, rel_tol, nthreads):
    """Group-by-coarse-count step 2 (``crossscale.py:255-279``)."""
    p_all = ys_rows.shape[0]
    counts = np.zeros(p_all, np.int64)
    sel = np.full((p_all, k_high), -1, np.int64)
    alpha = np.zeros((p_all, k_high))
    rnorm = np.zeros(p_all)
    scans = np.zeros(p_all, np.int64)
    flag = np.zeros(p_all, bool)
    for nb in np.unique(low["counts"]):
        members = np.flatnonzero(low["counts"] == nb)
        if nb == 0:
            rnorm[members] = np.linalg.norm(ys_rows[members], axis=1)
            continue
        blocks = np.sort(low["sel"][members, :nb], axis=1)
        sub = omp_many_arrays(high_t, ys_rows[members], k_high, rel_tol=rel_tol,
                              allowed_blocks=blocks, block_q=q, nthreads=nthreads)
        kw = sub["sel"].shape[1]
        counts[members] = sub["counts"]
        sel[members, :kw] = sub["sel"]
        alpha[members, :kw] = sub["alpha"]
        rnorm[members] = sub["rnorm"]
        scans[members] = sub["scans"]
        flag[members] = sub["flag"]
    return dict(counts=counts, sel=sel, alpha=alpha, rnorm=rnorm, scans=scans, flag=flag,
                dim=high_t.shape[0])


def zero_tree_many_arrays(low_t, high_t, fine_shape, factors, k_low, k_high, ys_rows,
                          *, rel_tol=1e-6, nthreads=1):
    """``crossscale.zero_tree_many_arrays`` (``crossscale.py:235-283``), identity Phi."""
    q = high_t.shape[0] // low_t.shape[0]
    yl = downsample_rows(ys_rows, fine_shape, factors)
    low = omp_many_arrays(low_t, yl, k_low, rel_tol=rel_tol, nthreads=nthreads)
    high = _zero_tree_step2(high_t, ys_rows, low, k_high, q, rel_tol, nthreads)
    return low, high


def zero_tree_phi_many(e_low_t, e_high_t, k_low, k_high, ys_rows, *, rel_tol=1e-6,
                       nthreads=1):
    """Phi-composed zero-tree (``crossscale.py:194-220``) on precomputed
    effective dictionaries: step 1 codes y against E_low = Phi U D_low with
    budget min(k_low, M, T_low); step 2 codes y against the block expansion in
    E_high = Phi D_high with budget min(k_high, nb*Q, M)."""
    m = ys_rows.shape[1]
    q = e_high_t.shape[0] // e_low_t.shape[0]
    budget1 = min(k_low, m, e_low_t.shape[0])
    low = omp_many_arrays(e_low_t, ys_rows, budget1, rel_tol=rel_tol, nthreads=nthreads)
    high = _zero_tree_step2(e_high_t, ys_rows, low, k_high, q, rel_tol, nthreads)
    return low, high
