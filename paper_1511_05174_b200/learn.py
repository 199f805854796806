"""K-SVD on the device: the coding stage -- mirror of
crossdict ``learn._code_stage`` (learn.py:240-262), the call K-SVD training
makes every iteration with the dictionary it is refitting -- and the
dictionary-update stage, ``learn._update_stage`` (learn.py:169-199).

The reference groups the samples by their block count and issues one
block-restricted ``omp_many`` per group, because its kernel takes rectangular
``allowed_blocks``; here one ragged device call codes every sample
(``cdb_omp_batch_blocked_ragged``: per-sample block count, budget
min(k, nb * Q, N) -- the per-group rule of pursuit.py:423).  Results are the
reference's per-sample ``PursuitResult`` list in sample order.  ``install()``
binds this function as ``crossdict.learn._code_stage``.

``update_stage`` runs the sequential rank-one refits in one device call
(``cdb_ksvd_update``, csrc/ksvd_engine.cu) and is bound as
``crossdict.learn._update_stage``.
"""

from __future__ import annotations

import numpy as np

from . import _native as _N
from . import device as _dev
from . import pursuit as _pursuit
from .pursuit import PursuitConfig


def code_stage(d, y, k, allowed_sets, block_hint):
    """Sparse-code every column of ``y`` against ``d`` (learn.py:240-262)."""
    d = np.asarray(d, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    m = y.shape[1]
    if allowed_sets is None:
        return _pursuit.omp_many(d, y, PursuitConfig(k))
    if block_hint is not None:
        blocks_list, q = block_hint
        n, t = d.shape
        nb = np.array([len(b) for b in blocks_list], dtype=np.int64)
        nb_max = max(1, int(nb.max()) if m else 1)
        blocks = np.zeros((m, nb_max), dtype=np.int64)
        for p, b in enumerate(blocks_list):
            if len(b):
                blocks[p, :len(b)] = sorted(b)
        k_out = int(max(1, min(k, nb_max * q, n)))
        if m == 0:
            return []
        ys_rows = _dev.rows_for_device(y)
        cfg = PursuitConfig(k)
        if cfg.residual_tolerance is not None:
            eps = np.full(m, float(cfg.residual_tolerance))
        else:
            eps = _pursuit._rel_tol() * np.sqrt(np.einsum("pn,pn->p", ys_rows, ys_rows))
        dd = _dev.device_dictionary(np.ascontiguousarray(d.T))
        o = _dev.omp_batch_blocked_ragged_raw(dd, ys_rows, m, k_out, eps, blocks, nb, int(q),
                                              _pursuit.ENGINE)
        solve = _pursuit._make_batch(t, o)
        return [solve.result(p) for p in range(m)]
    return [
        _pursuit.omp(d, y[:, p], PursuitConfig(min(k, len(allowed_sets[p])),
                                               allowed_support=frozenset(allowed_sets[p])))
        for p in range(m)
    ]


def update_stage(y, d, x, threshold: int):
    """Sequential rank-one atom refits (learn.py:169-199): updates ``d``
    (N x T) and ``x`` (T x M, dense) in place and returns ``(replaced, e)``
    with e = Y - D X after the refits.

    E starts as the reference's own product ``y - d @ x``; the per-atom loop
    runs on the device.  Atom signs follow the largest-magnitude-entry-
    positive convention (the reference's LAPACK SVD sign is arbitrary;
    products d_j x_j and E do not depend on it)."""
    y = np.asarray(y, dtype=np.float64)
    n, m = y.shape
    t = d.shape[1]
    e = y - d @ x
    jj, pp = np.nonzero(x)  # by atom, then ascending signal: np.flatnonzero(x[j])
    vals = np.ascontiguousarray(x[jj, pp], dtype=np.float64)
    counts = np.bincount(jj, minlength=t)
    ptr = np.zeros(t + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    sig = np.ascontiguousarray(pp, dtype=np.int64)
    y_rows = np.ascontiguousarray(y.T)
    e_rows = np.ascontiguousarray(e.T)
    d_rows = np.ascontiguousarray(np.asarray(d, dtype=np.float64).T)
    replaced = np.zeros(1, dtype=np.int64)
    _N.check(_N.load().cdb_ksvd_update(n, m, t, _N.ptr(y_rows), _N.ptr(e_rows), _N.ptr(d_rows),
                                       _N.ptr(ptr), _N.ptr(sig), _N.ptr(vals), int(vals.size),
                                       int(counts.max()) if t else 0, int(threshold),
                                       _N.ptr(replaced), None))
    d[...] = d_rows.T
    x[jj, pp] = vals
    return int(replaced[0]), np.ascontiguousarray(e_rows.T)
