"""CPU restatement of crossdict's K-SVD dictionary-update stage -- TEST
INFRASTRUCTURE ONLY (imported by tests/ to check the device stage; never by
the product package).

* update_stage  learn.py:169-199: e = y - d @ x; per atom j in order, users =
  flatnonzero(x[j]); fewer than `threshold` users -> fold the atom's terms
  back into e, zero its row, re-seed it from the not-yet-taken signal with
  the largest residual column norm (np.argmax: first on ties); otherwise
  E_j = e[:, users] + d_j x_j[users], leading singular triple by
  np.linalg.svd (learn.py:139-166, `_leading_pair`), d_j = u, x_j = s v,
  e[:, users] = E_j - u (s v)^T.

Same numpy calls in the same order as the reference, so on this image it
reproduces the reference bit for bit (pinned by tests/test_ksvd_oracle.py on
tests/golden/ksvd_*.npz, made by tests/golden/make_golden_ksvd.py).  The
LAPACK SVD fixes each atom's sign arbitrarily; the device stage uses the
largest-magnitude-entry-positive convention, so tests compare per-atom up
to sign.
"""

from __future__ import annotations

import numpy as np


def leading_pair(ej):
    u, s, vt = np.linalg.svd(ej, full_matrices=False)
    return u[:, 0], s[0], vt[0]


def update_stage(y, d, x, threshold):
    """In place on d, x; returns (replaced, e)."""
    n, m = y.shape
    t = d.shape[1]
    e = y - d @ x
    replaced = 0
    taken = set()
    for j in range(t):
        users = np.flatnonzero(x[j])
        if users.size < threshold:
            if users.size:
                e[:, users] += np.outer(d[:, j], x[j, users])
                x[j, users] = 0.0
            rn = np.linalg.norm(e, axis=0)
            if taken:
                rn[list(taken)] = -1.0
            worst = int(np.argmax(rn))
            taken.add(worst)
            col = y[:, worst]
            cn = np.linalg.norm(col)
            if cn > 0:
                d[:, j] = col / cn
            replaced += 1
            continue
        ej = e[:, users] + np.outer(d[:, j], x[j, users])
        u, s, v = leading_pair(ej)
        d[:, j] = u
        row = s * v
        x[j, users] = row
        e[:, users] = ej - np.outer(u, row)
    return replaced, e


def problem(n, t, m, k, seed, dead=()):
    """Seeded K-SVD update inputs: y from a planted dictionary, d a perturbed
    copy, x random k-sparse codes; atoms in `dead` get 0 or 1 users."""
    rng = np.random.default_rng(seed)
    dt = rng.standard_normal((n, t))
    dt /= np.linalg.norm(dt, axis=0)
    x = np.zeros((t, m))
    live = np.setdiff1d(np.arange(t), np.asarray(dead, dtype=np.int64))
    for p in range(m):
        sup = rng.choice(live, size=k, replace=False)
        x[sup, p] = rng.standard_normal(k)
    for q, j in enumerate(dead):
        if q % 2:
            x[j, rng.integers(m)] = 0.5  # one user
    y = dt @ x + 0.05 * rng.standard_normal((n, m))
    d = dt + 0.1 * rng.standard_normal((n, t))
    d /= np.linalg.norm(d, axis=0)
    return y, d, x


_INIT_COHERENCE_CAP = 0.7
_DUPLICATE_COHERENCE = 0.99


def init_atoms(y, t, init, rng):
    """learn._init_atoms (learn.py:98-128)."""
    n, m = y.shape
    if init == "random-unit":
        g = rng.standard_normal((n, t))
        return g / np.linalg.norm(g, axis=0)
    norms = np.linalg.norm(y, axis=0)
    order = rng.permutation(np.flatnonzero(norms > 0))
    atoms = np.empty((t, n))
    filled = 0
    used = np.zeros(order.size, dtype=bool)
    for pos, c in enumerate(order):
        v = y[:, c] / norms[c]
        if filled and np.abs(atoms[:filled] @ v).max() > _INIT_COHERENCE_CAP:
            continue
        atoms[filled] = v
        filled += 1
        used[pos] = True
        if filled == t:
            break
    for pos, c in enumerate(order):
        if filled == t:
            break
        if not used[pos]:
            atoms[filled] = y[:, c] / norms[c]
            filled += 1
    while filled < t:
        v = rng.standard_normal(n)
        atoms[filled] = v / np.linalg.norm(v)
        filled += 1
    return np.ascontiguousarray(atoms.T)


def cleanup_duplicates(y, d, e):
    """learn._cleanup_duplicates (learn.py:201-228)."""
    t = d.shape[1]
    gram = np.abs(d.T @ d)
    np.fill_diagonal(gram, 0.0)
    resid_norms = np.linalg.norm(e, axis=0)
    taken = set()
    replaced = 0
    for j in range(t):
        if gram[:j, j].max(initial=0.0) <= _DUPLICATE_COHERENCE:
            continue
        rn = resid_norms.copy()
        if taken:
            rn[list(taken)] = -1.0
        worst = int(np.argmax(rn))
        taken.add(worst)
        cn = np.linalg.norm(y[:, worst])
        if cn > 0:
            d[:, j] = y[:, worst] / cn
        gram[j, :] = 0.0
        gram[:, j] = 0.0
        replaced += 1
    return replaced


def train(y, t, k, iterations, seed=0, threshold=1, init="data-columns", rel_tol=1e-6,
          blocks=None, q=None, nthreads=1):
    """learn._ksvd_core (learn.py:265-288) with the C kernel restatement for
    the coding stage (full, or block-restricted with a rectangular block
    list); returns (d, x, pre, post, replaced)."""
    import oracle as O
    n, m = y.shape
    rng = np.random.default_rng(seed)
    d = init_atoms(y, t, init, rng)
    ys_rows = np.ascontiguousarray(y.T)
    pre, post, replaced = [], [], 0
    x = None
    for it in range(iterations):
        if blocks is None:
            r = O.omp_many_arrays(np.ascontiguousarray(d.T), ys_rows, k, rel_tol=rel_tol,
                                  nthreads=nthreads)
        else:
            r = O.omp_many_arrays(np.ascontiguousarray(d.T), ys_rows, k, rel_tol=rel_tol,
                                  allowed_blocks=blocks, block_q=q, nthreads=nthreads)
        x = np.zeros((t, m))
        for p in range(m):
            c = int(r["counts"][p])
            x[r["sel"][p, :c], p] = r["alpha"][p, :c]
        pre.append(float(np.linalg.norm(y - d @ x)))
        rep, e = update_stage(y, d, x, threshold)
        replaced += rep
        post.append(float(np.linalg.norm(e)))
        if it + 1 < iterations:
            replaced += cleanup_duplicates(y, d, e)
    return d, x, np.array(pre), np.array(post), replaced
