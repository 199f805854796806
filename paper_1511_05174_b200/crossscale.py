"""Two-scale zero-tree OMP -- drop-in for crossdict.crossscale's solve path.

Mirrors crossdict/crossscale.py: ``CrossScaleModel`` 34-79, ``ZeroTreeResult``
82-98, ``cross_scale_map`` 101-119, ``omp_cost`` 122-127,
``predicted_speedup`` 130-136, ``zero_tree_omp`` 169-232,
``zero_tree_many_arrays`` 235-283, ``zero_tree_omp_many`` 286-312.

The whole two-step solve of a batch -- block-mean downsample, step-1 OMP on
D_low, per-signal sort of the coarse support, step-2 OMP restricted to the
child blocks -- is one call into the device (``cdb_zero_tree_batch``); the
reference's host-side grouping by coarse support size (crossscale.py:263-279)
is unnecessary because the device engines take a per-signal block count.

Extension (keeps the reference signature): ``zero_tree_many_arrays(model, ys,
phi=...)`` batches the Phi-composed solve of ``zero_tree_omp(model, y, phi)``
on the effective dictionaries Phi U D_low and Phi D_high, built once per
(model, phi) and cached on the device.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field
from functools import cached_property
from typing import Optional

import numpy as np

from . import device as _dev
from . import errors as E
from . import pursuit as _pursuit
from .scaling import upsample_columns


class CrossScaleModel:
    """Paired coarse/fine dictionaries with block map and sparsity budgets."""

    def __init__(self, d_low, d_high, scale, k_low: int, k_high: int):
        t_low, t_high = d_low.num_atoms, d_high.num_atoms
        if t_high % t_low:
            raise E.ConfigError(f"T_high={t_high} is not a multiple of T_low={t_low}")
        q = t_high // t_low
        if d_low.atom_dim != scale.coarse_size:
            raise E.DimensionError(
                f"coarse atom dim {d_low.atom_dim} != coarse patch size {scale.coarse_size}")
        if d_high.atom_dim != scale.fine_size:
            raise E.DimensionError(
                f"fine atom dim {d_high.atom_dim} != fine patch size {scale.fine_size}")
        if not 1 <= k_low <= min(d_low.atom_dim, t_low):
            raise E.ConfigError(f"k_low={k_low} outside [1, min(N_low, T_low)]")
        if k_high < k_low:
            raise E.ConfigError(f"k_high={k_high} must be at least k_low={k_low}")
        if k_high > q * k_low:
            raise E.ConfigError(f"k_high={k_high} exceeds the step-2 search space Q*k_low={q * k_low}")
        self.d_low = d_low
        self.d_high = d_high
        self.scale = scale
        self.k_low = int(k_low)
        self.k_high = int(k_high)
        self.q = int(q)

    @property
    def t_low(self) -> int:
        return self.d_low.num_atoms

    @property
    def t_high(self) -> int:
        return self.d_high.num_atoms

    @cached_property
    def upsampled_low_atoms(self) -> np.ndarray:
        return upsample_columns(self.d_low.atoms, self.scale)

    def __repr__(self):
        return (f"CrossScaleModel(T_low={self.t_low}, T_high={self.t_high}, Q={self.q}, "
                f"k_low={self.k_low}, k_high={self.k_high}, fine_shape={self.scale.fine_shape})")


@dataclass(frozen=True)
class ZeroTreeResult:
    """Two-step solve outcome with per-step instrumentation (crossscale.py:82-98)."""

    code_low: object
    code_high: object
    residual_norm: float
    timings: dict = field(default_factory=dict)
    scan_counts: dict = field(default_factory=dict)
    step1_empty: bool = False
    rank_deficient: bool = False


def cross_scale_map(omega_low, q: int, t_high: int) -> frozenset:
    """Expand coarse support indices (1-based) through the block map."""
    if q < 1:
        raise E.DomainError(f"q must be >= 1, got {q}")
    if t_high < 1 or t_high % q:
        raise E.DomainError(f"t_high={t_high} is not a positive multiple of q={q}")
    t_low = t_high // q
    out = set()
    for i in omega_low:
        i = int(i)
        if not 1 <= i <= t_low:
            raise E.DomainError(f"coarse index {i} outside [1, {t_low}]")
        base = (i - 1) * q
        out.update(range(base + 1, base + q + 1))
    return frozenset(out)


def omp_cost(n: int, t: int, k: int) -> float:
    """Abstract OMP operation count N*T*K + T*K + K^4 + K^3*N (unit constants)."""
    if n < 1 or t < 1 or k < 1:
        raise E.DomainError("cost model arguments must be positive")
    n, t, k = float(n), float(t), float(k)
    return n * t * k + t * k + k**4 + k**3 * n


def predicted_speedup(t_high: int, t_low: int, k_low: int, q: int) -> float:
    """Scan-dominated speedup estimate T_high / (T_low + K_low * Q)."""
    if t_high < 1 or t_low < 1 or q < 1:
        raise E.DomainError("t_high, t_low and q must be positive")
    if k_low < 0:
        raise E.DomainError("k_low must be non-negative")
    return t_high / (t_low + k_low * q)


# --------------------------------------------------------------------- Phi path
_phi_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _phi_matrix_apply(phi, cols):
    if hasattr(phi, "apply_matrix"):
        return np.asarray(phi.apply_matrix(cols), dtype=np.float64)
    return np.asarray(phi, dtype=np.float64) @ cols


def _effective(model, phi):
    """(E_low_t, E_high_t) = rows of Phi U D_low and Phi D_high, cached."""
    per_model = _phi_cache.setdefault(model, {})
    key = id(phi)
    hit = per_model.get(key)
    if hit is not None and hit[0] is phi:
        return hit[1], hit[2]
    e_low = np.ascontiguousarray(_phi_matrix_apply(phi, model.upsampled_low_atoms).T)
    e_high = np.ascontiguousarray(_phi_matrix_apply(phi, model.d_high.atoms).T)
    e_low.setflags(write=False)
    e_high.setflags(write=False)
    per_model[key] = (phi, e_low, e_high)
    return e_low, e_high


def _phi_dims(model, phi):
    n = model.scale.fine_size
    if phi is None:
        return n
    in_dim = phi.input_dim if hasattr(phi, "input_dim") else np.asarray(phi).shape[1]
    if in_dim != n:
        raise E.DimensionError(f"operator input dim {in_dim} != fine size {n}")
    return phi.output_dim if hasattr(phi, "output_dim") else np.asarray(phi).shape[0]


def _solve(model, ys_rows, phi, ys_cols=None):
    """Device two-step solve of signal rows (or, with ``ys_cols``, of the
    N x P column batch itself, transposed on the device); returns
    (low, high, timings)."""
    rel = _pursuit._rel_tol()
    if ys_cols is not None:
        m = ys_cols.shape[0]
    else:
        p_all = ys_rows.shape[0]
        m = ys_rows.shape[1]
    if phi is None:
        dl = _dev.device_dictionary(model.d_low.atoms_t)
        dh = _dev.device_dictionary(model.d_high.atoms_t)
        k1 = model.k_low
        fs, fa = model.scale.fine_shape, model.scale.factors
    else:
        e_low, e_high = _effective(model, phi)
        k1 = min(model.k_low, m, model.t_low)
        dl = _dev.device_dictionary(e_low)
        dh = _dev.device_dictionary(e_high)
        fs = fa = None
    if ys_cols is not None:
        lo, hi, ms = _dev.zero_tree_cols_raw(dl, dh, fs, fa, ys_cols, k1, model.k_high, rel,
                                             phi is not None, _pursuit.ENGINE)
    else:
        lo, hi, ms = _dev.zero_tree_raw(dl, dh, fs, fa, ys_rows, p_all, k1, model.k_high, rel,
                                        phi is not None, _pursuit.ENGINE)
    low = _pursuit._make_batch(model.t_low, lo)
    high = _pursuit._make_batch(model.t_high, hi)
    return low, high, {"step1": float(ms[0]) * 1e-3, "step2": float(ms[1]) * 1e-3}


def _check_ys(model, ys, phi):
    m = _phi_dims(model, phi)
    ys = np.asarray(ys)
    if ys.dtype != np.float32:
        ys = np.asarray(ys, dtype=np.float64)
    if ys.ndim != 2 or ys.shape[0] != m:
        raise E.DimensionError(f"ys must be {m} x P, got {ys.shape}")
    return ys


def zero_tree_many_arrays(model, ys, *, phi=None):
    """Vectorised zero-tree pursuit, raw arrays (crossscale.py:235-283).

    ``ys`` is N x P (or M x P with ``phi``); returns ``(low, high, timings)``
    with ``timings`` the per-step device times in seconds."""
    ys = _check_ys(model, ys, phi)
    p_all = ys.shape[1]
    if p_all == 0:
        z = np.zeros(0, np.int64)
        mk = _pursuit._types.get("BatchSolve", _pursuit.BatchSolve)
        k1 = model.k_low
        return (mk(model.t_low, z, z.reshape(0, k1), np.zeros((0, k1)), np.zeros(0), z),
                mk(model.t_high, z, z.reshape(0, model.k_high), np.zeros((0, model.k_high)),
                   np.zeros(0), z), {"step1": 0.0, "step2": 0.0})
    if _dev.cols_layout(ys):  # large batch: the device transposes, host staging overlaps
        return _solve(model, None, phi, ys_cols=ys)
    return _solve(model, _dev.rows_for_device(ys), phi)


def _zero_tree_result(low, high, p, timings, cls):
    r1 = low.result(p)
    r2 = high.result(p)
    return cls(
        code_low=r1.code,
        code_high=r2.code,
        residual_norm=float(high.rnorm[p]),
        timings=timings,
        scan_counts={"step1": r1.atom_scan_count, "step2": r2.atom_scan_count},
        step1_empty=r1.iterations == 0 and float(high.rnorm[p]) > 0.0,
        rank_deficient=r1.rank_deficient or r2.rank_deficient,
    )


def zero_tree_omp(model, y, phi: Optional[object] = None):
    """Two-step constrained pursuit of one signal (crossscale.py:169-232)."""
    y = np.asarray(y, dtype=np.float64).ravel()
    m = _phi_dims(model, phi)
    if y.size != m:
        raise E.DimensionError(f"measurement length {y.size} != operator output {m}")
    low, high, timings = _solve(model, y.reshape(1, -1), phi)
    cls = _pursuit._types.get("ZeroTreeResult", ZeroTreeResult)
    res = _zero_tree_result(low, high, 0, timings, cls)
    allowed = cross_scale_map(res.code_low.support, model.q, model.t_high)
    assert set(res.code_high.support) <= allowed  # nesting (crossscale.py:224)
    return res


def zero_tree_omp_many(model, ys, *, phi=None) -> list:
    """One ZeroTreeResult per column; timings split evenly (crossscale.py:286-312)."""
    p_all = np.asarray(ys).shape[1]
    if p_all == 0:
        return []
    low, high, timings = zero_tree_many_arrays(model, ys, phi=phi)
    share = {k: v / p_all for k, v in timings.items()}
    cls = _pursuit._types.get("ZeroTreeResult", ZeroTreeResult)
    return [_zero_tree_result(low, high, p, share, cls) for p in range(p_all)]
