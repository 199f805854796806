"""Orthogonal matching pursuit -- drop-in for crossdict.pursuit's OMP path.

Same names, arguments, validation (and messages), return types and error
classes as the reference (crossdict/pursuit.py):

* ``PursuitConfig`` 48-70, ``PursuitResult`` 73-87, ``BatchSolve`` 193-231,
  ``DenseColumns`` 96-123, ``as_columns`` 167-175, ``REL_RESIDUAL_TOL`` 37
* ``omp`` 253-300, ``omp_many_arrays`` 388-441, ``omp_many`` 444-461

but the pursuit itself runs on the B200 through the C ABI
(include/crossdict_b200.h): ``omp_batch_kernel`` (_kernels.py:50-168) is
replaced by ``cdb_omp_batch``.  There is no CPU fallback.

``REL_RESIDUAL_TOL`` is read at call time, exactly like the reference
(pursuit.py:181, 437); after :func:`install` the reference module's global is
the one read.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import device as _dev
from . import errors as E
from . import tensor as _tensor

#: default stopping tolerance is this fraction of ||y|| (pursuit.py:37)
REL_RESIDUAL_TOL = 1e-6

#: engine used by every entry point: "auto" | "exact" | "gram" | "tensor"
ENGINE = "auto"

# Types returned / raised; install() rebinds these to the reference's classes.
_types = {"SparseCode": _tensor.SparseCode}


def _rel_tol() -> float:
    ref = _types.get("pursuit_module")
    return float(ref.REL_RESIDUAL_TOL) if ref is not None else float(REL_RESIDUAL_TOL)


@dataclass(frozen=True)
class PursuitConfig:
    """Sparse-approximation problem parameters (pursuit.py:48-70)."""

    sparsity_budget: int
    residual_tolerance: Optional[float] = None
    allowed_support: Optional[frozenset] = None

    def __post_init__(self):
        if self.sparsity_budget < 1:
            raise E.ConfigError(f"sparsity_budget must be >= 1, got {self.sparsity_budget}")
        if self.residual_tolerance is not None and self.residual_tolerance < 0:
            raise E.ConfigError("residual_tolerance must be >= 0")
        if self.allowed_support is not None:
            allowed = frozenset(int(i) for i in self.allowed_support)
            if any(i < 1 for i in allowed):
                raise E.ConfigError("allowed_support indices are 1-based (must be >= 1)")
            object.__setattr__(self, "allowed_support", allowed)


@dataclass(frozen=True)
class PursuitResult:
    """Outcome of one pursuit run (pursuit.py:73-87)."""

    code: object
    residual_norm: float
    iterations: int
    atom_scan_count: int
    selected: tuple = ()
    rank_deficient: bool = False


class DenseColumns:
    """Column access over an explicit N x T matrix (pursuit.py:96-123)."""

    def __init__(self, matrix):
        mat = np.ascontiguousarray(matrix, dtype=np.float64)
        if mat.ndim != 2:
            raise E.DimensionError(f"column matrix must be 2-D, got ndim={mat.ndim}")
        self.mat = mat
        self._mat_t = None

    @property
    def shape(self):
        return self.mat.shape

    @property
    def mat_t(self) -> np.ndarray:
        if self._mat_t is None:
            self._mat_t = np.ascontiguousarray(self.mat.T)
        return self._mat_t

    def device(self):
        """The staged device dictionary: from `mat` itself (no host transpose
        on a cache hit) unless the rows are already at hand."""
        if self._mat_t is None:
            return _dev.device_dictionary_cols(self.mat)
        return _dev.device_dictionary(self._mat_t)

    def column(self, j0: int) -> np.ndarray:
        return self.mat[:, j0]

    def correlations(self, residual, cand0):
        return self.mat_t[cand0] @ residual

    def materialize(self, idx0) -> np.ndarray:
        return self.mat[:, list(idx0)]


def as_columns(obj):
    """Coerce a Dictionary, ndarray, or columns object to the column protocol.

    Any object with ``atoms`` / ``atoms_t`` (a Dictionary, ours or the
    reference's) keeps its cached read-only transpose, so its device staging
    is cached too.  Lazy column maps (the reference's LazyColumns) are
    materialised: the device needs the explicit matrix.
    """
    if isinstance(obj, DenseColumns):
        return obj
    if hasattr(obj, "atoms_t") and hasattr(obj, "atoms"):
        cols = DenseColumns(obj.atoms)
        cols._mat_t = obj.atoms_t
        return cols
    if hasattr(obj, "materialize") and hasattr(obj, "shape") and not isinstance(obj, np.ndarray):
        if hasattr(obj, "mat") and hasattr(obj, "mat_t"):  # reference DenseColumns
            cols = DenseColumns(obj.mat)
            cols._mat_t = obj.mat_t
            return cols
        n, t = obj.shape
        return DenseColumns(obj.materialize(range(t)))
    return DenseColumns(obj)


def _resolve_eps(config, ynorm: float) -> float:
    if config.residual_tolerance is not None:
        return float(config.residual_tolerance)
    return _rel_tol() * ynorm


@dataclass
class BatchSolve:
    """Raw per-signal arrays from the batched solver (pursuit.py:193-231)."""

    dim: int
    counts: np.ndarray
    sel: np.ndarray
    alpha: np.ndarray
    rnorm: np.ndarray
    scans: np.ndarray
    rank_deficient: frozenset = frozenset()

    def result(self, p: int):
        c = int(self.counts[p])
        chosen = self.sel[p, :c] + 1
        code = _types["SparseCode"].from_arrays(self.dim, chosen.tolist(), self.alpha[p, :c])
        return _types.get("PursuitResult", PursuitResult)(
            code=code,
            residual_norm=float(self.rnorm[p]),
            iterations=c,
            atom_scan_count=int(self.scans[p]),
            selected=tuple(int(j) for j in chosen),
            rank_deficient=p in self.rank_deficient,
        )

    def coefficient_matrix(self) -> np.ndarray:
        """Dense T x P coefficient matrix (columns are the sparse codes)."""
        p_all, k_max = self.sel.shape
        x = np.zeros((self.dim, p_all))
        if k_max:
            cols = np.broadcast_to(np.arange(p_all)[:, None], self.sel.shape)
            safe = np.where(self.sel >= 0, self.sel, 0)
            np.add.at(x, (safe.ravel(), cols.ravel()), self.alpha.ravel())
        return x


def _make_batch(dim, o) -> "BatchSolve":
    cls = _types.get("BatchSolve", BatchSolve)
    deficient = frozenset(int(i) for i in np.flatnonzero(o["flag"]))
    return cls(dim, o["counts"], o["sel"], o["alpha"], o["rnorm"], o["scans"], deficient)


def _empty_result(t: int, rnorm: float):
    return _types.get("PursuitResult", PursuitResult)(
        code=_types["SparseCode"](t, ()), residual_norm=float(rnorm), iterations=0,
        atom_scan_count=0)


def omp(columns, y, config) -> PursuitResult:
    """Orthogonal matching pursuit over the given columns (pursuit.py:253-300)."""
    cols = as_columns(columns)
    n, t = cols.shape
    y = np.asarray(y, dtype=np.float64).ravel()
    if y.size != n:
        raise E.DimensionError(f"signal length {y.size} != column length {n}")
    k_max = config.sparsity_budget
    if k_max > min(n, t):
        raise E.ConfigError(f"sparsity_budget {k_max} exceeds min(N, T) = {min(n, t)}")
    allowed0 = None
    if config.allowed_support is not None:
        allowed0 = np.array(sorted(config.allowed_support), dtype=np.int64) - 1
        if allowed0.size and (allowed0[0] < 0 or allowed0[-1] >= t):
            raise E.DomainError("allowed_support index outside [1, T]")
        if allowed0.size == 0:
            return _empty_result(t, np.linalg.norm(y))
        if k_max > allowed0.size:
            raise E.ConfigError(
                f"sparsity_budget {k_max} exceeds |allowed_support| = {allowed0.size}")
    ynorm = float(np.linalg.norm(y))
    eps = np.array([_resolve_eps(config, ynorm)])
    dd = cols.device()
    o = _dev.omp_batch_raw(dd, y.reshape(1, -1), 1, k_max, eps,
                           None if allowed0 is None else allowed0.reshape(1, -1), ENGINE)
    c = int(o["counts"][0])
    chosen = o["sel"][0, :c] + 1
    code = _types["SparseCode"].from_arrays(t, chosen.tolist(), o["alpha"][0, :c])
    return _types.get("PursuitResult", PursuitResult)(
        code=code, residual_norm=float(o["rnorm"][0]), iterations=c,
        atom_scan_count=int(o["scans"][0]), selected=tuple(int(j) for j in chosen),
        rank_deficient=bool(o["flag"][0]))


def omp_many_arrays(columns, ys, config, *, allowed_blocks=None, block_q=None):
    """Batched OMP over the columns of ``ys`` returning raw arrays
    (pursuit.py:388-441).  With ``allowed_blocks`` (P x nb sorted 0-based
    block ids) and ``block_q`` signal p is restricted to the atoms of its
    blocks and the budget is clipped to the restricted size."""
    cols = as_columns(columns)
    n, t = cols.shape
    ys = np.asarray(ys)
    if ys.dtype != np.float32:
        ys = np.asarray(ys, dtype=np.float64)
    if ys.ndim != 2 or ys.shape[0] != n:
        raise E.DimensionError(f"ys must be {n} x P, got {ys.shape}")
    p_all = ys.shape[1]
    blocks = None
    if allowed_blocks is not None:
        if block_q is None or block_q < 1 or t % block_q:
            raise E.ConfigError("block_q must be a positive divisor of T")
        blocks = np.asarray(allowed_blocks, dtype=np.int64)
        if blocks.ndim != 2 or blocks.shape[0] != p_all:
            raise E.DimensionError("allowed_blocks must be (P, nb)")
        if blocks.size and (blocks.min() < 0 or blocks.max() >= t // block_q):
            raise E.DomainError("block id outside [0, T/Q)")
        k_max = min(config.sparsity_budget, blocks.shape[1] * block_q, n)
    else:
        k_max = config.sparsity_budget
        if k_max > min(n, t):
            raise E.ConfigError(f"sparsity_budget {k_max} exceeds min(N, T) = {min(n, t)}")
    if p_all == 0:
        z = np.zeros(0, np.int64)
        return _types.get("BatchSolve", BatchSolve)(
            t, z, z.reshape(0, k_max), np.zeros((0, k_max)), np.zeros(0), z)

    if blocks is None and _dev.cols_layout(ys):
        # large column batch: staged and transposed on the device, the
        # tolerances rel * |y| computed there (pursuit.py:433-437)
        eps = None
        if config.residual_tolerance is not None:
            eps = np.full(p_all, float(config.residual_tolerance))
        o = _dev.omp_cols_raw(cols.device(), ys, k_max, eps, _rel_tol(),
                              ENGINE)
        return _make_batch(t, o)
    ys_rows = _dev.rows_for_device(ys)
    if config.residual_tolerance is not None:
        eps = np.full(p_all, float(config.residual_tolerance))
    else:
        y64 = ys_rows.astype(np.float64, copy=False)
        eps = _rel_tol() * np.sqrt(np.einsum("pn,pn->p", y64, y64))
    if blocks is not None and (k_max == 0 or blocks.shape[1] == 0):
        # no candidates: the reference kernel returns count 0 and rnorm ||y||
        o = dict(sel=np.full((p_all, k_max), -1, np.int64), alpha=np.zeros((p_all, k_max)),
                 counts=np.zeros(p_all, np.int64),
                 rnorm=np.linalg.norm(ys_rows.astype(np.float64), axis=1),
                 scans=np.zeros(p_all, np.int64), flag=np.zeros(p_all, np.uint8))
        return _make_batch(t, o)
    dd = cols.device()
    if blocks is not None:
        o = _dev.omp_batch_blocked_raw(dd, ys_rows, p_all, k_max, eps,
                                       np.ascontiguousarray(blocks), block_q, ENGINE)
    else:
        o = _dev.omp_batch_raw(dd, ys_rows, p_all, k_max, eps, None, ENGINE)
    return _make_batch(t, o)


def omp_many(columns, ys, config, *, allowed_blocks=None, block_q=None) -> list:
    """Vectorised equivalent of mapping :func:`omp` over columns (pursuit.py:444-461)."""
    solve = omp_many_arrays(columns, ys, config, allowed_blocks=allowed_blocks, block_q=block_q)
    return [solve.result(p) for p in range(np.asarray(ys).shape[1])]
