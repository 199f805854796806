"""Structured measurement operators and their per-patch slicing (SURVEY §8
row f3, host side).

Mirrors crossdict.sensing (sensing.py:25-199): the same constructors, kinds,
attribute names (``kind``, ``input_dim``, ``output_dim``, ``params``, the
gather / code / matrix payloads) and ``ConfigError`` behaviour, so an
operator built by either package works with
:func:`paper_1511_05174_b200.pipelines.recover_operator`.

:func:`coded_problems` is the all-patches form of ``sensing.patch_problem``
(sensing.py:205-279): instead of one sub-operator object per patch it emits
the arrays ``cdb_omp_batch_coded`` consumes -- per patch the measurements
and, per measurement, the atom coordinates whose ordered sum is the
effective atom entry (a gather for masks, mosaics and angular sampling; the
active frames of a binary temporal code).
"""

from __future__ import annotations

import numpy as np

from . import errors as E
from .tensor import as_array

KINDS = ("identity", "mask", "channel-mosaic", "temporal-code", "angular-sample", "dense")


class LinearOperator:
    """Measurement map (sensing.py:25-92); build it with the constructors."""

    def __init__(self, kind, input_dim, output_dim, *, gather=None, code=None, matrix=None,
                 params=None):
        if kind not in KINDS:
            raise E.ConfigError(f"unknown operator kind {kind!r}")
        self.kind = kind
        self.input_dim = int(input_dim)
        self.output_dim = int(output_dim)
        self._gather = gather
        self._code = code
        self._matrix = matrix
        self.params = params or {}

    def __repr__(self):
        return f"LinearOperator(kind={self.kind!r}, {self.output_dim}x{self.input_dim})"

    def apply_matrix(self, cols):
        """Forward map of every column of an N x C matrix (sensing.py:78-92)."""
        cols = np.asarray(cols, dtype=np.float64)
        if cols.shape[0] != self.input_dim:
            raise E.DimensionError(
                f"columns must have length {self.input_dim}, got {cols.shape[0]}")
        if self.kind == "identity":
            return cols.copy()
        if self._gather is not None:
            return cols[self._gather]
        if self.kind == "temporal-code":
            s, f = self._code.shape
            return (cols.reshape(s, f, -1) * self._code[:, :, None]).sum(axis=1)
        return self._matrix @ cols

    def apply(self, x):
        return self.apply_matrix(as_array(x).reshape(-1, 1))[:, 0]


def identity(n: int) -> LinearOperator:
    if n < 1:
        raise E.ConfigError("identity needs n >= 1")
    return LinearOperator("identity", n, n)


def make_mask(n: int, known_indices) -> LinearOperator:
    """Keep the listed coordinates (1-based) of a length-n signal."""
    idx = np.asarray(list(known_indices), dtype=np.int64)
    if idx.size < 1:
        raise E.ConfigError("mask must keep at least one coordinate")
    if idx.min() < 1 or idx.max() > n:
        raise E.ConfigError(f"mask index outside [1, {n}]")
    if np.unique(idx).size != idx.size:
        raise E.ConfigError("mask indices must be unique")
    gather = np.sort(idx) - 1
    return LinearOperator("mask", n, gather.size, gather=gather, params={"known": gather + 1})


def mask_from_tensor(known) -> LinearOperator:
    flags = as_array(known).ravel()
    return make_mask(flags.size, (np.flatnonzero(flags != 0) + 1).tolist())


def make_channel_mosaic(spatial_extent: int, channel_count: int, assignment) -> LinearOperator:
    """Pixel p reads channel assignment[p] (1-based); channel axis last."""
    a = np.asarray(list(assignment), dtype=np.int64).ravel()
    if a.size != spatial_extent:
        raise E.ConfigError(f"assignment length {a.size} != spatial extent {spatial_extent}")
    if channel_count < 1 or a.min() < 1 or a.max() > channel_count:
        raise E.ConfigError(f"assignment values must lie in [1, {channel_count}]")
    gather = np.arange(spatial_extent, dtype=np.int64) * channel_count + (a - 1)
    return LinearOperator("channel-mosaic", spatial_extent * channel_count, spatial_extent,
                          gather=gather, params={"assignment": a, "channels": channel_count})


def make_temporal_code(spatial_extent: int, frames: int, code) -> LinearOperator:
    """Coded exposure: pixel p sums the frames with code[p, f] = 1; frame axis last."""
    c = np.asarray(code, dtype=np.float64).reshape(spatial_extent, frames)
    if not np.isin(c, (0.0, 1.0)).all():
        raise E.ConfigError("temporal code must be binary (0/1)")
    active = c.sum(axis=1)
    dead = np.flatnonzero(active == 0)
    if dead.size:
        raise E.ConfigError(f"pixel {dead[0] + 1} is active in no frame")
    gather = None
    if (active == 1).all():
        gather = np.arange(spatial_extent, dtype=np.int64) * frames + np.argmax(c, axis=1)
    return LinearOperator("temporal-code", spatial_extent * frames, spatial_extent,
                          gather=gather, code=np.ascontiguousarray(c),
                          params={"frames": frames})


def make_angular_sample(spatial_extent: int, view_grid, kept_views) -> LinearOperator:
    """Keep whole views (1-based, row-major) of a (spatial, vr, vc) light field."""
    vr, vc = (int(v) for v in view_grid)
    n_views = vr * vc
    kept = np.asarray(list(kept_views), dtype=np.int64)
    if kept.size < 1:
        raise E.ConfigError("must keep at least one view")
    if kept.min() < 1 or kept.max() > n_views:
        raise E.ConfigError(f"view index outside [1, {n_views}]")
    if np.unique(kept).size != kept.size:
        raise E.ConfigError("kept views must be unique")
    kept = np.sort(kept)
    gather = (np.arange(spatial_extent, dtype=np.int64)[:, None] * n_views
              + (kept - 1)[None, :]).ravel()
    return LinearOperator("angular-sample", spatial_extent * n_views,
                          spatial_extent * kept.size, gather=gather,
                          params={"view_grid": (vr, vc), "kept": kept})


def make_dense(matrix) -> LinearOperator:
    m = np.ascontiguousarray(matrix, dtype=np.float64)
    if m.ndim != 2:
        raise E.DimensionError("dense operator needs a 2-D matrix")
    return LinearOperator("dense", m.shape[1], m.shape[0], matrix=m)


def signal_shape_for(op, meas_shape, explicit=None):
    """pipelines._signal_shape_for (pipelines.py:120-135)."""
    if explicit is not None:
        return tuple(int(e) for e in explicit)
    if op is None or op.kind in ("identity", "mask"):
        return tuple(meas_shape)
    if op.kind == "channel-mosaic":
        return tuple(meas_shape) + (op.params["channels"],)
    if op.kind == "temporal-code":
        return tuple(meas_shape) + (op.params["frames"],)
    if op.kind == "angular-sample":
        return tuple(meas_shape[:-1]) + tuple(op.params["view_grid"])
    raise E.ConfigError(f"signal_shape required for operator kind {op.kind!r}")


def window_index(shape, pshape, strides):
    """(P, prod(pshape)) flat row-major indices of every patch window, the
    patches in extract_patches' row-major origin order (patchwork.py:58-89)."""
    shape, pshape, strides = tuple(shape), tuple(pshape), tuple(strides)
    flat = [int(np.prod(shape[a + 1:])) for a in range(len(shape))]
    base = np.zeros(1, dtype=np.int64)
    local = np.zeros(1, dtype=np.int64)
    for a in range(len(shape)):
        g = (shape[a] - pshape[a]) // strides[a] + 1
        base = np.add.outer(base, np.arange(g, dtype=np.int64) * strides[a] * flat[a]).ravel()
        local = np.add.outer(local, np.arange(pshape[a], dtype=np.int64) * flat[a]).ravel()
    return base[:, None] + local[None, :]


def coded_problems(op, measurement, sig_shape, pshape, strides, slots: bool = False):
    """All patches' measurement problems (sensing.patch_problem, sensing.py:
    205-279, vectorised).  Returns ``(ys, rows, m)``: ys P x M fp64 (first
    m[p] used), rows P x M x fan int32 patch-local atom coordinates (-1 pad),
    m[p] the measurement count (0: unrecoverable patch, mask kind only).
    A temporal code lists each pixel's active frames in order (the
    sequential-sum form), or with ``slots`` all F frame slots, -1 where the
    code is 0 (the form cdb_omp_batch_coded sums in numpy's pairwise order)."""
    sig_shape, pshape, strides = tuple(sig_shape), tuple(pshape), tuple(strides)
    meas = np.asarray(as_array(measurement), dtype=np.float64)
    kind = op.kind
    if kind == "mask":
        if meas.shape != sig_shape:
            raise E.DimensionError(
                f"embedded measurement shape {meas.shape} != signal {sig_shape}")
        known = np.zeros(int(np.prod(sig_shape)), dtype=bool)
        known[op._gather] = True
        idx = window_index(sig_shape, pshape, strides)
        kept = known[idx]
        m = kept.sum(axis=1).astype(np.int64)
        order = np.argsort(~kept, axis=1, kind="stable")  # kept cells first, ascending
        ys = np.take_along_axis(meas.ravel()[idx], order, axis=1)
        ys[np.arange(idx.shape[1])[None, :] >= m[:, None]] = 0.0
        return ys, np.ascontiguousarray(order[:, :, None], dtype=np.int32), m
    if kind in ("channel-mosaic", "temporal-code"):
        depth = op.params["channels"] if kind == "channel-mosaic" else op.params["frames"]
        what = "mosaic patches must span the full channel axis" if kind == "channel-mosaic" \
            else "temporal patches must span the full frame axis"
        if sig_shape[-1] != depth or pshape[-1] != depth:
            raise E.DimensionError(what)
        spatial = sig_shape[:-1]
        if meas.shape != spatial:
            raise E.DimensionError(f"coded image shape {meas.shape} != spatial {spatial}")
        idx = window_index(spatial, pshape[:-1], strides[:-1])
        p, s = idx.shape
        ys = np.ascontiguousarray(meas.ravel()[idx])
        base = (np.arange(s, dtype=np.int64) * depth)[None, :, None]
        if kind == "channel-mosaic":
            a = op.params["assignment"].reshape(-1)[idx]
            rows = base + (a - 1)[:, :, None]
        elif slots:
            code = op._code.reshape(-1, depth)[idx] != 0.0      # P x S x F
            rows = np.where(code, base + np.arange(depth)[None, None, :], -1)
        else:
            code = op._code.reshape(-1, depth)[idx] != 0.0      # P x S x F
            fan = int(code.sum(axis=2).max())
            order = np.argsort(~code, axis=2, kind="stable")[:, :, :fan]  # active frames first
            live = np.take_along_axis(code, order, axis=2)
            rows = np.where(live, base + order, -1)
        return ys, np.ascontiguousarray(rows, dtype=np.int32), np.full(p, s, dtype=np.int64)
    if kind == "angular-sample":
        vr, vc = op.params["view_grid"]
        kept = op.params["kept"]
        if sig_shape[-2:] != (vr, vc) or pshape[-2:] != (vr, vc):
            raise E.DimensionError("angular patches must span the full view grid")
        spatial = sig_shape[:-2]
        if meas.shape != spatial + (kept.size,):
            raise E.DimensionError(
                f"measurement shape {meas.shape} != {spatial + (kept.size,)}")
        idx = window_index(spatial, pshape[:-2], strides[:-2])
        p, s = idx.shape
        ys = np.ascontiguousarray(meas.reshape(-1, kept.size)[idx].reshape(p, s * kept.size))
        one = (np.arange(s, dtype=np.int64)[:, None] * (vr * vc) + (kept - 1)[None, :]).ravel()
        rows = np.broadcast_to(one[None, :, None], (p, one.size, 1))
        return ys, np.ascontiguousarray(rows, dtype=np.int32), np.full(p, one.size, np.int64)
    raise E.ConfigError(f"cannot slice operator kind {kind!r} per patch")
