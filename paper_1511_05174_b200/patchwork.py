"""Overlapping patch extraction and overlap-averaged assembly on the device
 -- mirror of crossdict ``patchwork`` (patchwork.py:23-122).

Same names, arguments, validation, warnings and results as the reference:
``extract_patches`` returns the N x P column matrix (here a transposed view
of the P x N rows the pursuit kernels consume, so feeding it back into
``omp_many_arrays`` / ``zero_tree_many_arrays`` costs no transpose) and the
``PatchGrid``; ``aggregate_patches`` averages columns back into a signal.
``reconstruct_aggregate`` fuses the reference's ``dictionary.atoms @ coef``
(pipelines.py:246) with the aggregation, without the dense T x P coefficient
matrix.  Patch values are fp64 throughout; extraction (values and means) is
bit-identical to the reference, aggregation adds in the reference's order.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import device as _dev
from . import errors as E
from .tensor import Tensor, as_array

_types: dict = {}  # reference classes when installed (install.py)


@dataclass(frozen=True)
class PatchGrid:
    """Geometry of one extraction: shapes, strides, origins, optional DC."""

    signal_shape: tuple
    patch_shape: tuple
    stride: tuple
    origins: np.ndarray
    dc_values: Optional[np.ndarray] = None

    @property
    def patch_count(self) -> int:
        return self.origins.shape[0]

    @property
    def patch_size(self) -> int:
        return int(np.prod(self.patch_shape))


def _as_tuple(value, rank, name):
    if np.isscalar(value):
        return (int(value),) * rank
    t = tuple(int(v) for v in value)
    if len(t) != rank:
        raise E.DimensionError(f"{name} must have {rank} entries, got {len(t)}")
    return t


def patch_count(signal_shape, patch_shape, stride) -> int:
    """Number of patch positions (patchwork.py:50-55)."""
    total = 1
    for ext, pe, st in zip(signal_shape, patch_shape, stride):
        total *= (ext - pe) // st + 1
    return total


def _geometry(arr_shape, patch_shape, stride):
    rank = len(arr_shape)
    pshape = _as_tuple(patch_shape, rank, "patch_shape")
    strides = _as_tuple(stride, rank, "stride")
    if any(s < 1 for s in strides):
        raise E.DimensionError("stride entries must be >= 1")
    if any(pe > ext for pe, ext in zip(pshape, arr_shape)):
        raise E.DimensionError(f"patch {pshape} larger than signal {tuple(arr_shape)}")
    return pshape, strides


def _origins(shape, pshape, strides):
    grid_shape = [(e - q) // s + 1 for e, q, s in zip(shape, pshape, strides)]
    axes = [np.arange(g) * s for g, s in zip(grid_shape, strides)]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1).astype(np.int64)


def extract_rows(signal, patch_shape, stride=1, remove_dc: bool = False):
    """Device extraction: (rows P x N fp64, PatchGrid).  ``signal`` may be a
    CUDA tensor (fp32/fp64) -- then ``rows``/``dc`` stay on the device."""
    on_dev = not isinstance(signal, np.ndarray) and hasattr(signal, "is_cuda") and signal.is_cuda
    arr = signal if on_dev else as_array(signal)
    if arr.ndim < 1 or arr.ndim > 4:
        raise E.DimensionError(f"tensor rank must be 1..4, got {arr.ndim}")
    pshape, strides = _geometry(tuple(arr.shape), patch_shape, stride)
    rows, dc = _dev.extract_patches_raw(arr, pshape, strides, remove_dc)
    grid_cls = _types.get("PatchGrid", PatchGrid)
    grid = grid_cls(tuple(arr.shape), pshape, strides, _origins(arr.shape, pshape, strides), dc)
    return rows, grid


def extract_patches(signal, patch_shape, stride=1, remove_dc: bool = False):
    """Slide a patch window over ``signal``; ``(columns N x P, grid)``
    (patchwork.py:58-89)."""
    rows, grid = extract_rows(signal, patch_shape, stride, remove_dc)
    return rows.T, grid


def _finish(out, uncovered):
    if uncovered:
        warnings.warn(f"{uncovered} signal cells are covered by no patch; left at 0",
                      stacklevel=3)
    return _types.get("Tensor", Tensor)(out)


def aggregate_patches(patch_columns, grid, add_dc: bool = False):
    """Assemble a signal by averaging overlapping patches (patchwork.py:92-122)."""
    cols = np.asarray(patch_columns, dtype=np.float64)
    if cols.shape != (grid.patch_size, grid.patch_count):
        raise E.DimensionError(
            f"expected columns {grid.patch_size} x {grid.patch_count}, got {cols.shape}")
    dc = None
    if add_dc:
        if grid.dc_values is None:
            raise E.DimensionError("grid carries no dc_values to re-add")
        dc = np.ascontiguousarray(grid.dc_values, dtype=np.float64)
    rows = _dev.rows_for_device(cols)  # P x N (threaded transpose into pinned memory)
    out, unc = _dev.aggregate_patches_raw(rows, dc, grid.signal_shape, grid.patch_shape,
                                          grid.stride)
    return _finish(out, unc)


def reconstruct_aggregate(atoms_t, solve, grid, add_dc: bool = False):
    """``aggregate_patches(atoms @ solve.coefficient_matrix(), grid, add_dc)``
    (pipelines.py:246-248) in one device pass: each patch is D_S x from the
    solve's (sel, alpha) rows, no dense coefficient matrix."""
    sel = np.ascontiguousarray(solve.sel, dtype=np.int64)
    alpha = np.ascontiguousarray(solve.alpha, dtype=np.float64)
    if sel.shape[0] != grid.patch_count:
        raise E.DimensionError(f"solve has {sel.shape[0]} codes for {grid.patch_count} patches")
    dc = None
    if add_dc:
        if grid.dc_values is None:
            raise E.DimensionError("grid carries no dc_values to re-add")
        dc = np.ascontiguousarray(grid.dc_values, dtype=np.float64)
    dd = _dev.device_dictionary(np.ascontiguousarray(atoms_t))
    out, unc = _dev.reconstruct_aggregate_raw(dd, sel, alpha, sel.shape[0], dc, grid.signal_shape,
                                              grid.patch_shape, grid.stride)
    return _finish(out, unc)
