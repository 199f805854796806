"""B200-native batched OMP and zero-tree OMP -- a drop-in for the pursuit path
of ``crossdict`` (arXiv 1511.05174, "Cross-Scale Predictive Dictionaries").

Public API (same names and semantics as the reference):
``PursuitConfig, PursuitResult, BatchSolve, DenseColumns, omp, omp_many,
omp_many_arrays, CrossScaleModel, ZeroTreeResult, cross_scale_map,
zero_tree_omp, zero_tree_omp_many, zero_tree_many_arrays, ScaleSpec,
Dictionary, SparseCode`` plus :func:`install`, which rebinds the reference
package's pursuit entry points to this implementation.
"""

from . import errors
from .crossscale import (CrossScaleModel, ZeroTreeResult, cross_scale_map, omp_cost,
                         predicted_speedup, zero_tree_many_arrays, zero_tree_omp,
                         zero_tree_omp_many)
from .errors import (ChecksumError, ConfigError, CrossdictError, DegenerateAtomError,
                     DimensionError, DomainError, FormatError)
from .fileio import SingleScaleModel, load_model, save_model
from .install import install, uninstall
from .patchwork import (PatchGrid, aggregate_patches, extract_patches, patch_count,
                        reconstruct_aggregate)
from .pipelines import denoise, recover_masked, recover_operator
from . import sensing
from .pursuit import (BatchSolve, DenseColumns, PursuitConfig, PursuitResult, as_columns, omp,
                      omp_many, omp_many_arrays)
from .scaling import ScaleSpec, downsample_columns, upsample_columns
from .tensor import Dictionary, SparseCode, Tensor, as_array, normalize_atoms


def set_engine(name: str) -> None:
    """Select the device engine: "auto" (default), "exact", "gram" or "tensor"."""
    from . import _native, pursuit
    if name not in _native.ENGINES:
        raise ConfigError(f"unknown engine {name!r}")
    pursuit.ENGINE = name


__version__ = "0.1.0"
