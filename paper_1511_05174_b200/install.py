"""Drop-in installation into the reference package ``crossdict``.

``install()`` rebinds the reference's pursuit entry points -- wherever the
reference imported them by name -- to this package's B200 implementations:

* ``crossdict.pursuit.{omp, omp_many, omp_many_arrays}``      (pursuit.py:253-461)
* ``crossdict.crossscale.{zero_tree_omp, zero_tree_omp_many,
  zero_tree_many_arrays}``                                    (crossscale.py:169-312)
* ``crossdict.patchwork.{extract_patches, aggregate_patches}`` (patchwork.py:58-122)
* ``crossdict.fileio.load_model`` (fileio.py:216-256): the native CRC-checked
  .csd reader, returning the reference's model classes
* ``crossdict.learn._code_stage`` (learn.py:240-262): K-SVD's coding stage as
  one ragged block-restricted device call, and ``crossdict.learn._update_stage``
  (learn.py:169-199): the rank-one dictionary refits in one device call, and
  ``crossdict.learn._ksvd_core`` (learn.py:265-288): the whole training loop
  with codes, residual and refits kept on the device
* ``crossdict.pipelines._recover_operator`` (pipelines.py:258-322): operator
  recovery (masks, mosaics, temporal codes, angular sampling) with every
  patch coded in one coded-rows device call per step
* the re-exports in ``crossdict/__init__.py:12-33`` and the by-name imports
  of the callers ``crossdict.pipelines`` (pipelines.py:214-297) and
  ``crossdict.learn`` (learn.py:245-260).

After installation results are the reference's own types (``PursuitResult``,
``BatchSolve``, ``SparseCode``, ``ZeroTreeResult``), errors are its own
exception classes, and ``crossdict.pursuit.REL_RESIDUAL_TOL`` is the global
read at call time -- callers cannot tell the difference except for speed.
"""

from __future__ import annotations

import importlib

from . import crossscale as _cs
from . import errors as _errors
from . import fileio as _fileio
from . import learn as _learn
from . import patchwork as _pw
from . import pipelines as _pipelines
from . import pursuit as _pursuit

_saved: dict = {}
_ERRORS = ("CrossdictError", "DimensionError", "DomainError", "DegenerateAtomError",
           "DegenerateDataError", "ConfigError", "ChecksumError", "FormatError")
_FUNCS = {
    "omp": _pursuit.omp,
    "omp_many": _pursuit.omp_many,
    "omp_many_arrays": _pursuit.omp_many_arrays,
    "zero_tree_omp": _cs.zero_tree_omp,
    "zero_tree_omp_many": _cs.zero_tree_omp_many,
    "zero_tree_many_arrays": _cs.zero_tree_many_arrays,
    "extract_patches": _pw.extract_patches,
    "aggregate_patches": _pw.aggregate_patches,
    "_code_stage": _learn.code_stage,  # crossdict.learn only (learn.py:240-262)
    "_update_stage": _learn.update_stage,  # crossdict.learn only (learn.py:169-199)
    "_ksvd_core": _learn.ksvd_core,  # crossdict.learn only (learn.py:265-288)
    "load_model": _fileio.load_model,  # .csd models (fileio.py:216-256)
    "_recover_operator": _pipelines.recover_operator_stage,  # crossdict.pipelines only
}
_MODULES = ("crossdict.pursuit", "crossdict.crossscale", "crossdict", "crossdict.pipelines",
            "crossdict.learn", "crossdict.patchwork", "crossdict.fileio")


def install(package: str = "crossdict") -> list:
    """Rebind the reference's entry points; returns the patched 'module.name' list."""
    if _saved:
        return sorted(k for k in _saved if not k.startswith("#"))
    ref_pursuit = importlib.import_module(f"{package}.pursuit")
    ref_cs = importlib.import_module(f"{package}.crossscale")
    ref_tensor = importlib.import_module(f"{package}.tensor")
    ref_errors = importlib.import_module(f"{package}.errors")
    patched = []
    for modname in _MODULES:
        modname = modname.replace("crossdict", package, 1)
        try:
            mod = importlib.import_module(modname)
        except ImportError:
            continue
        for name, fn in _FUNCS.items():
            if hasattr(mod, name):
                _saved[f"{modname}.{name}"] = (mod, name, getattr(mod, name))
                setattr(mod, name, fn)
                patched.append(f"{modname}.{name}")
    _saved["#types"] = dict(_pursuit._types)
    _saved["#learntypes"] = dict(_learn._types)
    _saved["#fiotypes"] = dict(_fileio._types)
    try:
        ref_fio = importlib.import_module(f"{package}.fileio")
        ref_scaling = importlib.import_module(f"{package}.scaling")
        _fileio._types.update(Dictionary=ref_tensor.Dictionary,
                              SingleScaleModel=ref_fio.SingleScaleModel,
                              CrossScaleModel=ref_cs.CrossScaleModel,
                              ScaleSpec=ref_scaling.ScaleSpec)
    except (ImportError, AttributeError):
        pass
    try:
        ref_learn = importlib.import_module(f"{package}.learn")
        _learn._types.update(TrainReport=ref_learn.TrainReport, report_log=ref_learn.report_log,
                             Dictionary=ref_tensor.Dictionary)
    except (ImportError, AttributeError):
        pass
    _saved["#pwtypes"] = dict(_pw._types)
    try:
        ref_pw = importlib.import_module(f"{package}.patchwork")
        _pw._types.update(PatchGrid=ref_pw.PatchGrid, Tensor=ref_tensor.Tensor)
    except (ImportError, AttributeError):
        pass
    _pursuit._types.update(SparseCode=ref_tensor.SparseCode, PursuitResult=ref_pursuit.PursuitResult,
                           BatchSolve=ref_pursuit.BatchSolve, ZeroTreeResult=ref_cs.ZeroTreeResult,
                           pursuit_module=ref_pursuit)
    _saved["#errors"] = {n: getattr(_errors, n) for n in _ERRORS}
    for n in _ERRORS:
        if hasattr(ref_errors, n):
            setattr(_errors, n, getattr(ref_errors, n))
    return patched


def uninstall() -> None:
    """Restore everything install() changed."""
    for key, val in list(_saved.items()):
        if key == "#types":
            _pursuit._types.clear()
            _pursuit._types.update(val)
        elif key == "#pwtypes":
            _pw._types.clear()
            _pw._types.update(val)
        elif key == "#learntypes":
            _learn._types.clear()
            _learn._types.update(val)
        elif key == "#fiotypes":
            _fileio._types.clear()
            _fileio._types.update(val)
        elif key == "#errors":
            for n, cls in val.items():
                setattr(_errors, n, cls)
        else:
            mod, name, orig = val
            setattr(mod, name, orig)
    _saved.clear()
