"""Device-resident patch recovery: the identity-
measurement path of crossdict ``pipelines._recover_identity``
(pipelines.py:200-253) -- extract_patches -> pursuit -> atoms @ coef ->
aggregate_patches -- with the patch rows, codes and reconstructions kept in
HBM between the stages (the reference round-trips an N x P column matrix, a
dense T x P coefficient matrix and the reconstructed columns through host
memory).  Single-scale OMP (``dictionary`` + ``sparsity``) or zero-tree
(``model``) coding; the stages are the same kernels as the public calls.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import device as _dev
from . import errors as E
from . import patchwork as _pw
from . import pursuit as _pursuit
from . import sensing as _sensing


def _outs(p, k, dev):
    import torch
    return dict(sel=torch.empty((p, k), dtype=torch.int64, device=dev),
                alpha=torch.empty((p, k), dtype=torch.float64, device=dev),
                counts=torch.empty(p, dtype=torch.int64, device=dev),
                rnorm=torch.empty(p, dtype=torch.float64, device=dev),
                scans=torch.empty(p, dtype=torch.int64, device=dev),
                flag=torch.empty(p, dtype=torch.uint8, device=dev))


def _host(o):
    return {k: v.cpu().numpy() for k, v in o.items()}


def denoise(signal, patch_shape, stride=1, *, dictionary=None, sparsity=None, model=None,
            remove_dc: bool = True):
    """Recover ``signal`` (rank 1..4) from its patches' sparse codes.

    Exactly one of ``dictionary`` (N x T atoms, with ``sparsity``) or
    ``model`` (CrossScaleModel: zero-tree coding on its fine dictionary).
    Returns ``(estimate, solve, timings)``: the overlap-averaged
    reconstruction (Tensor), the BatchSolve (or ``(low, high)``) of the
    patch codes, and per-stage seconds.
    """
    import torch
    if (dictionary is None) == (model is None):
        raise E.ConfigError("pass exactly one of dictionary= or model=")
    t0 = time.perf_counter()
    sig = torch.as_tensor(np.asarray(_pw.as_array(signal)), device="cuda")
    pshape, strides = _pw._geometry(tuple(sig.shape), patch_shape, stride)
    p = _pw.patch_count(sig.shape, pshape, strides)
    n = int(np.prod(pshape))
    rows = torch.empty((p, n), dtype=torch.float64, device="cuda")
    dc = torch.empty(p, dtype=torch.float64, device="cuda") if remove_dc else None
    _dev.extract_patches_raw(sig, pshape, strides, remove_dc, rows, dc)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rel = _pursuit._rel_tol()
    if dictionary is not None:
        atoms = np.asarray(getattr(dictionary, "atoms", dictionary), dtype=np.float64)
        if atoms.shape[0] != n:
            raise E.DimensionError(f"atom dim {atoms.shape[0]} != patch size {n}")
        k = int(min(sparsity, atoms.shape[0], atoms.shape[1]))
        atoms_t = np.ascontiguousarray(atoms.T)
        dd = _dev.device_dictionary(atoms_t)
        eps = rel * torch.sqrt((rows * rows).sum(dim=1))
        out = _outs(p, k, "cuda")
        _dev.omp_batch_raw(dd, rows, p, k, eps, None, _pursuit.ENGINE, out)
        code = out
        t_dim = atoms.shape[1]
    else:
        if model.d_high.atom_dim != n:
            raise E.DimensionError(f"model fine size {model.d_high.atom_dim} != patch size {n}")
        atoms_t = model.d_high.atoms_t
        dd = _dev.device_dictionary(atoms_t)
        dl = _dev.device_dictionary(model.d_low.atoms_t)
        lo, code = _outs(p, model.k_low, "cuda"), _outs(p, model.k_high, "cuda")
        fs = model.scale.fine_shape
        if tuple(fs) != tuple(pshape):
            raise E.DimensionError(f"model patch shape {fs} != {pshape}")
        _dev.zero_tree_raw(dl, dd, fs, model.scale.factors, rows, p, model.k_low, model.k_high,
                           rel, False, _pursuit.ENGINE, lo, code)
        t_dim = model.t_high
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    est = torch.empty(tuple(sig.shape), dtype=torch.float64, device="cuda")
    _, unc = _dev.reconstruct_aggregate_raw(dd, code["sel"], code["alpha"], p, dc, tuple(sig.shape),
                                            pshape, strides, est)
    estimate = _pw._finish(est.cpu().numpy(), unc)
    t3 = time.perf_counter()
    mk = _pursuit._make_batch
    solve = mk(t_dim, _host(code)) if model is None else (mk(model.t_low, _host(lo)),
                                                          mk(model.t_high, _host(code)))
    return estimate, solve, {"extract": t1 - t0, "coding": t2 - t1, "reconstruct": t3 - t2}


@dataclass
class RecoveryMetrics:
    """Per-run instrumentation (pipelines.RecoveryMetrics, pipelines.py:80-96;
    the fields the operator path fills)."""

    method: str
    patch_count: int = 0
    residual_norms: np.ndarray = field(default_factory=lambda: np.zeros(0))
    scan_count_step1: int = 0
    scan_count_step2: int = 0
    nesting_ok_fraction: Optional[float] = None
    flagged_patches: int = 0
    coding_time_s: float = 0.0
    aggregate_time_s: float = 0.0


def _default_stride(patch_shape, signal_shape):
    return tuple(ext if pe == ext else max(1, pe // 2) for pe, ext in zip(patch_shape, signal_shape))


def recover_operator(measurements, phi, patch_shape, stride=None, *, dictionary=None,
                     sparsity=None, model=None, remove_dc=None, signal_shape=None):
    """Patch recovery through a structured measurement operator (SURVEY §8
    row f3): crossdict ``pipelines._recover_operator`` (pipelines.py:258-322)
    with ``sensing.patch_problem`` (sensing.py:205-279) for masks, channel
    mosaics, temporal codes and angular sampling, coding every patch in ONE
    batched exact-engine call per step (``cdb_omp_batch_coded``) instead of
    one scalar ``omp`` / ``zero_tree_omp(phi=sub_op)`` per patch.

    ``dictionary`` + ``sparsity``: method "omp-single" (OMP on phi_p D, budget
    min(sparsity, T, m_p)).  ``model`` (CrossScaleModel): method "zerotree",
    the Phi form of zero_tree_omp per patch (crossscale.py:194-222): step 1 on
    phi_p U D_low with budget min(k_low, m_p, T_low), step 2 on phi_p D_high
    restricted to the step-1 blocks with budget min(k_high, nb Q, m_p).
    ``remove_dc`` defaults to on for masks only (and is refused otherwise).
    Returns ``(estimate, metrics, codes)``: the overlap-averaged estimate
    (Tensor), a RecoveryMetrics, and the device outputs (``{"step1", "step2"}``
    for zero-tree, ``{"code"}`` otherwise).
    """
    if (dictionary is None) == (model is None):
        raise E.ConfigError("pass exactly one of dictionary= (with sparsity=) or model=")
    if phi is None or phi.kind == "identity":
        raise E.ConfigError("identity measurements: use pipelines.denoise")
    meas = np.asarray(_pw.as_array(measurements), dtype=np.float64)
    sig_shape = _sensing.signal_shape_for(phi, meas.shape, signal_shape)
    pshape = tuple(int(e) for e in patch_shape)
    if len(pshape) != len(sig_shape):
        raise E.DimensionError(f"patch rank {len(pshape)} != signal rank {len(sig_shape)}")
    if stride is None:
        stride = _default_stride(pshape, sig_shape)
    pshape, strides = _pw._geometry(sig_shape, pshape, stride)
    if remove_dc is None:
        remove_dc = phi.kind == "mask"
    if remove_dc and phi.kind != "mask":
        raise E.ConfigError(f"DC removal is only supported for mask measurements, not {phi.kind}")
    n = int(np.prod(pshape))
    if phi.input_dim != int(np.prod(sig_shape)):
        raise E.DimensionError(f"operator input dim {phi.input_dim} != signal size "
                               f"{int(np.prod(sig_shape))}")
    ys, rows, m = _sensing.coded_problems(phi, meas, sig_shape, pshape, strides)
    p = ys.shape[0]

    def slot_rows():
        if phi.kind != "temporal-code":
            return rows
        return _sensing.coded_problems(phi, meas, sig_shape, pshape, strides, slots=True)[1]

    dc = np.zeros(p)
    if remove_dc:
        for mm in np.unique(m[m > 0]):  # numpy's own mean of each compacted row
            sel = np.flatnonzero(m == mm)
            dc[sel] = ys[sel, :mm].mean(axis=1)
            ys[sel, :mm] = ys[sel, :mm] - dc[sel, None]
    # np.linalg.norm of a 1-D real vector is sqrt(x.dot(x)) (numpy _linalg.py
    # norm): the same BLAS dot per patch, without the wrapper's overhead
    ynorm = np.array([math.sqrt(r.dot(r)) for r in (ys[i, :m[i]] for i in range(p))])
    eps = _pursuit._rel_tol() * ynorm
    empty = m == 0  # unrecoverable patch: skipped, contributes 0 (pipelines.py:279-281)
    metrics = RecoveryMetrics("zerotree" if model is not None else "omp-single", patch_count=p)
    t0 = time.perf_counter()
    if dictionary is not None:
        atoms = np.asarray(getattr(dictionary, "atoms", dictionary), dtype=np.float64)
        if atoms.shape[0] != n:
            raise E.DimensionError(f"atom dim {atoms.shape[0]} != patch size {n}")
        dd = _dev.device_dictionary(np.ascontiguousarray(atoms.T))
        k = int(min(sparsity, atoms.shape[1]))
        pw = atoms.shape[1] == 1  # one column: numpy reduces the frame axis pairwise
        code = _dev.omp_batch_coded_raw(dd, ys, slot_rows() if pw else rows, m, p, k, eps,
                                        pairwise=pw)
        metrics.scan_count_step1 = int(code["scans"].sum())
        codes = {"code": code}
    else:
        if model.d_high.atom_dim != n:
            raise E.DimensionError(f"model fine size {model.d_high.atom_dim} != patch size {n}")
        dlow = _dev.device_dictionary(np.ascontiguousarray(model.upsampled_low_atoms.T))
        dd = _dev.device_dictionary(model.d_high.atoms_t)
        pw1 = model.t_low == 1
        s1 = _dev.omp_batch_coded_raw(dlow, ys, slot_rows() if pw1 else rows, m, p, model.k_low,
                                      eps, pairwise=pw1)
        c1 = np.asarray(s1["counts"])
        kb = max(int(c1.max()) if p else 0, 1)
        blocks = np.sort(np.where(np.arange(s1["sel"].shape[1])[None, :] < c1[:, None],
                                  s1["sel"], np.iinfo(np.int64).max), axis=1)[:, :kb]
        blocks = np.ascontiguousarray(np.where(blocks == np.iinfo(np.int64).max, 0, blocks))
        # step 2 applies phi to d_high.atoms_t[allowed0].T (crossscale.py:215): the
        # frame axis is the contiguous one, so numpy sums it pairwise
        code = _dev.omp_batch_coded_raw(dd, ys, slot_rows(), m, p, model.k_high, eps, blocks,
                                        np.ascontiguousarray(c1, dtype=np.int64), model.q,
                                        pairwise=True)
        s1_empty = (c1 == 0) & ~empty & (ynorm > 0)  # step1_empty (crossscale.py:204)
        code["rnorm"][c1 == 0] = ynorm[c1 == 0]  # _zero_result (crossscale.py:139-148)
        metrics.scan_count_step1 = int(s1["scans"].sum())
        metrics.scan_count_step2 = int(code["scans"].sum())
        live = ~empty
        hs, hc = code["sel"], code["counts"]
        ok = [set((hs[i, :hc[i]] // model.q).tolist()) <= set(s1["sel"][i, :c1[i]].tolist())
              for i in np.flatnonzero(live)]
        metrics.nesting_ok_fraction = float(np.mean(ok)) if ok else 1.0
        metrics.flagged_patches += int(s1_empty.sum())
        codes = {"step1": s1, "step2": code}
    metrics.coding_time_s = time.perf_counter() - t0
    metrics.flagged_patches += int(empty.sum())
    resid = np.asarray(code["rnorm"], dtype=np.float64).copy()
    resid[empty] = 0.0
    metrics.residual_norms = resid
    if empty.any():
        code["sel"][empty] = -1
        code["counts"][empty] = 0
        dc[empty] = 0.0
    t1 = time.perf_counter()
    est, unc = _dev.reconstruct_aggregate_raw(dd, code["sel"], code["alpha"], p, dc, sig_shape,
                                              pshape, strides)
    metrics.aggregate_time_s = time.perf_counter() - t1
    return _pw._finish(est, unc), metrics, codes


def recover_operator_stage(meas, phi, sig_shape, patch_shape, stride, config, metrics):
    """Drop-in for crossdict ``pipelines._recover_operator`` (pipelines.py:
    258-322): same arguments, fills the caller's RecoveryMetrics, returns
    ``(estimate, metrics)``; every patch is coded in one device call per
    step (see :func:`recover_operator`)."""
    t0 = time.perf_counter()
    if config.method == "zerotree":
        kw = dict(model=config.model)
    else:
        d = config.fine_dictionary()
        kw = dict(dictionary=d.atoms, sparsity=config.resolved_sparsity())
    est, met, _ = recover_operator(meas, phi, patch_shape, stride, remove_dc=config.remove_dc,
                                   signal_shape=sig_shape, **kw)
    total = time.perf_counter() - t0
    metrics.patch_count = met.patch_count
    metrics.coding_time_s = met.coding_time_s
    metrics.aggregate_time_s = met.aggregate_time_s
    metrics.prep_time_s = total - met.coding_time_s - met.aggregate_time_s
    metrics.residual_norms = met.residual_norms
    metrics.scan_count_step1 += met.scan_count_step1
    metrics.scan_count_step2 += met.scan_count_step2
    if config.method == "zerotree":
        metrics.nesting_ok_fraction = met.nesting_ok_fraction
    metrics.flagged_patches += met.flagged_patches
    return est, metrics


def recover_masked(measurements, known, patch_shape, stride=1, *, dictionary, sparsity,
                   remove_dc: bool = True):
    """Inpainting / masked recovery: crossdict
    ``pipelines._recover_operator`` for a mask operator with single-scale OMP
    (pipelines.py:256-322, sensing.patch_problem mask branch sensing.py:222-231).

    ``measurements``: the signal-domain array (unknown cells arbitrary);
    ``known``: boolean array of the same shape.  Each patch is coded against
    the rows of ``dictionary`` at its known cells (OMP on the compacted
    effective dictionary, device exact engine), reconstructed with the full
    atoms plus its DC, and the patches are overlap-averaged.  Patches with no
    known cell are flagged and contribute 0.  Returns ``(estimate, solve,
    flagged)``.
    """
    meas = np.asarray(_pw.as_array(measurements), dtype=np.float64)
    known = np.asarray(known, dtype=bool)
    if known.shape != meas.shape:
        raise E.DimensionError(f"mask shape {known.shape} != measurement shape {meas.shape}")
    atoms = np.asarray(getattr(dictionary, "atoms", dictionary), dtype=np.float64)
    phi = _sensing.mask_from_tensor(known)
    estimate, metrics, codes = recover_operator(meas, phi, patch_shape, stride,
                                                dictionary=atoms, sparsity=sparsity,
                                                remove_dc=remove_dc, signal_shape=meas.shape)
    return estimate, _pursuit._make_batch(atoms.shape[1], codes["code"]), metrics.flagged_patches
