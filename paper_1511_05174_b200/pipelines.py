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

import time

import numpy as np

from . import device as _dev
from . import errors as E
from . import patchwork as _pw
from . import pursuit as _pursuit


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
    pshape, strides = _pw._geometry(meas.shape, patch_shape, stride)
    n = int(np.prod(pshape))
    if atoms.shape[0] != n:
        raise E.DimensionError(f"atom dim {atoms.shape[0]} != patch size {n}")
    t = atoms.shape[1]
    k_single = int(min(sparsity, t))
    vals, _ = _dev.extract_patches_raw(meas, pshape, strides, False)
    kept, _ = _dev.extract_patches_raw(known.astype(np.float64), pshape, strides, False)
    vals, kept = np.asarray(vals), np.asarray(kept) != 0.0
    p = vals.shape[0]
    m = kept.sum(axis=1).astype(np.int64)
    order = np.argsort(~kept, axis=1, kind="stable")  # kept cells first, ascending
    rows = np.ascontiguousarray(order, dtype=np.int32)
    ys = np.take_along_axis(vals, order, axis=1)
    ys[np.arange(n)[None, :] >= m[:, None]] = 0.0
    dc = np.zeros(p)
    if remove_dc:
        for mm in np.unique(m[m > 0]):  # numpy's own mean of each compacted row
            sel = np.flatnonzero(m == mm)
            dc[sel] = ys[sel, :mm].mean(axis=1)
            ys[sel, :mm] = ys[sel, :mm] - dc[sel, None]
    rel = _pursuit._rel_tol()
    eps = np.array([rel * float(np.linalg.norm(ys[i, :m[i]])) for i in range(p)])
    dd = _dev.device_dictionary(np.ascontiguousarray(atoms.T))
    o = _dev.omp_batch_masked_raw(dd, np.ascontiguousarray(ys), rows, m, p, k_single, eps)
    flagged = m == 0
    if flagged.any():  # unrecoverable patches contribute 0 (pipelines.py:279-281)
        o["sel"][flagged] = -1
        o["counts"][flagged] = 0
        dc[flagged] = 0.0
    est, unc = _dev.reconstruct_aggregate_raw(dd, o["sel"], o["alpha"], p, dc, meas.shape,
                                              pshape, strides)
    estimate = _pw._finish(est, unc)
    return estimate, _pursuit._make_batch(t, o), int(flagged.sum())
