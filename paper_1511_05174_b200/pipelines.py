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
