"""Golden outputs of the REFERENCE's operator recovery:
crossdict.pipelines.recover with channel-mosaic, temporal-code (multi- and
single-active), angular-sample and mask operators, single-scale OMP and
zero-tree (pipelines.py:175-197, _recover_operator 256-322,
sensing.patch_problem 205-279, crossscale.zero_tree_omp phi branch 194-222).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_operators.py
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import crossdict.pursuit as cpursuit  # noqa: E402
from crossdict import sensing as S  # noqa: E402
from crossdict.crossscale import CrossScaleModel  # noqa: E402
from crossdict.pipelines import PipelineConfig, recover  # noqa: E402
from crossdict.scaling import ScaleSpec  # noqa: E402
from crossdict.tensor import normalize_atoms  # noqa: E402


def _model(fine, factors, t_low, q, k_low, k_high, rng):
    spec = ScaleSpec(fine, factors)
    d_low = normalize_atoms(rng.standard_normal((spec.coarse_size, t_low)))
    d_high = normalize_atoms(rng.standard_normal((spec.fine_size, t_low * q)))
    return CrossScaleModel(d_low, d_high, spec, k_low, k_high)


def _save(name, meas, op_kind, op_arrays, sig_shape, patch, stride, method, est, metrics, **extra):
    np.savez_compressed(
        os.path.join(HERE, f"operator_{name}.npz"), meas=meas, kind=op_kind,
        sig_shape=np.array(sig_shape), patch=np.array(patch), stride=np.array(stride),
        method=method, estimate=np.asarray(est), flagged=metrics.flagged_patches,
        resid=np.asarray(metrics.residual_norms), scans1=metrics.scan_count_step1,
        scans2=metrics.scan_count_step2,
        nesting=-1.0 if metrics.nesting_ok_fraction is None else metrics.nesting_ok_fraction,
        **op_arrays, **extra)


def _run(meas, phi, cfg, sig_shape):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return recover(meas, phi, cfg, signal_shape=sig_shape)


def mosaic(name, spatial, channels, patch, stride, method, rng, k=4):
    sig = np.cumsum(rng.standard_normal(spatial + (channels,)), axis=0) / 3.0
    a = rng.integers(1, channels + 1, size=int(np.prod(spatial)))
    phi = S.make_channel_mosaic(a.size, channels, a)
    coded = phi.apply(sig.ravel()).reshape(spatial)
    sig_shape = spatial + (channels,)
    n = int(np.prod(patch))
    if method == "zerotree":
        model = _model(patch, (2, 2, 1), 10, 3, 3, 5, rng)
        cfg = PipelineConfig("zerotree", model, patch_shape=patch, stride=stride)
        est, met = _run(coded, phi, cfg, sig_shape)
        extra = dict(d_low=model.d_low.atoms, d_high=model.d_high.atoms,
                     factors=np.array((2, 2, 1)), k_low=3, k_high=5)
    else:
        d = normalize_atoms(rng.standard_normal((n, 2 * n)))
        cfg = PipelineConfig("omp-single", d, patch_shape=patch, stride=stride, sparsity=k)
        est, met = _run(coded, phi, cfg, sig_shape)
        extra = dict(atoms=d.atoms, k=k)
    _save(name, coded, "channel-mosaic", dict(assignment=a, channels=channels), sig_shape, patch,
          stride, method, est, met, **extra)


def temporal(name, spatial, frames, patch, stride, method, single, rng, k=4):
    sig = np.cumsum(rng.standard_normal(spatial + (frames,)), axis=-1) / 3.0
    ns = int(np.prod(spatial))
    if single:
        code = np.zeros((ns, frames))
        code[np.arange(ns), rng.integers(0, frames, ns)] = 1.0
    else:
        code = (rng.random((ns, frames)) < 0.5).astype(float)
        code[code.sum(1) == 0, 0] = 1.0
        code[:3] = 1.0  # fully active pixels: the widest sums
    phi = S.make_temporal_code(ns, frames, code)
    coded = phi.apply(sig.ravel()).reshape(spatial)
    sig_shape = spatial + (frames,)
    n = int(np.prod(patch))
    if method == "zerotree":
        model = _model(patch, (2, 2, 2), 12, 4, 3, 6, rng)  # fine (4, 4, F)
        cfg = PipelineConfig("zerotree", model, patch_shape=patch, stride=stride)
        est, met = _run(coded, phi, cfg, sig_shape)
        extra = dict(d_low=model.d_low.atoms, d_high=model.d_high.atoms,
                     factors=np.array((2, 2, 2)), k_low=3, k_high=6)
    else:
        d = normalize_atoms(rng.standard_normal((n, 2 * n)))
        cfg = PipelineConfig("omp-single", d, patch_shape=patch, stride=stride, sparsity=k)
        est, met = _run(coded, phi, cfg, sig_shape)
        extra = dict(atoms=d.atoms, k=k)
    _save(name, coded, "temporal-code", dict(code=code, frames=frames), sig_shape, patch, stride,
          method, est, met, **extra)


def angular(name, spatial, grid, kept, patch, stride, rng, k=4):
    sig = np.cumsum(rng.standard_normal(spatial + grid), axis=0) / 3.0
    ns = int(np.prod(spatial))
    phi = S.make_angular_sample(ns, grid, kept)
    meas = phi.apply(sig.ravel()).reshape(spatial + (len(kept),))
    sig_shape = spatial + grid
    n = int(np.prod(patch))
    d = normalize_atoms(rng.standard_normal((n, 2 * n)))
    cfg = PipelineConfig("omp-single", d, patch_shape=patch, stride=stride, sparsity=k)
    est, met = _run(meas, phi, cfg, sig_shape)
    _save(name, meas, "angular-sample", dict(view_grid=np.array(grid), kept=np.array(kept)),
          sig_shape, patch, stride, "omp-single", est, met, atoms=d.atoms, k=k)


def mask_zt(name, shape, patch, stride, frac, hole, rng):
    sig = np.cumsum(rng.standard_normal(shape), axis=-1) / 4.0
    known = rng.random(shape) < frac
    if hole is not None:
        known[hole] = False
    phi = S.make_mask(int(np.prod(shape)), (np.flatnonzero(known.ravel()) + 1).tolist())
    meas = np.where(known, sig, 0.0)
    model = _model(patch, (2, 2), 8, 4, 3, 6, rng)
    cfg = PipelineConfig("zerotree", model, patch_shape=patch, stride=stride)
    est, met = _run(meas, phi, cfg, shape)
    _save(name, meas, "mask", dict(known=known), shape, patch, stride, "zerotree", est, met,
          d_low=model.d_low.atoms, d_high=model.d_high.atoms, factors=np.array((2, 2)),
          k_low=3, k_high=6)


def main():
    cpursuit.REL_RESIDUAL_TOL = 1e-6
    rng = np.random.default_rng(1479)
    mosaic("mosaic", (14, 13), 3, (4, 4, 3), (2, 2, 1), "omp-single", rng)
    mosaic("mosaic_zt", (12, 12), 3, (4, 4, 3), (2, 2, 1), "zerotree", rng)
    temporal("temporal", (12, 11), 4, (4, 4, 4), (2, 2, 1), "omp-single", False, rng)
    temporal("temporal_single", (10, 10), 4, (4, 4, 4), (3, 3, 1), "omp-single", True, rng)
    temporal("temporal_zt", (12, 12), 4, (4, 4, 4), (2, 2, 1), "zerotree", False, rng)
    angular("angular", (9, 8), (3, 3), [1, 3, 5, 7, 9], (3, 3, 3, 3), (1, 1, 1, 1), rng)
    mask_zt("mask_zt", (20, 18), (4, 4), (2, 2), 0.55, (slice(3, 9), slice(3, 9)), rng)
    # 8 frames: the step-2 frame sums take numpy's pairwise order
    temporal("temporal_zt8", (10, 9), 8, (4, 4, 8), (2, 1, 1), "zerotree", False, rng)
    print("wrote operator goldens")


if __name__ == "__main__":
    main()
