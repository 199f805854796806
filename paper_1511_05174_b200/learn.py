"""K-SVD on the device: the coding stage -- mirror of
crossdict ``learn._code_stage`` (learn.py:240-262), the call K-SVD training
makes every iteration with the dictionary it is refitting -- and the
dictionary-update stage, ``learn._update_stage`` (learn.py:169-199).

The reference groups the samples by their block count and issues one
block-restricted ``omp_many`` per group, because its kernel takes rectangular
``allowed_blocks``; here one ragged device call codes every sample
(``cdb_omp_batch_blocked_ragged``: per-sample block count, budget
min(k, nb * Q, N) -- the per-group rule of pursuit.py:423).  Results are the
reference's per-sample ``PursuitResult`` list in sample order.  ``install()``
binds this function as ``crossdict.learn._code_stage``.

``update_stage`` runs the sequential rank-one refits in one device call
(``cdb_ksvd_update``, csrc/ksvd_engine.cu) and is bound as
``crossdict.learn._update_stage``.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as _N
from . import device as _dev
from . import errors as E
from . import tensor as _tensor
from . import pursuit as _pursuit
from .pursuit import PursuitConfig


def code_stage(d, y, k, allowed_sets, block_hint):
    """Sparse-code every column of ``y`` against ``d`` (learn.py:240-262)."""
    d = np.asarray(d, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    m = y.shape[1]
    if allowed_sets is None:
        return _pursuit.omp_many(d, y, PursuitConfig(k))
    if block_hint is not None:
        blocks_list, q = block_hint
        n, t = d.shape
        # the reference reaches omp_many's block checks (pursuit.py:414-420)
        if q is None or q < 1 or t % q:
            raise E.ConfigError("block_q must be a positive divisor of T")
        for b in blocks_list:
            if len(b) and (min(b) < 0 or max(b) >= t // q):
                raise E.DomainError("block id outside [0, T/Q)")
        nb = np.array([len(b) for b in blocks_list], dtype=np.int64)
        nb_max = max(1, int(nb.max()) if m else 1)
        blocks = np.zeros((m, nb_max), dtype=np.int64)
        for p, b in enumerate(blocks_list):
            if len(b):
                blocks[p, :len(b)] = sorted(b)
        k_out = int(max(1, min(k, nb_max * q, n)))
        if m == 0:
            return []
        ys_rows = _dev.rows_for_device(y)
        cfg = PursuitConfig(k)
        if cfg.residual_tolerance is not None:
            eps = np.full(m, float(cfg.residual_tolerance))
        else:
            eps = _pursuit._rel_tol() * np.sqrt(np.einsum("pn,pn->p", ys_rows, ys_rows))
        dd = _dev.device_dictionary(np.ascontiguousarray(d.T))
        o = _dev.omp_batch_blocked_ragged_raw(dd, ys_rows, m, k_out, eps, blocks, nb, int(q),
                                              _pursuit.ENGINE)
        solve = _pursuit._make_batch(t, o)
        return [solve.result(p) for p in range(m)]
    # arbitrary per-sample sets (the reference runs one scalar omp per sample,
    # learn.py:258-261): ONE ragged call with Q = 1 -- the "blocks" are the
    # sorted allowed atom ids, the budget min(k, |set|, N) per sample
    n, t = d.shape
    if m == 0:
        return []
    for s_ in allowed_sets:
        if min(k, len(s_)) > min(n, t):
            raise E.ConfigError(f"sparsity_budget {min(k, len(s_))} exceeds min(N, T) = {min(n, t)}")
    sizes = np.array([len(s_) for s_ in allowed_sets], dtype=np.int64)
    width = max(1, int(sizes.max()))
    ids = np.zeros((m, width), dtype=np.int64)
    for p, s_ in enumerate(allowed_sets):
        srt = np.sort(np.fromiter(s_, dtype=np.int64, count=len(s_))) - 1
        if srt.size and (srt[0] < 0 or srt[-1] >= t):
            raise E.DomainError("allowed_support index outside [1, T]")
        ids[p, :srt.size] = srt
    ys_rows = np.ascontiguousarray(y.T)
    # scalar omp's tolerance: REL * np.linalg.norm(y_p) = REL * sqrt(y_p . y_p)
    eps = _pursuit._rel_tol() * np.array([math.sqrt(r.dot(r)) for r in ys_rows])
    k_out = int(max(1, min(k, width, n)))
    dd = _dev.device_dictionary(np.ascontiguousarray(d.T))
    o = _dev.omp_batch_blocked_ragged_raw(dd, ys_rows, m, k_out, eps, ids, sizes, 1,
                                          _pursuit.ENGINE)
    solve = _pursuit._make_batch(t, o)
    return [solve.result(p) for p in range(m)]


def update_stage(y, d, x, threshold: int):
    """Sequential rank-one atom refits (learn.py:169-199): updates ``d``
    (N x T) and ``x`` (T x M, dense) in place and returns ``(replaced, e)``
    with e = Y - D X after the refits.

    E starts as the reference's own product ``y - d @ x``; the per-atom loop
    runs on the device.  Atom signs follow the largest-magnitude-entry-
    positive convention (the reference's LAPACK SVD sign is arbitrary;
    products d_j x_j and E do not depend on it)."""
    y = np.asarray(y, dtype=np.float64)
    n, m = y.shape
    t = d.shape[1]
    e = y - d @ x
    jj, pp = np.nonzero(x)  # by atom, then ascending signal: np.flatnonzero(x[j])
    vals = np.ascontiguousarray(x[jj, pp], dtype=np.float64)
    counts = np.bincount(jj, minlength=t)
    ptr = np.zeros(t + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    sig = np.ascontiguousarray(pp, dtype=np.int64)
    y_rows = np.ascontiguousarray(y.T)
    e_rows = np.ascontiguousarray(e.T)
    d_rows = np.ascontiguousarray(np.asarray(d, dtype=np.float64).T)
    replaced = np.zeros(1, dtype=np.int64)
    _N.check(_N.load().cdb_ksvd_update(n, m, t, _N.ptr(y_rows), _N.ptr(e_rows), _N.ptr(d_rows),
                                       _N.ptr(ptr), _N.ptr(sig), _N.ptr(vals), int(vals.size),
                                       int(counts.max()) if t else 0, int(threshold),
                                       _N.ptr(replaced), None))
    d[...] = d_rows.T
    x[jj, pp] = vals
    return int(replaced[0]), np.ascontiguousarray(e_rows.T)


# ---------------------------------------------------------------- training loop
# K-SVD with both stages on the device (mirror of crossdict learn.py:44-331).
# Hyper-parameters, initialisation, duplicate cleanup and the report follow
# the reference; the codes, the residual E = Y - D X and the rank-one refits
# stay in HBM across the stages (the reference materialises a dense T x M
# code matrix and re-forms E on the host every iteration).

@dataclass(frozen=True)
class TrainConfig:
    """K-SVD hyperparameters (learn.py:44-61)."""

    num_atoms: int
    sparsity: int
    iterations: int = 20
    seed: int = 0
    dead_atom_threshold: int = 1
    init: str = "data-columns"

    def __post_init__(self):
        if self.num_atoms < 1 or self.sparsity < 1 or self.iterations < 1:
            raise E.ConfigError("num_atoms, sparsity and iterations must be >= 1")
        if self.dead_atom_threshold < 0:
            raise E.ConfigError("dead_atom_threshold must be >= 0")
        if self.init not in ("data-columns", "random-unit"):
            raise E.ConfigError(f"unknown init {self.init!r}")


@dataclass
class TrainReport:
    """Objective trace of one run (learn.py:64-76): after / before each update."""

    objective_per_iteration: list = field(default_factory=list)
    objective_pre_update: list = field(default_factory=list)
    replaced_atoms: int = 0
    wall_clock: float = 0.0


report_log: list = []  # every run's report (learn.py:80)
_types: dict = {}       # install(): the reference's Dictionary / TrainReport / report_log

_INIT_COHERENCE_CAP = 0.7   # learn.py:92
_DUPLICATE_COHERENCE = 0.99  # learn.py:95


def _validate_samples(samples) -> np.ndarray:
    y = np.asarray(samples, dtype=np.float64)
    if y.ndim != 2:
        raise E.DimensionError(f"samples must be an N x P matrix, got ndim={y.ndim}")
    if not np.any(y):
        raise E.DegenerateDataError("all training samples are zero")
    return y


def init_atoms(y, config: TrainConfig, rng) -> np.ndarray:
    """Starting dictionary (learn.py:98-128): distinct data columns, skipping
    candidates more coherent than 0.7 with the atoms already chosen, then the
    skipped ones, then random unit vectors; or random unit columns."""
    n, m = y.shape
    t = config.num_atoms
    if config.init == "random-unit":
        g = rng.standard_normal((n, t))
        return g / np.linalg.norm(g, axis=0)
    norms = np.linalg.norm(y, axis=0)
    order = rng.permutation(np.flatnonzero(norms > 0))
    atoms = np.empty((t, n))
    filled = 0
    used = np.zeros(order.size, dtype=bool)
    for pos, c in enumerate(order):
        v = y[:, c] / norms[c]
        if filled and np.abs(atoms[:filled] @ v).max() > _INIT_COHERENCE_CAP:
            continue
        atoms[filled] = v
        filled += 1
        used[pos] = True
        if filled == t:
            break
    for pos, c in enumerate(order):
        if filled == t:
            break
        if not used[pos]:
            atoms[filled] = y[:, c] / norms[c]
            filled += 1
    while filled < t:
        v = rng.standard_normal(n)
        atoms[filled] = v / np.linalg.norm(v)
        filled += 1
    return np.ascontiguousarray(atoms.T)


def cleanup_duplicates(y, d, resid_norms) -> int:
    """Re-seed atoms collapsed onto an earlier atom (learn.py:201-228)."""
    t = d.shape[1]
    gram = np.abs(d.T @ d)
    np.fill_diagonal(gram, 0.0)
    taken: set = set()
    replaced = 0
    for j in range(t):
        if gram[:j, j].max(initial=0.0) <= _DUPLICATE_COHERENCE:
            continue
        rn = np.array(resid_norms, dtype=np.float64)
        if taken:
            rn[list(taken)] = -1.0
        worst = int(np.argmax(rn))
        taken.add(worst)
        cn = np.linalg.norm(y[:, worst])
        if cn > 0:
            d[:, j] = y[:, worst] / cn
        gram[j, :] = 0.0
        gram[:, j] = 0.0
        replaced += 1
    return replaced


def _code_device(d, yrows, eps, k, block_hint, outs):
    """The coding stage into device arrays: full OMP, or the ragged
    block-restricted call for the block hint (as code_stage)."""
    n, t = d.shape
    m = yrows.shape[0]
    dd = _dev.DeviceDictionary(np.ascontiguousarray(d.T))
    if block_hint is None:
        return _dev.omp_batch_raw(dd, yrows, m, k, eps, None, _pursuit.ENGINE, outs)
    blocks, nb, q = block_hint
    nb_max = int(blocks.shape[1])
    k_out = int(max(1, min(k, nb_max * q, n)))
    return _dev.omp_batch_blocked_ragged_raw(dd, yrows, m, k_out, eps, blocks, nb, int(q),
                                             _pursuit.ENGINE, outs[k_out])


def _codes_to_device(results, k, outs):
    """Per-sample PursuitResults (1-based picks in pick order) -> device arrays."""
    import torch
    m = len(results)
    sel = np.full((m, k), -1, dtype=np.int64)
    coef = np.zeros((m, k))
    for p, r in enumerate(results):
        idx = np.asarray(r.code.support, dtype=np.int64) - 1
        sel[p, :idx.size] = idx
        coef[p, :idx.size] = r.code.coefficients
    outs["sel"].copy_(torch.from_numpy(sel))
    outs["alpha"].copy_(torch.from_numpy(coef))
    return outs


def ksvd_core(y, config: TrainConfig, allowed_sets, block_hint):
    """K-SVD iterations (learn.py:265-288) with device-resident stages;
    returns (Dictionary, codes, TrainReport) like the reference."""
    import torch
    start = time.perf_counter()
    n, m = y.shape
    t, k = config.num_atoms, config.sparsity
    if t > m:
        raise E.ConfigError(f"num_atoms {t} exceeds sample count {m}")
    if k > min(n, t):
        raise E.ConfigError(f"sparsity {k} exceeds min(N, T) = {min(n, t)}")
    rng = np.random.default_rng(config.seed)
    d = init_atoms(y, config, rng)
    report = _types.get("TrainReport", TrainReport)()
    dev = "cuda"
    yrows = torch.from_numpy(np.ascontiguousarray(y.T)).to(dev)
    eps = torch.from_numpy(_pursuit._rel_tol() * np.linalg.norm(y, axis=0)).to(dev)
    hint = None
    widths = {k}
    if block_hint is not None:
        blocks_list, q = block_hint
        nb = np.array([len(b) for b in blocks_list], dtype=np.int64)
        nb_max = max(1, int(nb.max()))
        blocks = np.zeros((m, nb_max), dtype=np.int64)
        for p, b in enumerate(blocks_list):
            if len(b):
                blocks[p, :len(b)] = sorted(b)
        hint = (torch.from_numpy(blocks).to(dev), torch.from_numpy(nb).to(dev), int(q))
        widths = {int(max(1, min(k, nb_max * q, n)))}

    def outs_for(kk):
        mk = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)  # noqa: E731
        return dict(sel=mk((m, kk), torch.int64), alpha=mk((m, kk), torch.float64),
                    counts=mk((m,), torch.int64), rnorm=mk((m,), torch.float64),
                    scans=mk((m,), torch.int64), flag=mk((m,), torch.uint8))
    outs = {kk: outs_for(kk) for kk in widths}
    o = None
    for it in range(config.iterations):
        if allowed_sets is not None and block_hint is None:  # arbitrary per-sample sets
            o = _codes_to_device(code_stage(d, y, k, allowed_sets, None), k, outs[k])
        else:
            o = _code_device(d, yrows, eps, k, hint, outs if hint is not None else outs[k])
        sel, coef = o["sel"], o["alpha"]
        drows = torch.from_numpy(np.ascontiguousarray(d.T)).to(dev)
        valid = (sel >= 0) & (coef != 0.0)
        selc = sel.clamp(min=0)
        e = yrows.clone()
        for l in range(sel.shape[1]):  # E = Y - D X, one support slot at a time
            e -= torch.where(valid[:, l, None], coef[:, l, None] * drows[selc[:, l]], 0.0)
        report.objective_pre_update.append(float(torch.linalg.norm(e)))
        pp, ll = torch.nonzero(valid, as_tuple=True)
        atoms = sel[pp, ll]
        order = torch.argsort(atoms * m + pp)
        pp, ll, atoms = pp[order], ll[order], atoms[order]
        vals = coef[pp, ll].contiguous()
        counts = torch.bincount(atoms, minlength=t)
        ptr = torch.zeros(t + 1, dtype=torch.int64, device=dev)
        ptr[1:] = torch.cumsum(counts, 0)
        sig = pp.contiguous()
        replaced = np.zeros(1, dtype=np.int64)
        _N.check(_N.load().cdb_ksvd_update(
            n, m, t, _N.ptr(yrows), _N.ptr(e), _N.ptr(drows), _N.ptr(ptr), _N.ptr(sig),
            _N.ptr(vals), int(vals.numel()), int(counts.max()) if t else 0,
            int(config.dead_atom_threshold), _N.ptr(replaced), None))
        coef[pp, ll] = vals
        report.replaced_atoms += int(replaced[0])
        report.objective_per_iteration.append(float(torch.linalg.norm(e)))
        d = np.ascontiguousarray(drows.cpu().numpy().T)
        if it + 1 < config.iterations:
            report.replaced_atoms += cleanup_duplicates(
                y, d, torch.linalg.norm(e, dim=1).cpu().numpy())
    sel_h, coef_h = o["sel"].cpu().numpy(), o["alpha"].cpu().numpy()
    sc = _pursuit._types["SparseCode"]
    # entries sorted by atom per sample, vectorised (the reference's
    # _codes_from_matrix order, learn.py:231-237); only the objects are per sample
    keep = (sel_h >= 0) & (coef_h != 0.0)
    key = np.where(keep, sel_h, np.iinfo(np.int64).max)
    order = np.argsort(key, axis=1, kind="stable")
    ids = (np.take_along_axis(sel_h, order, axis=1) + 1).tolist()
    vals = np.take_along_axis(coef_h, order, axis=1).tolist()
    cnt = keep.sum(axis=1).tolist()
    codes = [sc(t, tuple(zip(ids[p][:cnt[p]], vals[p][:cnt[p]]))) for p in range(m)]
    report.wall_clock = time.perf_counter() - start
    _types.get("report_log", report_log).append(report)
    return _types.get("Dictionary", _tensor.Dictionary)(d), codes, report


def ksvd(samples, config: TrainConfig):
    """K-SVD (learn.py:291-300) with the device stages."""
    return ksvd_core(_validate_samples(samples), config, None, None)


def ksvd_constrained(samples, per_sample_allowed_support, config: TrainConfig, *,
                     block_hint=None):
    """Support-constrained K-SVD (learn.py:303-331); the device path needs
    ``block_hint`` (the two-scale trainer always passes it)."""
    y = _validate_samples(samples)
    m = y.shape[1]
    t = config.num_atoms
    sets = [frozenset(int(i) for i in s) for s in per_sample_allowed_support]
    if len(sets) != m:
        raise E.ConfigError(f"need {m} allowed sets, got {len(sets)}")
    for p, s in enumerate(sets):
        if not s:
            raise E.ConfigError(f"sample {p + 1} has an empty allowed support")
        if min(s) < 1 or max(s) > t:
            raise E.ConfigError(f"sample {p + 1} allowed support outside [1, {t}]")
    if all(len(s) == t for s in sets):
        return ksvd_core(y, config, None, None)
    return ksvd_core(y, config, sets, block_hint)


def train_cross_scale(samples, scale, t_low: int, t_high: int, k_low: int, k_high: int,
                      iterations: int = 20, seed: int = 0, dead_atom_threshold: int = 1,
                      init: str = "data-columns"):
    """Two-step cross-scale training (learn.py:334-379): K-SVD on the
    block-averaged samples, then block-restricted K-SVD at full resolution
    (each sample confined to its coarse support's children; an empty coarse
    code gets block 1 as placeholder).  Returns ``(model, (low, high))``."""
    from .crossscale import CrossScaleModel, cross_scale_map
    from .scaling import downsample_columns
    y = _validate_samples(samples)
    if t_low < 1 or t_high % t_low:
        raise E.ConfigError(f"t_high={t_high} must be a positive multiple of t_low={t_low}")
    q = t_high // t_low
    if y.shape[0] != scale.fine_size:
        raise E.DimensionError(f"sample length {y.shape[0]} != fine patch size {scale.fine_size}")
    y_low = downsample_columns(y, scale)
    cfg_low = TrainConfig(t_low, k_low, iterations, seed, dead_atom_threshold, init)
    d_low, codes_low, report_low = ksvd(y_low, cfg_low)
    blocks_list, allowed_sets = [], []
    for code in codes_low:
        sup = code.support if code.support else (1,)
        blocks_list.append([i - 1 for i in sup])
        allowed_sets.append(cross_scale_map(sup, q, t_high))
    cfg_high = TrainConfig(t_high, k_high, iterations, seed, dead_atom_threshold, init)
    d_high, _, report_high = ksvd_constrained(y, allowed_sets, cfg_high,
                                              block_hint=(blocks_list, q))
    model = CrossScaleModel(d_low, d_high, scale, k_low, k_high)
    return model, (report_low, report_high)
