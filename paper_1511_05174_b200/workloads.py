"""Seeded synthetic workloads for the five BASELINE.json configurations.

The reference measures on synthetic data only (``BASELINE.json`` configs,
SURVEY.md §8(d)); no dataset ships with it.  This module is the generator
that SURVEY §8(d) specifies, written for this repo:

* ``D_low``: N_low x T_low iid N(0,1) columns, unit-normalised.
* child ``j*Q + c`` of coarse atom ``j``: ``normalize(U d_low_j + 0.3 * N(0,1)^N)``
  where ``U`` is the nearest-neighbour upsample of the reference
  (``scaling.py:119-131``).  The 0.3 applies per fine entry before the
  normalisation (recorded interpretation).
* signals: K distinct parents uniform over ``T_low``, one uniform child each,
  coefficients N(0,1), ``y = D_high x + sigma * N(0,1)^N``.
* cfg 3 (light-field CS): ``Phi`` is 256 x 1024 with N(0, 1/256) entries,
  ``y = Phi D_high x + 0.01 N(0,1)^256``; OMP runs on the effective
  dictionaries ``E_high = Phi D_high`` and ``E_low = Phi U D_low`` (the
  reference's ``zero_tree_omp(phi=...)`` semantics, ``crossscale.py:194-220``).

Precision contract: every array is rounded to fp32 first
(the GPU's input precision); unit-norm dictionaries are then re-normalised in
fp64 so that the reference ``Dictionary`` accepts them (``tensor.py:102-107``).
The fp64 arrays returned here are exactly what both the GPU path and the CPU
oracle consume.

Signals are produced in independent blocks (``BLOCK`` signals, RNG stream
``(seed, 1, block)``) so that any rank can generate just its own shard.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

BLOCK = 256


@dataclass(frozen=True)
class Workload:
    name: str
    fine_shape: tuple
    factors: tuple
    t_low: int
    q: int
    k: int
    signals: int
    sigma: float
    measurements: int = 0  # >0: dense compressive-sensing operator (cfg 3)

    @property
    def n_high(self) -> int:
        return int(np.prod(self.fine_shape))

    @property
    def n_low(self) -> int:
        return int(np.prod([e // f for e, f in zip(self.fine_shape, self.factors)]))

    @property
    def t_high(self) -> int:
        return self.t_low * self.q

    @property
    def n_signal(self) -> int:
        """Length of each coded signal (M for the CS config, else N_high)."""
        return self.measurements or self.n_high


# BASELINE.json "configs", in order.
CONFIGS = (
    Workload("image", (8, 8), (2, 2), 64, 4, 8, 10_000, 0.01),
    Workload("video", (8, 8, 4), (2, 2, 2), 256, 8, 16, 100_000, 0.01),
    Workload("hyperspectral", (8, 8, 16), (2, 2, 2), 512, 8, 32, 200_000, 0.02),
    Workload("lightfield_cs", (8, 8, 4, 4), (2, 2, 2, 2), 256, 16, 24, 100_000, 0.01, 256),
    Workload("large", (16, 16, 16), (2, 2, 2), 2048, 8, 64, 1_000_000, 0.01),
)

#: stopping rule of every BASELINE config: K atoms or ||r|| <= 1e-3 ||y||
REL_TOL = 1e-3


def upsample_rows(low: np.ndarray, fine_shape, factors) -> np.ndarray:
    """Nearest-neighbour upsample of row-major coarse patches, one per ROW.

    Same map as the reference ``upsample_columns`` (``scaling.py:119-131``)
    but with signals as rows.
    """
    coarse = tuple(e // f for e, f in zip(fine_shape, factors))
    arr = low.reshape((low.shape[0],) + coarse)
    for axis, f in enumerate(factors):
        if f > 1:
            arr = np.repeat(arr, f, axis=axis + 1)
    return np.ascontiguousarray(arr.reshape(low.shape[0], -1))


def _unit_rows(m: np.ndarray) -> np.ndarray:
    return m / np.linalg.norm(m, axis=1, keepdims=True)


def _round_unit(rows64: np.ndarray) -> np.ndarray:
    """fp32 rounding, then fp64 re-normalisation."""
    r32 = rows64.astype(np.float32).astype(np.float64)
    return _unit_rows(r32)


@dataclass
class Dictionaries:
    """Atoms as ROWS (T x N, the reference's ``atoms_t`` layout)."""

    low_t: np.ndarray    # T_low x N_low  (identity step-1 dictionary)
    high_t: np.ndarray   # T_high x N_high
    phi: np.ndarray | None = None       # M x N_high (cfg 3)
    e_low_t: np.ndarray | None = None   # T_low x M  (Phi U D_low)
    e_high_t: np.ndarray | None = None  # T_high x M (Phi D_high)


@lru_cache(maxsize=4)
def dictionaries(cfg_index: int, seed: int = 0) -> Dictionaries:
    w = CONFIGS[cfg_index]
    rng = np.random.default_rng([seed, 0, cfg_index])
    low = _unit_rows(rng.standard_normal((w.t_low, w.n_low)))
    up = upsample_rows(low, w.fine_shape, w.factors)
    high = np.repeat(up, w.q, axis=0) + 0.3 * rng.standard_normal((w.t_high, w.n_high))
    low_t = _round_unit(low)
    high_t = _round_unit(_unit_rows(high))
    out = Dictionaries(low_t=low_t, high_t=high_t)
    if w.measurements:
        phi = rng.standard_normal((w.measurements, w.n_high)) / np.sqrt(w.measurements)
        phi = phi.astype(np.float32).astype(np.float64)
        out.phi = phi
        out.e_high_t = (high_t @ phi.T).astype(np.float32).astype(np.float64)
        out.e_low_t = (upsample_rows(low_t, w.fine_shape, w.factors) @ phi.T).astype(
            np.float32).astype(np.float64)
    for a in (out.low_t, out.high_t, out.phi, out.e_low_t, out.e_high_t):
        if a is not None:
            a.setflags(write=False)
    return out


def signal_block(cfg_index: int, block: int, seed: int = 0, count: int | None = None):
    """Signals of block ``block`` as ROWS (count x n_signal), fp32-exact fp64.

    Returns ``(ys_rows, atoms, coefs)`` where ``atoms``/``coefs`` (count x K)
    are the planted fine atoms and coefficients.
    """
    w = CONFIGS[cfg_index]
    d = dictionaries(cfg_index, seed)
    count = BLOCK if count is None else count
    rng = np.random.default_rng([seed, 1, cfg_index, block])
    parents = np.argsort(rng.random((count, w.t_low)), axis=1)[:, : w.k]
    child = rng.integers(0, w.q, size=(count, w.k))
    atoms = parents * w.q + child
    coefs = rng.standard_normal((count, w.k))
    x_sig = np.zeros((count, w.n_high))
    for j in range(w.k):
        x_sig += coefs[:, j, None] * d.high_t[atoms[:, j]]
    if w.measurements:
        y = x_sig @ d.phi.T + w.sigma * rng.standard_normal((count, w.measurements))
    else:
        y = x_sig + w.sigma * rng.standard_normal((count, w.n_high))
    return y.astype(np.float32).astype(np.float64), atoms, coefs


def signals(cfg_index: int, start: int, stop: int, seed: int = 0) -> np.ndarray:
    """Signals ``start:stop`` of the config's deterministic stream, as ROWS."""
    out = []
    if stop <= start:
        return np.zeros((0, CONFIGS[cfg_index].n_signal))
    for b in range(start // BLOCK, (stop - 1) // BLOCK + 1):
        ys, _, _ = signal_block(cfg_index, b, seed)
        lo = max(start - b * BLOCK, 0)
        hi = min(stop - b * BLOCK, BLOCK)
        out.append(ys[lo:hi])
    if not out:
        return np.zeros((0, CONFIGS[cfg_index].n_signal))
    return np.ascontiguousarray(np.concatenate(out, axis=0))


def subset_indices(cfg_index: int, count: int, seed: int = 7) -> np.ndarray:
    """Seeded sorted subset of signal ids (the parity / CPU-baseline subsets)."""
    w = CONFIGS[cfg_index]
    rng = np.random.default_rng([seed, 2, cfg_index])
    return np.sort(rng.choice(w.signals, size=min(count, w.signals), replace=False))


def signals_at(cfg_index: int, ids, seed: int = 0) -> np.ndarray:
    """Rows for arbitrary signal ids (groups ids by generation block)."""
    ids = np.asarray(ids, dtype=np.int64)
    w = CONFIGS[cfg_index]
    out = np.zeros((ids.size, w.n_signal))
    for b in np.unique(ids // BLOCK):
        sel = np.flatnonzero(ids // BLOCK == b)
        ys, _, _ = signal_block(cfg_index, int(b), seed)
        out[sel] = ys[ids[sel] - b * BLOCK]
    return out


#: signals per device-generation block (``signals_device``)
DEVICE_BLOCK = 65536


def _block_seed(seed: int, cfg_index: int, block: int) -> int:
    return int(np.random.default_rng([seed, 3, cfg_index, block]).integers(0, 2**62))


def signals_device(cfg_index: int, start: int, stop: int, seed: int = 0, device="cuda"):
    """Signals ``start:stop`` of the config's DEVICE stream, as fp32 ROWS on ``device``.

    Same distribution as ``signal_block`` (K distinct parents uniform over
    T_low, one uniform child each, N(0,1) coefficients, sigma noise; Phi for
    the CS config), drawn with torch's device generator in independent blocks
    of ``DEVICE_BLOCK`` signals seeded from ``(seed, cfg, block)`` -- so any rank
    generates just its own shard and the stream does not depend on the
    sharding.  At cfg 4's full size (1M x 4096) the host stream
    (``signals``) takes ~12 min; this takes seconds.  It is a different
    stream from ``signals``: parity tests copy the rows they check back to
    the host and feed exactly those to the oracle.
    """
    import torch
    w = CONFIGS[cfg_index]
    d = dictionaries(cfg_index, seed)
    dev = torch.device(device)
    dh = torch.from_numpy(np.array(d.high_t)).to(dev)
    phi_t = torch.from_numpy(np.array(d.phi)).to(dev).T.contiguous() if w.measurements else None
    out = torch.empty((max(stop - start, 0), w.n_signal), dtype=torch.float32, device=dev)
    if stop <= start:
        return out
    sub = max(1, min(DEVICE_BLOCK, (512 << 20) // (8 * w.n_high)))
    for b in range(start // DEVICE_BLOCK, (stop - 1) // DEVICE_BLOCK + 1):
        g = torch.Generator(device=dev)
        g.manual_seed(_block_seed(seed, cfg_index, b))
        parents = torch.topk(torch.rand((DEVICE_BLOCK, w.t_low), generator=g, device=dev), w.k,
                             dim=1, largest=False).indices
        atoms = parents * w.q + torch.randint(0, w.q, (DEVICE_BLOCK, w.k), generator=g, device=dev)
        coefs = torch.randn((DEVICE_BLOCK, w.k), generator=g, device=dev, dtype=torch.float64)
        lo = max(start - b * DEVICE_BLOCK, 0)
        hi = min(stop - b * DEVICE_BLOCK, DEVICE_BLOCK)
        for s in range(0, DEVICE_BLOCK, sub):
            e = min(s + sub, DEVICE_BLOCK)
            # noise is drawn for every sub-block so the stream is independent of lo/hi
            noise = torch.randn((e - s, w.n_signal), generator=g, device=dev, dtype=torch.float64)
            if e <= lo or s >= hi:
                continue
            x = torch.zeros((e - s, w.n_high), dtype=torch.float64, device=dev)
            for j in range(w.k):
                x += coefs[s:e, j, None] * dh[atoms[s:e, j]]
            if phi_t is not None:
                x = x @ phi_t
            x += w.sigma * noise
            a, z = max(lo, s), min(hi, e)
            out[b * DEVICE_BLOCK + a - start: b * DEVICE_BLOCK + z - start] = x[a - s: z - s].float()
    return out
