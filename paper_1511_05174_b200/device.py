"""Device-resident dictionaries and the raw batched calls (C ABI wrappers).

A dictionary enters the path as ``atoms_t`` (T x N fp64, the reference's
kernel operand, crossdict/tensor.py:124-129).  ``device_dictionary`` stages it
once per array (identity for read-only arrays such as ``Dictionary.atoms_t``,
content digest for writable ones) and keeps the handle cached, so repeated
calls -- K-SVD coding stages, pipelines over many images -- pay the upload,
bf16 conversion and Gram build once.

Every array argument of the ``*_raw`` calls may be a host numpy array or a
CUDA tensor (anything with ``data_ptr()``); the library stages host memory.
"""

from __future__ import annotations

import ctypes
import weakref
from collections import OrderedDict

import numpy as np

from . import _native as N

#: build the fp64 Gram matrix when T*T*8 bytes fit this budget
GRAM_BUDGET_BYTES = 4 << 30
#: number of staged dictionaries kept alive
CACHE_ENTRIES = 8


class DeviceDictionary:
    """Opaque ``cdb_dictionary`` handle (fp64 atoms, bf16 operand, fp64 Gram)."""

    def __init__(self, atoms_t: np.ndarray, gram_budget: int = GRAM_BUDGET_BYTES):
        atoms_t = np.ascontiguousarray(atoms_t, dtype=np.float64)
        self.t, self.n = atoms_t.shape
        self._handle = ctypes.c_void_p()
        self._lib = N.load()
        N.check(self._lib.cdb_dictionary_create(N.ptr(atoms_t), self.t, self.n, int(gram_budget),
                                                None, ctypes.byref(self._handle)))

    @property
    def handle(self):
        return self._handle

    @property
    def nbytes(self) -> int:
        return int(self._lib.cdb_dictionary_bytes(self._handle))

    def close(self):
        if self._handle:
            self._lib.cdb_dictionary_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache: "OrderedDict[tuple, tuple]" = OrderedDict()


def _current_device() -> int:
    try:
        import torch
        return torch.cuda.current_device() if torch.cuda.is_available() else -1
    except Exception:
        return -1


def _host_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Exact comparison of two host arrays; same-layout fp64 blocks go through
    the library's multi-threaded memcmp (512 MB in tens of milliseconds; a bit
    pattern that differs, -0.0 against 0.0 included, only costs a re-staging)."""
    if (a.shape == b.shape and a.dtype == b.dtype and a.flags.c_contiguous
            and b.flags.c_contiguous and a.nbytes >= (1 << 22)):
        return bool(N.load().cdb_host_equal(N.ptr(a), N.ptr(b), a.nbytes, 0))
    return np.array_equal(a, b)


def _sample(flat: np.ndarray) -> tuple:
    return tuple(float(flat[i]) for i in (0, flat.size // 3, flat.size // 2, flat.size - 1)) \
        if flat.size else ()


def device_dictionary_cols(mat: np.ndarray) -> DeviceDictionary:
    """Cached device staging of an N x T column matrix (the reference's
    `columns`, pursuit.py:84-94) without the host transpose on a hit: the entry
    is found by a few sampled values and confirmed against the stored host copy
    of `mat` itself; on a miss the T x N rows come from the library's threaded
    transpose."""
    data = np.ascontiguousarray(mat, dtype=np.float64)
    dev = _current_device()
    key = ("cols", dev, data.shape, _sample(data.reshape(-1)))
    hit = _cache.get(key)
    if hit is not None and _host_equal(hit[2], data):
        _cache.move_to_end(key)
        return hit[1]
    n, t = data.shape
    rows = np.empty((t, n), dtype=np.float64)
    if data.size:
        N.check(N.load().cdb_rows_from_cols(N.ptr(data), n, t, 8, N.ptr(rows), 0))
    dd = DeviceDictionary(rows)
    _cache[key] = ((lambda: None), dd, data.copy())
    while len(_cache) > CACHE_ENTRIES:
        _cache.popitem(last=False)[1][1].close()
    return dd


def device_dictionary(atoms_t: np.ndarray) -> DeviceDictionary:
    """Cached device staging of a T x N atom-row matrix (per CUDA device)."""
    atoms_t = np.asarray(atoms_t)
    dev = _current_device()
    if not atoms_t.flags.writeable:
        key = ("ro", dev, id(atoms_t), atoms_t.shape)
        hit = _cache.get(key)
        if hit is not None and hit[0]() is atoms_t:
            _cache.move_to_end(key)
            return hit[1]
        ref = weakref.ref(atoms_t)
    else:
        # writeable (so mutable) arrays: a few sampled values find the entry and
        # an exact comparison with the stored host copy confirms it -- no false
        # hits, ~10 us instead of hashing the whole matrix on every call
        data = np.ascontiguousarray(atoms_t, dtype=np.float64)
        flat = data.reshape(-1)
        key = ("rw", dev, data.shape, _sample(flat))
        hit = _cache.get(key)
        if hit is not None and _host_equal(hit[2], data):
            _cache.move_to_end(key)
            return hit[1]
        ref = (lambda: None)
        dd = DeviceDictionary(data)
        _cache[key] = (ref, dd, data.copy())
        while len(_cache) > CACHE_ENTRIES:
            _cache.popitem(last=False)[1][1].close()
        return dd
    dd = DeviceDictionary(atoms_t)
    _cache[key] = (ref, dd)
    while len(_cache) > CACHE_ENTRIES:
        _cache.popitem(last=False)[1][1].close()
    return dd


def clear_cache():
    while _cache:
        _cache.popitem(last=False)[1][1].close()


# Batches at least this large use page-locked host staging: the library then
# pipelines chunked H2D / compute / D2H; pageable buffers would make every
# copy host-synchronous (api.cu run_pipelined).
PIN_MIN = 4096


def pinned_empty(shape, dtype):
    """Page-locked numpy array (torch's caching host allocator keeps the block
    alive through the array's base and reuses it after release)."""
    import torch
    if not torch.cuda.is_available():  # staging only: plain memory is equally correct
        return np.empty(shape, dtype)
    t = torch.empty(shape, dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True)
    return t.numpy()


def rows_for_device(ys_cols):
    """The reference's N x P column batch as contiguous P x N rows -- the copy
    the drop-in makes anyway -- written into pinned memory for large batches."""
    ys_cols = np.asarray(ys_cols)
    n, p = ys_cols.shape
    if ys_cols.T.flags.c_contiguous:  # already rows (e.g. extract_patches output)
        return ys_cols.T
    if p < PIN_MIN or ys_cols.dtype not in (np.float32, np.float64):
        return np.ascontiguousarray(ys_cols.T)
    src = np.ascontiguousarray(ys_cols)
    dst = pinned_empty((p, n), src.dtype)
    N.check(N.load().cdb_rows_from_cols(N.ptr(src), n, p, src.itemsize, N.ptr(dst), 0))
    return dst


def _out(p, k):
    mk = pinned_empty if p >= PIN_MIN else np.empty
    return dict(sel=mk((p, k), np.int64), alpha=mk((p, k), np.float64),
                counts=mk((p,), np.int64), rnorm=mk((p,), np.float64),
                scans=mk((p,), np.int64), flag=mk((p,), np.uint8))


_OUT_DTYPES = (("sel", np.int64), ("alpha", np.float64), ("counts", np.int64),
               ("rnorm", np.float64), ("scans", np.int64), ("flag", np.uint8))


def _is_tensor(a) -> bool:
    return hasattr(a, "data_ptr") and hasattr(a, "is_contiguous")


def _check_tensor(a, dtypes, name):
    import torch
    allowed = [getattr(torch, np.dtype(d).name) for d in dtypes]
    if a.dtype not in allowed:
        raise TypeError(f"{name}: tensor dtype {a.dtype}, expected one of {allowed}")
    if not a.is_contiguous():
        raise TypeError(f"{name}: tensor must be contiguous")


def _arg(a, dtype, name):
    """(keepalive, pointer) of an input array: numpy arrays are converted to a
    C-contiguous ``dtype`` copy when needed (the caller keeps the returned
    object alive across the C call); tensors must already match."""
    if a is None:
        return None, None
    if _is_tensor(a):
        _check_tensor(a, (dtype,), name)
        return a, N.ptr(a)
    c = np.ascontiguousarray(a, dtype=dtype)
    return c, N.ptr(c)


def _out_ptrs(o):
    ptrs = []
    for k, dt in _OUT_DTYPES:
        a = o[k]
        if _is_tensor(a):
            _check_tensor(a, (dt,), k)
        elif not (isinstance(a, np.ndarray) and a.dtype == dt and a.flags.c_contiguous
                  and a.flags.writeable):
            raise TypeError(f"output {k!r} must be a writeable C-contiguous {np.dtype(dt).name} array")
        ptrs.append(N.ptr(a))
    return ptrs


def _ys_arg(ys):
    """(keepalive, pointer, is_f32) for fp32/fp64 signal rows (numpy or tensor).
    Other numpy dtypes are converted to fp64; tensors must be contiguous fp32
    or fp64 (read as raw rows by the library)."""
    if _is_tensor(ys):
        _check_tensor(ys, (np.float32, np.float64), "ys")
        import torch
        return ys, N.ptr(ys), 1 if ys.dtype == torch.float32 else 0
    ys = np.asarray(ys)
    c = np.ascontiguousarray(ys, dtype=np.float32 if ys.dtype == np.float32 else np.float64)
    return c, N.ptr(c), 1 if c.dtype == np.float32 else 0


def omp_batch_raw(dd: DeviceDictionary, ys, p: int, k_max: int, eps, allowed=None,
                  engine: str = "auto", out=None, stream=None):
    """cdb_omp_batch: signals as rows; returns the BatchSolve arrays (dict)."""
    o = out if out is not None else _out(p, k_max)
    yk, yptr, f32 = _ys_arg(ys)
    ek, eptr = _arg(eps, np.float64, "eps")
    ak, aptr = _arg(allowed, np.int64, "allowed")
    s = 0 if allowed is None else int(allowed.shape[1])
    N.check(N.load().cdb_omp_batch(dd.handle, yptr, f32, p, k_max, eptr, aptr, s,
                                   0 if allowed is None else 1, *_out_ptrs(o),
                                   N.ENGINES[engine], stream))
    del yk, ek, ak
    return o


def omp_batch_blocked_raw(dd: DeviceDictionary, ys, p: int, k_max: int, eps, blocks, q: int,
                          engine: str = "auto", out=None, stream=None):
    """cdb_omp_batch_blocked: allowed = blocks * q + [0, q)."""
    o = out if out is not None else _out(p, k_max)
    yk, yptr, f32 = _ys_arg(ys)
    ek, eptr = _arg(eps, np.float64, "eps")
    bk, bptr = _arg(blocks, np.int64, "blocks")
    N.check(N.load().cdb_omp_batch_blocked(dd.handle, yptr, f32, p, k_max, eptr, bptr,
                                           int(blocks.shape[1]), int(q),
                                           *_out_ptrs(o), N.ENGINES[engine], stream))
    del yk, ek, bk
    return o


def zero_tree_raw(low: DeviceDictionary, high: DeviceDictionary, fine_shape, factors, ys,
                  p: int, k1: int, k_high: int, rel_tol: float, phi_mode: bool,
                  engine: str = "auto", out_low=None, out_high=None, stream=None):
    """cdb_zero_tree_batch; returns (low dict, high dict, [step1_ms, step2_ms])."""
    lo = out_low if out_low is not None else _out(p, k1)
    hi = out_high if out_high is not None else _out(p, k_high)
    fs = np.asarray(fine_shape if fine_shape is not None else [1], dtype=np.int64)
    fa = np.asarray(factors if factors is not None else [1], dtype=np.int64)
    ms = np.zeros(2, np.float32)
    yk, yptr, f32 = _ys_arg(ys)
    N.check(N.load().cdb_zero_tree_batch(low.handle, high.handle, N.ptr(fs), N.ptr(fa), int(fs.size),
                                         yptr, f32, p, k1, k_high, float(rel_tol), int(phi_mode),
                                         *_out_ptrs(lo), *_out_ptrs(hi), N.ENGINES[engine],
                                         N.ptr(ms), stream))
    del yk
    return lo, hi, ms


def cols_layout(ys_cols):
    """True when an N x P batch can cross the ABI as columns as it is: a
    float32 / float64 numpy array with unit stride along P (the reference's
    own layout); batches that already are rows in memory (ys.T C-contiguous)
    take the rows path."""
    a = ys_cols
    return (isinstance(a, np.ndarray) and a.ndim == 2 and a.dtype in (np.float32, np.float64)
            and a.shape[1] >= PIN_MIN and not a.T.flags.c_contiguous
            and a.strides[1] == a.itemsize and a.strides[0] % a.itemsize == 0
            and a.strides[0] // a.itemsize >= a.shape[1])


def omp_cols_raw(dd: DeviceDictionary, ys_cols, k_max: int, eps=None, rel_tol: float = 0.0,
                 engine: str = "auto", out=None, stream=None):
    """cdb_omp_batch_cols: the N x P column batch as the reference holds it
    (host memory); eps None -> rel_tol * |y| per signal on the device."""
    p = int(ys_cols.shape[1])
    o = out if out is not None else _out(p, k_max)
    ek, eptr = _arg(eps, np.float64, "eps")
    ld = ys_cols.strides[0] // ys_cols.itemsize
    N.check(N.load().cdb_omp_batch_cols(dd.handle, N.ptr(ys_cols),
                                        1 if ys_cols.dtype == np.float32 else 0, ld, p, k_max,
                                        eptr, float(rel_tol), *_out_ptrs(o), N.ENGINES[engine],
                                        stream))
    del ek
    return o


def zero_tree_cols_raw(low: DeviceDictionary, high: DeviceDictionary, fine_shape, factors,
                       ys_cols, k1: int, k_high: int, rel_tol: float, phi_mode: bool,
                       engine: str = "auto", out_low=None, out_high=None, stream=None):
    """cdb_zero_tree_batch_cols: the N x P column batch as the reference holds
    it (host memory); the transpose to rows happens on the device."""
    p = int(ys_cols.shape[1])
    lo = out_low if out_low is not None else _out(p, k1)
    hi = out_high if out_high is not None else _out(p, k_high)
    fs = np.asarray(fine_shape if fine_shape is not None else [1], dtype=np.int64)
    fa = np.asarray(factors if factors is not None else [1], dtype=np.int64)
    ms = np.zeros(2, np.float32)
    ld = ys_cols.strides[0] // ys_cols.itemsize
    N.check(N.load().cdb_zero_tree_batch_cols(low.handle, high.handle, N.ptr(fs), N.ptr(fa),
                                              int(fs.size), N.ptr(ys_cols),
                                              1 if ys_cols.dtype == np.float32 else 0, ld, p, k1,
                                              k_high, float(rel_tol), int(phi_mode),
                                              *_out_ptrs(lo), *_out_ptrs(hi), N.ENGINES[engine],
                                              N.ptr(ms), stream))
    return lo, hi, ms


# ---------------------------------------------------------------- patch pipeline ends
def _geom(signal_shape, patch_shape, stride):
    rank = len(signal_shape)
    return (rank, np.asarray(signal_shape, np.int64), np.asarray(patch_shape, np.int64),
            np.asarray(stride, np.int64))


def extract_patches_raw(signal, patch_shape, stride, remove_dc, rows=None, dc=None, stream=None):
    """cdb_extract_patches: rows (P x N fp64) and per-patch means (or None).

    ``signal`` is a numpy array or a CUDA tensor (fp32 / fp64); ``rows`` /
    ``dc`` may be preallocated (numpy or CUDA tensors)."""
    shape = tuple(signal.shape)
    rank, sg, pt, st = _geom(shape, patch_shape, stride)
    n = int(np.prod(pt))
    p = int(np.prod([(e - q) // s + 1 for e, q, s in zip(shape, patch_shape, stride)]))
    if isinstance(signal, np.ndarray):
        src = np.ascontiguousarray(signal)
        if src.dtype not in (np.float32, np.float64):
            src = src.astype(np.float64)
        f32 = 1 if src.dtype == np.float32 else 0
    else:
        import torch
        src = signal.contiguous()
        f32 = 1 if src.dtype == torch.float32 else 0
    if rows is None:
        rows = (pinned_empty if p >= PIN_MIN else np.empty)((p, n), np.float64)
    if remove_dc and dc is None:
        dc = np.empty(p, np.float64)
    N.check(N.load().cdb_extract_patches(N.ptr(src), f32, rank, N.ptr(sg), N.ptr(pt), N.ptr(st),
                                         int(bool(remove_dc)), N.ptr(rows),
                                         N.ptr(dc) if remove_dc else None, stream))
    return rows, (dc if remove_dc else None)


def aggregate_patches_raw(rows, dc, signal_shape, patch_shape, stride, out=None, stream=None):
    """cdb_aggregate_patches: overlap-averaged signal (fp64) and uncovered count."""
    rank, sg, pt, st = _geom(signal_shape, patch_shape, stride)
    if out is None:
        out = np.empty(tuple(signal_shape), np.float64)
    unc = np.zeros(1, np.int64)
    N.check(N.load().cdb_aggregate_patches(N.ptr(rows), N.ptr(dc), rank, N.ptr(sg), N.ptr(pt),
                                           N.ptr(st), N.ptr(out), N.ptr(unc), stream))
    return out, int(unc[0])


def reconstruct_aggregate_raw(dd: DeviceDictionary, sel, coef, p, dc, signal_shape, patch_shape,
                              stride, out=None, stream=None):
    """cdb_reconstruct_aggregate: D_S x (+ dc) per patch, overlap-averaged."""
    rank, sg, pt, st = _geom(signal_shape, patch_shape, stride)
    kw = int(sel.shape[1]) if len(sel.shape) > 1 else 0
    if out is None:
        out = np.empty(tuple(signal_shape), np.float64)
    unc = np.zeros(1, np.int64)
    N.check(N.load().cdb_reconstruct_aggregate(dd.handle, N.ptr(sel), N.ptr(coef), kw, int(p),
                                               N.ptr(dc), rank, N.ptr(sg), N.ptr(pt), N.ptr(st),
                                               N.ptr(out), N.ptr(unc), stream))
    return out, int(unc[0])


def omp_batch_blocked_ragged_raw(dd: DeviceDictionary, ys, p: int, k_max: int, eps, blocks, nb,
                                 q: int, engine: str = "auto", out=None, stream=None):
    """cdb_omp_batch_blocked_ragged: signal p uses the first nb[p] ids of row p."""
    o = out if out is not None else _out(p, k_max)
    yk, yptr, f32 = _ys_arg(ys)
    ek, eptr = _arg(eps, np.float64, "eps")
    bk, bptr = _arg(blocks, np.int64, "blocks")
    nk, nptr = _arg(nb, np.int64, "nb")
    N.check(N.load().cdb_omp_batch_blocked_ragged(dd.handle, yptr, f32, p, k_max, eptr, bptr,
                                                  int(blocks.shape[1]), nptr,
                                                  int(q), *_out_ptrs(o), N.ENGINES[engine],
                                                  stream))
    del yk, ek, bk, nk
    return o


def omp_batch_masked_raw(dd: DeviceDictionary, ys, rows, m, p: int, k_max: int, eps, out=None,
                         stream=None):
    """cdb_omp_batch_masked: OMP of ys[p][:m[p]] over D[rows[p][:m[p]], :]."""
    o = out if out is not None else _out(p, k_max)
    keep = [_arg(ys, np.float64, "ys"), _arg(rows, np.int32, "rows"), _arg(m, np.int64, "m"),
            _arg(eps, np.float64, "eps")]
    (_, yptr), (_, rptr), (_, mptr), (_, eptr) = keep
    N.check(N.load().cdb_omp_batch_masked(dd.handle, yptr, rptr, mptr, int(p),
                                          int(k_max), eptr, *_out_ptrs(o), stream))
    del keep
    return o


def omp_batch_coded_raw(dd: DeviceDictionary, ys, rows, m, p: int, k_max: int, eps,
                        blocks=None, nb=None, q: int = 1, pairwise: bool = False, out=None,
                        stream=None):
    """cdb_omp_batch_coded: OMP of ys[p][:m[p]] over the coded effective
    dictionary of rows (P x M x fan int32, -1 padded; ``pairwise``: numpy's
    pairwise order over all fan slots), optionally restricted to the ragged
    blocks (P x nb_max, nb[p] used)."""
    o = out if out is not None else _out(p, k_max)
    m_stride, fan = int(rows.shape[1]), int(rows.shape[2])
    nb_max = int(blocks.shape[1]) if blocks is not None else 0
    keep = [_arg(ys, np.float64, "ys"), _arg(rows, np.int32, "rows"), _arg(m, np.int64, "m"),
            _arg(eps, np.float64, "eps"), _arg(blocks, np.int64, "blocks"),
            _arg(nb, np.int64, "nb")]
    (_, yptr), (_, rptr), (_, mptr), (_, eptr), (_, bptr), (_, nptr) = keep
    N.check(N.load().cdb_omp_batch_coded(dd.handle, yptr, m_stride, rptr, fan,
                                         1 if pairwise else 0, mptr, int(p), int(k_max), eptr,
                                         bptr, nb_max, nptr, int(q), *_out_ptrs(o), stream))
    del keep
    return o
