"""``.csd`` model files -- mirror of crossdict
``fileio.save_model`` / ``load_model`` (fileio.py:146-256).

Reading goes through the native ``cdb_csd_read`` (CRC-32 verified before any
parsing, every structural rule and message of the reference loader).  The
file's column-major N x T atom block is byte-for-byte the T x N row layout
the device dictionaries use, so ``load_model(..., stage=True)`` hands it to
the GPU without a transpose.  Writing is the reference's byte layout.
"""

from __future__ import annotations

import ctypes
import struct
import zlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from . import device as _dev
from . import errors as E
from .crossscale import CrossScaleModel
from .scaling import ScaleSpec
from .tensor import Dictionary

_CSD_MAGIC = b"CSDM"
_VERSION = 1


@dataclass(frozen=True)
class SingleScaleModel:
    """A plain dictionary plus the patch geometry and budget it was trained for."""

    dictionary: Dictionary
    patch_shape: tuple
    sparsity: int


class _Scale(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("extents", ctypes.c_int64 * 4),
                ("n", ctypes.c_int64), ("t", ctypes.c_int64), ("k", ctypes.c_int64),
                ("q", ctypes.c_int64)]


def _read(path):
    lib = N.load()
    raw = Path(path).read_bytes()  # read once (as the reference): both parses see these bytes
    data = np.frombuffer(raw, dtype=np.uint8)
    name = str(path).encode()
    count = ctypes.c_int32()
    scales = (_Scale * 2)()
    _raise(lib.cdb_csd_parse(N.ptr(data) if data.size else ctypes.c_char_p(b""), data.size, name,
                             ctypes.byref(count), scales, None, None))
    bufs = [np.empty((scales[i].t, scales[i].n), np.float64) for i in range(count.value)]
    arr = (ctypes.c_void_p * 2)(*[b.ctypes.data for b in bufs], *([None] * (2 - len(bufs))))
    cap = np.array([b.size for b in bufs] + [0] * (2 - len(bufs)), dtype=np.int64)
    _raise(lib.cdb_csd_parse(N.ptr(data) if data.size else ctypes.c_char_p(b""), data.size, name,
                             ctypes.byref(count), scales, arr, N.ptr(cap)))
    out = []
    for i in range(count.value):
        s = scales[i]
        out.append((tuple(int(s.extents[d]) for d in range(s.rank)), bufs[i], int(s.k), int(s.q)))
    return out


def _raise(status):
    if status == 0:
        return
    msg = N.load().cdb_last_error().decode()
    if status == 6:
        raise E.ChecksumError(msg)
    if status == 5:
        raise E.FormatError(msg)
    if status == 1 and msg.endswith("cannot open"):
        raise FileNotFoundError(msg)
    N.check(status)


# install(): the reference's model / dictionary classes, so the drop-in
# load_model returns the caller's own types
_types: dict = {}


def load_model(path, stage: bool = False):
    """Load a .csd file -> CrossScaleModel or SingleScaleModel (fileio.py:216-256).

    ``stage=True`` also creates the device dictionaries now (cached for the
    pursuit calls that follow)."""
    recs = _read(path)
    dict_cls = _types.get("Dictionary", Dictionary)
    dicts = []
    for shape, atoms_t, k, q in recs:
        d = dict_cls(np.asarray(atoms_t).T)  # validates unit norms as the reference
        dicts.append((shape, d, k, q))
    if stage:
        for _, d, _, _ in dicts:
            _dev.device_dictionary(np.ascontiguousarray(d.atoms_t))
    if len(dicts) == 1:
        shape, d, k, _ = dicts[0]
        return _types.get("SingleScaleModel", SingleScaleModel)(d, shape, k)
    (coarse, d_low, k_low, _), (fine, d_high, k_high, _) = dicts
    factors = tuple(f // c for f, c in zip(fine, coarse))
    scale = _types.get("ScaleSpec", ScaleSpec)(fine, factors)
    return _types.get("CrossScaleModel", CrossScaleModel)(d_low, d_high, scale, k_low, k_high)


def _pack_record(buf: bytearray, patch_shape, dictionary: Dictionary, k: int, q: int):
    shape = tuple(int(e) for e in patch_shape)
    buf += struct.pack("<I", len(shape))
    buf += struct.pack(f"<{len(shape)}I", *shape)
    buf += struct.pack("<IIII", dictionary.atom_dim, dictionary.num_atoms, int(k), int(q))
    buf += np.asarray(dictionary.atoms, dtype="<f8").tobytes(order="F")


def save_model(path, model, patch_shape=None, sparsity=None) -> None:
    """Serialize a model to .csd (fileio.py:156-179)."""
    buf = bytearray(_CSD_MAGIC)
    buf += struct.pack("<I", _VERSION)
    if isinstance(model, CrossScaleModel):
        buf += struct.pack("<I", 2)
        _pack_record(buf, model.scale.coarse_shape, model.d_low, model.k_low, model.q)
        _pack_record(buf, model.scale.fine_shape, model.d_high, model.k_high, 0)
    elif isinstance(model, SingleScaleModel):
        buf += struct.pack("<I", 1)
        _pack_record(buf, model.patch_shape, model.dictionary, model.sparsity, 0)
    else:
        if patch_shape is None or sparsity is None:
            raise E.DimensionError("bare Dictionary needs patch_shape and sparsity")
        buf += struct.pack("<I", 1)
        _pack_record(buf, patch_shape, model, sparsity, 0)
    buf += struct.pack("<I", zlib.crc32(bytes(buf)) & 0xFFFFFFFF)
    Path(path).write_bytes(bytes(buf))
