"""Golden .csd files for the model loader, written and
parsed by the REFERENCE (crossdict.fileio) in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_csd.py

* csd_single.csd / csd_cross.csd: reference save_model output of a single-
  scale and a cross-scale model; csd_expect.npz: what reference load_model
  returns for them (atoms, shapes, budgets).
* csd_errors.npz: for each malformed variant (built here from csd_cross.csd
  with a recomputed CRC unless the case is the CRC itself) the reference's
  exception class and message, with the path replaced by {path}.
"""

from __future__ import annotations

import os
import struct
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from crossdict.crossscale import CrossScaleModel  # noqa: E402
from crossdict.fileio import SingleScaleModel, load_model, save_model  # noqa: E402
from crossdict.scaling import ScaleSpec  # noqa: E402
from crossdict.tensor import normalize_atoms  # noqa: E402


def with_crc(body: bytes) -> bytes:
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def main():
    rng = np.random.default_rng(5)
    single = SingleScaleModel(normalize_atoms(rng.standard_normal((12, 20))), (3, 4), 5)
    save_model(os.path.join(HERE, "csd_single.csd"), single)
    d_low = normalize_atoms(rng.standard_normal((4, 6)))
    d_high = normalize_atoms(rng.standard_normal((16, 18)))
    cross = CrossScaleModel(d_low, d_high, ScaleSpec((4, 4), (2, 2)), 2, 4)
    save_model(os.path.join(HERE, "csd_cross.csd"), cross)
    s = load_model(os.path.join(HERE, "csd_single.csd"))
    c = load_model(os.path.join(HERE, "csd_cross.csd"))
    np.savez(os.path.join(HERE, "csd_expect.npz"), single_atoms=s.dictionary.atoms,
             single_shape=np.array(s.patch_shape), single_k=s.sparsity,
             low_atoms=c.d_low.atoms, high_atoms=c.d_high.atoms,
             fine_shape=np.array(c.scale.fine_shape), factors=np.array(c.scale.factors),
             k_low=c.k_low, k_high=c.k_high)
    raw = open(os.path.join(HERE, "csd_cross.csd"), "rb").read()
    body = raw[:-4]
    rec0 = 12  # after magic, version, count
    cases = {
        "crc": raw[:-5] + bytes([raw[-5] ^ 1]) + raw[-4:],
        "short": with_crc(b"CSDM" + b"\x01\x00\x00"),
        "magic": with_crc(b"XSDM" + body[4:]),
        "version": with_crc(body[:4] + struct.pack("<I", 2) + body[8:]),
        "count": with_crc(body[:8] + struct.pack("<I", 3) + body[12:]),
        "rank": with_crc(body[:rec0] + struct.pack("<I", 5) + body[rec0 + 4:]),
        "n_mismatch": with_crc(body[:rec0 + 12] + struct.pack("<I", 5) + body[rec0 + 16:]),
        "truncated_atoms": with_crc(body[:rec0 + 28 + 40]),
        "truncated_header": with_crc(body[:rec0 + 6]),
        "q_fine": None,
        "t_high": None,
    }
    # fine record starts after the coarse one: rank 2, extents 2, N T K Q, atoms
    fine0 = rec0 + 4 + 8 + 16 + 8 * 4 * 6
    cases["q_fine"] = with_crc(body[:fine0 + 4 + 8 + 12] + struct.pack("<I", 7) +
                               body[fine0 + 4 + 8 + 16:])
    cases["t_high"] = with_crc(body[:rec0 + 4 + 8 + 12] + struct.pack("<I", 4) +
                               body[rec0 + 4 + 8 + 16:])
    names, classes, msgs = [], [], []
    for name, data in cases.items():
        path = os.path.join(HERE, f"csd_bad_{name}.csd")
        with open(path, "wb") as f:
            f.write(data)
        try:
            load_model(path)
            cls, msg = "none", ""
        except Exception as e:  # the reference's own classes
            cls, msg = type(e).__name__, str(e).replace(path, "{path}")
        names.append(name)
        classes.append(cls)
        msgs.append(msg)
    np.savez(os.path.join(HERE, "csd_errors.npz"), names=np.array(names),
             classes=np.array(classes), msgs=np.array(msgs))
    for n, c_, m in zip(names, classes, msgs):
        print(f"{n:18s} {c_:16s} {m}")


if __name__ == "__main__":
    main()
