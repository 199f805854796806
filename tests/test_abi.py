"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1511_05174_b200 import _native as N

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "crossdict_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cdb_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_python_symbol_list():
    assert declared_functions() == sorted(N.SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    lib = N.load()
    for name in declared_functions():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr), name


def test_library_is_sm100a_only():
    # every kernel image in the .so is sm_100a SASS (no PTX JIT fallback)
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        return  # cuobjdump unavailable
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_launch_counter_callable_without_gpu():
    assert N.launch_count() >= 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (64, 64), (256, 1000), (33, 4097)])
def test_rows_from_cols_host_transpose(dtype, shape):
    # cdb_rows_from_cols is host code (no GPU): the N x P -> P x N copy the
    # drop-in makes (the reference's pursuit.py:433)
    from paper_1511_05174_b200 import _native as N
    n, p = shape
    cols = np.random.default_rng(n * p).standard_normal((n, p)).astype(dtype)
    rows = np.empty((p, n), dtype)
    N.check(N.load().cdb_rows_from_cols(N.ptr(cols), n, p, cols.itemsize, N.ptr(rows), 3))
    assert np.array_equal(rows, cols.T)
    with pytest.raises(N.NativeError):
        N.check(N.load().cdb_rows_from_cols(N.ptr(cols), n, p, 2, N.ptr(rows), 1))


@pytest.mark.parametrize("nbytes", [0, 1, 4096, (1 << 20) + 17, 5 * (1 << 20) + 3])
def test_host_equal(nbytes):
    # cdb_host_equal is host code: the exact check behind the dictionary cache
    a = np.random.default_rng(nbytes).integers(0, 256, size=max(nbytes, 1), dtype=np.uint8)
    b = a.copy()
    lib = N.load()
    assert lib.cdb_host_equal(N.ptr(a), N.ptr(b), nbytes, 3) == 1
    assert lib.cdb_host_equal(N.ptr(a), N.ptr(a), nbytes, 0) == 1
    for pos in {0, nbytes // 2, nbytes - 1} if nbytes else ():
        b[pos] ^= 1
        assert lib.cdb_host_equal(N.ptr(a), N.ptr(b), nbytes, 3) == 0, pos
        b[pos] ^= 1
    assert lib.cdb_host_equal(N.ptr(a), N.ptr(b), nbytes, 1) == 1
