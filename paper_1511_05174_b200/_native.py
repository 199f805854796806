"""ctypes binding of the C ABI in include/crossdict_b200.h.

There is no fallback: if ``_lib/libcrossdict_b200.so`` is missing the import of
any compute entry point raises immediately (build it with
``python -c "import __graft_entry__ as g; g.build()"`` or ``make -C
paper_1511_05174_b200/csrc``).  The library itself returns CDB_ERR_NODEV on a
machine without an sm_100 GPU; the host layer turns that into a RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                        "libcrossdict_b200.so")

ENGINES = {"auto": 0, "exact": 1, "gram": 2, "tensor": 3, "resident": 4}

#: every symbol include/crossdict_b200.h declares (checked by tests/test_abi.py)
SYMBOLS = ("cdb_last_error", "cdb_device_info", "cdb_dictionary_create",
           "cdb_dictionary_destroy", "cdb_dictionary_bytes", "cdb_omp_batch",
           "cdb_omp_batch_blocked", "cdb_zero_tree_batch", "cdb_launch_count",
           "cdb_last_run_info", "cdb_profile_enable", "cdb_profile_read",
           "cdb_debug_corr_topk", "cdb_rows_from_cols", "cdb_extract_patches",
           "cdb_reconstruct_aggregate", "cdb_aggregate_patches", "cdb_csd_read", "cdb_csd_parse",
           "cdb_omp_batch_blocked_ragged", "cdb_omp_batch_masked", "cdb_omp_batch_coded", "cdb_ksvd_update",
           "cdb_zero_tree_batch_cols", "cdb_omp_batch_cols", "cdb_host_equal")

_lib = None


class NativeError(RuntimeError):
    """A non-OK cdb_status from the native library."""


def load():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(
            f"native library not built: {LIB_PATH} is missing "
            "(run `make -C paper_1511_05174_b200/csrc`); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    lib.cdb_last_error.restype = ctypes.c_char_p
    lib.cdb_launch_count.restype = I64
    lib.cdb_device_info.argtypes = [P, P, P]
    lib.cdb_last_run_info.argtypes = [P, P, P]
    lib.cdb_rows_from_cols.argtypes = [P, I64, I64, I32, P, I32]
    lib.cdb_host_equal.argtypes = [P, P, I64, I32]
    lib.cdb_host_equal.restype = I32
    lib.cdb_extract_patches.argtypes = [P, I32, I32, P, P, P, I32, P, P, P]
    lib.cdb_reconstruct_aggregate.argtypes = [P, P, P, I64, I64, P, I32, P, P, P, P, P, P]
    lib.cdb_aggregate_patches.argtypes = [P, P, I32, P, P, P, P, P, P]
    lib.cdb_csd_read.argtypes = [ctypes.c_char_p, P, P, P]
    lib.cdb_csd_parse.argtypes = [P, I64, ctypes.c_char_p, P, P, P, P]
    lib.cdb_omp_batch_masked.argtypes = [P, P, P, P, I64, I64, P, P, P, P, P, P, P, P]
    lib.cdb_ksvd_update.argtypes = [I64, I64, I64, P, P, P, P, P, P, I64, I64, I64, P, P]
    lib.cdb_omp_batch_coded.argtypes = [P, P, I64, P, I64, I32, P, I64, I64, P, P, I64, P, I64,
                                        P, P, P, P, P, P, P]
    lib.cdb_omp_batch_blocked_ragged.argtypes = [P, P, I32, I64, I64, P, P, I64, P, I64, P, P, P,
                                                 P, P, P, I32, P]
    lib.cdb_last_run_info.restype = None
    lib.cdb_debug_corr_topk.argtypes = [P, P, I64, P, P, P, I32, P]
    lib.cdb_debug_corr_topk.restype = I32
    lib.cdb_profile_enable.argtypes = [I32]
    lib.cdb_profile_enable.restype = None
    lib.cdb_profile_read.argtypes = [I32, P, I32, P, P]
    lib.cdb_profile_read.restype = I32
    lib.cdb_dictionary_create.argtypes = [P, I64, I64, I64, P, P]
    lib.cdb_dictionary_destroy.argtypes = [P]
    lib.cdb_dictionary_bytes.argtypes = [P]
    lib.cdb_dictionary_bytes.restype = I64
    lib.cdb_omp_batch.argtypes = [P, P, I32, I64, I64, P, P, I64, I32, P, P, P, P, P, P, I32, P]
    lib.cdb_omp_batch_blocked.argtypes = [P, P, I32, I64, I64, P, P, I64, I64, P, P, P, P, P, P,
                                          I32, P]
    lib.cdb_zero_tree_batch.argtypes = [P, P, P, P, I32, P, I32, I64, I64, I64, D, I32,
                                        P, P, P, P, P, P, P, P, P, P, P, P, I32, P, P]
    lib.cdb_zero_tree_batch_cols.argtypes = [P, P, P, P, I32, P, I32, I64, I64, I64, I64, D, I32,
                                             P, P, P, P, P, P, P, P, P, P, P, P, I32, P, P]
    lib.cdb_omp_batch_cols.argtypes = [P, P, I32, I64, I64, I64, P, D, P, P, P, P, P, P, I32, P]
    for name in ("cdb_device_info", "cdb_dictionary_create", "cdb_dictionary_destroy",
                 "cdb_omp_batch", "cdb_omp_batch_blocked", "cdb_zero_tree_batch",
                 "cdb_zero_tree_batch_cols", "cdb_omp_batch_cols", "cdb_host_equal"):
        getattr(lib, name).restype = I32
    _lib = lib
    return lib


def check(status: int):
    if status != 0:
        msg = load().cdb_last_error()
        raise NativeError(f"cdb status {status}: {msg.decode() if msg else ''}")


def ptr(a) -> ctypes.c_void_p | None:
    """Address of a numpy array, a torch tensor or an int; None for None."""
    if a is None:
        return None
    if isinstance(a, int):
        return ctypes.c_void_p(a)
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())  # torch.Tensor (device or pinned host)


def last_run_info():
    """(engine, delegated signals, inline exact rescans) of the last OMP pass."""
    e, d, r = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    load().cdb_last_run_info(ctypes.byref(e), ctypes.byref(d), ctypes.byref(r))
    names = {v: k for k, v in ENGINES.items()}
    return names.get(e.value, str(e.value)), d.value, r.value


def profile_enable(on: bool = True) -> None:
    load().cdb_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel name: (total ms, launches)} recorded since profile_enable()."""
    lib = load()
    n = lib.cdb_profile_read(0, None, 0, None, None)
    if n <= 0:
        return {}
    names = ctypes.create_string_buffer(n * 64)
    ms = np.zeros(n)
    cnt = np.zeros(n, np.int64)
    lib.cdb_profile_read(n, names, 64, ptr(ms), ptr(cnt))
    out = {}
    for i in range(n):
        nm = names.raw[i * 64:(i + 1) * 64].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(cnt[i]))
    return out


def launch_count() -> int:
    return int(load().cdb_launch_count())


def device_info():
    sms, major, minor = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    check(load().cdb_device_info(ctypes.byref(sms), ctypes.byref(major), ctypes.byref(minor)))
    return sms.value, major.value, minor.value
