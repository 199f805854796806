"""Pin the CPU oracle (oracle/) against the reference's own outputs.

tests/golden/*.npz were produced by running the reference package itself
(tests/golden/make_golden.py).  The oracle restates the reference kernel's
arithmetic operation for operation, so outside the rank-deficient dense mode
(LAPACK in the reference, Jacobi SVD here: "parity unpinned") every output
must be BIT-identical.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import edge_names, load_golden

import oracle as O
from paper_1511_05174_b200 import workloads as W

NTHREADS = max(1, min(8, os.cpu_count() or 1))


def _assert_same(ref, got, flagged=()):
    assert np.array_equal(ref["counts"], got["counts"])
    assert np.array_equal(ref["sel"], got["sel"])
    assert np.array_equal(ref["scans"], got["scans"])
    keep = np.ones(len(ref["counts"]), bool)
    keep[list(flagged)] = False
    assert np.array_equal(ref["alpha"][keep], got["alpha"][keep])
    assert np.array_equal(ref["rnorm"][keep], got["rnorm"][keep])


def _golden(g, prefix=""):
    return {k: g[prefix + k] for k in ("counts", "sel", "alpha", "rnorm", "scans")}


@pytest.mark.parametrize("name", [n for n in edge_names() if not n.startswith("edge_zt")])
def test_oracle_edge_omp(name):
    g = load_golden(name)
    tol = None if g["tol"] < 0 else float(g["tol"])
    kw = {}
    if "blocks" in g:
        kw = dict(allowed_blocks=g["blocks"], block_q=int(g["q"]))
    got = O.omp_many_arrays(g["mat_t"], g["ys_rows"], int(g["k"]), rel_tol=float(g["rel"]),
                            residual_tolerance=tol, **kw)
    _assert_same(_golden(g), got, flagged=g["flag"])
    assert sorted(np.flatnonzero(got["flag"]).tolist()) == sorted(g["flag"].tolist())


@pytest.mark.parametrize("name", [n for n in edge_names() if n.startswith("edge_zt")])
def test_oracle_edge_zero_tree(name):
    g = load_golden(name)
    low, high = O.zero_tree_many_arrays(g["low_t"], g["high_t"], tuple(g["fine_shape"]),
                                        tuple(g["factors"]), int(g["k_low"]), int(g["k_high"]),
                                        g["ys_rows"], rel_tol=float(g["rel"]))
    _assert_same(_golden(g, "low_"), low)
    _assert_same(_golden(g, "high_"), high)


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("ci", [0, 1, 2, 3, 4])
def test_oracle_baseline_configs(ci):
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    high_t = d.e_high_t if w.measurements else d.high_t
    low_t = d.e_low_t if w.measurements else d.low_t
    g = load_golden(f"cfg{ci}_full")
    ys = W.signals_at(ci, g["ids"])
    assert _digest(high_t) == str(g["d_sha"]) and _digest(ys) == str(g["y_sha"]), \
        "workload generator drifted from the golden fixtures"
    got = O.omp_many_arrays(high_t, ys, w.k, rel_tol=W.REL_TOL, nthreads=NTHREADS)
    _assert_same(_golden(g), got, flagged=g["flag"])

    g = load_golden(f"cfg{ci}_zt")
    ys = W.signals_at(ci, g["ids"])
    assert _digest(ys) == str(g["y_sha"]) and _digest(low_t) == str(g["dl_sha"])
    if w.measurements:
        low, high = O.zero_tree_phi_many(low_t, high_t, w.k, w.k, ys, rel_tol=W.REL_TOL,
                                         nthreads=NTHREADS)
    else:
        low, high = O.zero_tree_many_arrays(low_t, high_t, w.fine_shape, w.factors, w.k, w.k, ys,
                                            rel_tol=W.REL_TOL, nthreads=NTHREADS)
    _assert_same(_golden(g, "low_"), low)
    _assert_same(_golden(g, "high_"), high)


def test_oracle_threads_do_not_change_results():
    g = load_golden("edge_batch")
    a = O.omp_many_arrays(g["mat_t"], g["ys_rows"], int(g["k"]), nthreads=1)
    b = O.omp_many_arrays(g["mat_t"], g["ys_rows"], int(g["k"]), nthreads=4)
    _assert_same(a, b)


def test_downsample_rows_matches_reference_layout():
    # scaling.py:99-116 on signals-as-columns == oracle on signals-as-rows
    from paper_1511_05174_b200.scaling import ScaleSpec, downsample_columns
    rng = np.random.default_rng(3)
    spec = ScaleSpec((4, 4, 2), (2, 2, 2))
    fine = rng.standard_normal((spec.fine_size, 7))
    assert np.allclose(downsample_columns(fine, spec).T,
                       O.downsample_rows(fine.T, spec.fine_shape, spec.factors))
