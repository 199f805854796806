"""The public drop-in entry points on the GPU -- what a crossdict caller
imports -- against the reference's golden outputs: omp (pursuit.py:253-300),
omp_many_arrays (pursuit.py:388-441), omp_many (444-461), zero_tree_omp
(crossscale.py:169-232), zero_tree_many_arrays (235-283) and
zero_tree_omp_many (286-312).  Inputs are pageable N x P fp64 column batches
(the reference's layout; the drop-in makes the P x N row copy, pinned for
large batches); results are checked for their types, 1-based codes, pick
order, timings, and the parity contract against the goldens."""

import numpy as np
import pytest

from conftest import edge_names, load_golden
from parity import batch_dict, check_zero_tree, compare, golden_dict

import paper_1511_05174_b200 as P
from paper_1511_05174_b200 import pursuit as PU
from paper_1511_05174_b200 import workloads as W
from paper_1511_05174_b200.crossscale import ZeroTreeResult
from paper_1511_05174_b200.pursuit import BatchSolve, PursuitResult

pytestmark = pytest.mark.gpu

OMP_EDGES = [n for n in edge_names() if not n.startswith("edge_zt")]
ZT_EDGES = [n for n in edge_names() if n.startswith("edge_zt")]


@pytest.fixture
def rel_tol():
    old = PU.REL_RESIDUAL_TOL

    def set_(v):
        PU.REL_RESIDUAL_TOL = float(v)
    yield set_
    PU.REL_RESIDUAL_TOL = old


def _config(g):
    k = int(g["k"])
    tol = float(g["tol"])
    return PU.PursuitConfig(k, residual_tolerance=tol if tol >= 0 else None)


def _eps(g, ys_rows):
    if g["tol"] >= 0:
        return np.full(ys_rows.shape[0], float(g["tol"]))
    return float(g["rel"]) * np.linalg.norm(ys_rows, axis=1)


def _allowed(g):
    if "blocks" not in g:
        return None
    q = int(g["q"])
    return (g["blocks"][:, :, None] * q + np.arange(q)[None, None, :]).reshape(len(g["blocks"]), -1)


def _check_batch(s, p, k_width):
    assert isinstance(s, BatchSolve)
    assert s.counts.shape == (p,) and s.counts.dtype == np.int64
    assert s.sel.shape == (p, k_width) and s.sel.dtype == np.int64
    assert s.alpha.shape == (p, k_width) and s.alpha.dtype == np.float64
    assert s.rnorm.dtype == np.float64 and s.scans.dtype == np.int64
    assert isinstance(s.rank_deficient, frozenset)


@pytest.mark.parametrize("name", OMP_EDGES)
def test_omp_many_arrays_edges(name, rel_tol):
    g = load_golden(name)
    rel_tol(g["rel"])
    ys_rows = g["ys_rows"]
    cols = np.array(ys_rows.T)  # pageable N x P fp64
    kw = {}
    if "blocks" in g:
        kw = dict(allowed_blocks=g["blocks"], block_q=int(g["q"]))
    s = P.omp_many_arrays(np.ascontiguousarray(g["mat_t"].T), cols, _config(g), **kw)
    _check_batch(s, ys_rows.shape[0], g["sel"].shape[1])
    rep = compare(golden_dict(g), batch_dict(s), g["mat_t"], ys_rows, _eps(g, ys_rows),
                  _allowed(g))
    assert not rep["bad"], rep["bad"][:3]


@pytest.mark.parametrize("name", ["edge_batch", "edge_ties", "edge_scans", "edge_mixed",
                                  "edge_rank_deficient"])
def test_scalar_omp_and_omp_many_edges(name, rel_tol):
    g = load_golden(name)
    rel_tol(g["rel"])
    ys_rows = g["ys_rows"]
    d = np.ascontiguousarray(g["mat_t"].T)
    ref = golden_dict(g)
    many = P.omp_many(d, np.array(ys_rows.T), _config(g))
    assert len(many) == ys_rows.shape[0]
    for p in range(min(ys_rows.shape[0], 12)):
        r = P.omp(d, ys_rows[p], _config(g))
        assert isinstance(r, PursuitResult)
        c = int(ref["counts"][p])
        for res in (r, many[p]):
            assert res.iterations == c and res.atom_scan_count == int(ref["scans"][p])
            assert res.selected == tuple(int(j) + 1 for j in ref["sel"][p, :c])  # pick order
            assert res.code.support == tuple(sorted(res.selected))           # sorted, 1-based
            assert res.rank_deficient == bool(ref["flag"][p])
            if not ref["flag"][p]:
                got = dict(res.code.entries)
                for i, j in enumerate(res.selected):
                    assert got[j] == pytest.approx(ref["alpha"][p, i], rel=1e-9, abs=1e-12)
                assert res.residual_norm == pytest.approx(ref["rnorm"][p], rel=1e-9, abs=1e-12)


def _zt_model(low_t, high_t, fine_shape, factors, k_low, k_high):
    return P.CrossScaleModel(P.Dictionary(np.ascontiguousarray(low_t.T)),
                             P.Dictionary(np.ascontiguousarray(high_t.T)),
                             P.ScaleSpec(tuple(int(e) for e in fine_shape),
                                         tuple(int(f) for f in factors)),
                             int(k_low), int(k_high))


def _check_zt_api(model, q, ys_rows, rl, rh, low_t, high_t, fine_shape, factors):
    low, high, tim = P.zero_tree_many_arrays(model, np.array(ys_rows.T))
    _check_batch(low, ys_rows.shape[0], model.k_low)
    _check_batch(high, ys_rows.shape[0], model.k_high)
    assert set(tim) == {"step1", "step2"} and all(v >= 0.0 for v in tim.values())
    import oracle as O
    yl = O.downsample_rows(ys_rows, tuple(fine_shape), tuple(factors))
    check_zero_tree(low_t, high_t, q, ys_rows, batch_dict(low), batch_dict(high), rl, rh, yl,
                    min_same=0.75)
    return low, high


@pytest.mark.parametrize("name", ZT_EDGES)
def test_zero_tree_api_edges(name, rel_tol):
    g = load_golden(name)
    rel_tol(g["rel"])
    model = _zt_model(g["low_t"], g["high_t"], g["fine_shape"], g["factors"], g["k_low"],
                      g["k_high"])
    ys = g["ys_rows"]
    rl, rh = golden_dict(g, "low_"), golden_dict(g, "high_")
    low, high = _check_zt_api(model, model.q, ys, rl, rh, g["low_t"], g["high_t"],
                              g["fine_shape"], g["factors"])
    # the per-signal entry points agree with the batch
    many = P.zero_tree_omp_many(model, np.array(ys.T))
    assert len(many) == ys.shape[0]
    for p in range(min(ys.shape[0], 8)):
        r = P.zero_tree_omp(model, ys[p])
        for res in (r, many[p]):
            assert isinstance(res, ZeroTreeResult)
            assert res.code_low.support == tuple(sorted(int(j) + 1 for j in
                                                        low.sel[p, :low.counts[p]]))
            assert res.code_high.support == tuple(sorted(int(j) + 1 for j in
                                                         high.sel[p, :high.counts[p]]))
            assert res.scan_counts == {"step1": int(low.scans[p]), "step2": int(high.scans[p])}
            assert res.residual_norm == pytest.approx(float(high.rnorm[p]), rel=1e-12)
            assert set(res.timings) == {"step1", "step2"}


@pytest.mark.parametrize("ci", [0, 1, 2, 4])
def test_zero_tree_api_configs(ci, rel_tol):
    rel_tol(W.REL_TOL)
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    g = load_golden(f"cfg{ci}_zt")
    ys = W.signals_at(ci, g["ids"])
    model = _zt_model(d.low_t, d.high_t, w.fine_shape, w.factors, w.k, w.k)
    _check_zt_api(model, w.q, ys, golden_dict(g, "low_"), golden_dict(g, "high_"), d.low_t,
                  d.high_t, w.fine_shape, w.factors)


def test_zero_tree_api_large_batch_pinned_path(rel_tol):
    """>= 4096 signals: the drop-in stages rows in pinned memory and the library
    pipelines the host copies; results equal the small-batch path's."""
    rel_tol(W.REL_TOL)
    ci = 1
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    ys = W.signals(ci, 0, 40_000)
    model = _zt_model(d.low_t, d.high_t, w.fine_shape, w.factors, w.k, w.k)
    low, high, tim = P.zero_tree_many_arrays(model, np.array(ys.T))
    lo2, hi2, _ = P.zero_tree_many_arrays(model, np.array(ys[:3000].T))
    for a, b in ((low, lo2), (high, hi2)):
        assert np.array_equal(a.sel[:3000], b.sel) and np.array_equal(a.counts[:3000], b.counts)
        assert np.array_equal(a.alpha[:3000], b.alpha)
    assert tim["step1"] > 0 and tim["step2"] > 0


@pytest.mark.parametrize("ci", [0, 1, 3])
def test_omp_many_arrays_configs(ci, rel_tol):
    rel_tol(W.REL_TOL)
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    g = load_golden(f"cfg{ci}_full")
    ys = W.signals_at(ci, g["ids"])
    hi_t = d.e_high_t if w.measurements else d.high_t
    s = P.omp_many_arrays(np.ascontiguousarray(hi_t.T), np.array(ys.T), PU.PursuitConfig(w.k))
    _check_batch(s, ys.shape[0], w.k)
    rep = compare(golden_dict(g), batch_dict(s), hi_t, ys, W.REL_TOL * np.linalg.norm(ys, axis=1))
    assert not rep["bad"], rep["bad"][:3]


def _zt_rows(model, ys_rows, f32):
    """The rows-ABI solve of the same batch (cdb_zero_tree_batch)."""
    from paper_1511_05174_b200 import device as D
    dl = D.device_dictionary(model.d_low.atoms_t)
    dh = D.device_dictionary(model.d_high.atoms_t)
    rows = np.ascontiguousarray(ys_rows, dtype=np.float32 if f32 else np.float64)
    lo, hi, _ = D.zero_tree_raw(dl, dh, model.scale.fine_shape, model.scale.factors, rows,
                                len(rows), model.k_low, model.k_high, W.REL_TOL, False, "auto")
    return lo, hi


@pytest.mark.parametrize("case", ["f64_exact", "f32_input", "strided", "f64_inexact",
                                  "late_inexact"])
def test_zero_tree_cols_path(case, rel_tol):
    """Large N x P batches cross the ABI as columns (cdb_zero_tree_batch_cols):
    host-staged slabs (fp32 when exact), device transpose, chunk pipeline.
    Results equal the rows ABI on the same values -- fp32 rows when every value
    is fp32-exact, fp64 rows otherwise (including a batch whose only inexact
    value sits in a later chunk: the call is redone in fp64)."""
    from paper_1511_05174_b200 import device as D
    rel_tol(W.REL_TOL)
    ci = 1
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    p = 50_000
    ys = W.signals(ci, 0, p)
    f32 = True
    if case == "f64_inexact":
        ys = ys * (1.0 + 2.0 ** -40)
        f32 = False
    elif case == "late_inexact":
        ys = ys.copy()
        ys[41_234, 7] += 2.0 ** -35 * abs(ys[41_234, 7])
        f32 = False
    model = _zt_model(d.low_t, d.high_t, w.fine_shape, w.factors, w.k, w.k)
    if case == "f32_input":
        cols = np.ascontiguousarray(ys.T, dtype=np.float32)
    elif case == "strided":
        wide = np.zeros((ys.shape[1], p + 37))
        wide[:, 5:5 + p] = ys.T
        cols = wide[:, 5:5 + p]
    else:
        cols = np.ascontiguousarray(ys.T)
    assert D.cols_layout(cols)
    low, high, tim = P.zero_tree_many_arrays(model, cols)
    assert tim["step1"] > 0 and tim["step2"] > 0
    rl, rh = _zt_rows(model, ys, f32)
    for a, b in ((low, rl), (high, rh)):
        assert np.array_equal(a.sel, b["sel"]) and np.array_equal(a.counts, b["counts"])
        assert np.array_equal(a.scans, b["scans"])
        np.testing.assert_allclose(a.alpha, b["alpha"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(a.rnorm, b["rnorm"], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("case", ["f64_exact", "f32_input", "fixed_tol"])
def test_omp_many_arrays_cols_path(case, rel_tol):
    """Large N x P batches of omp_many_arrays cross the ABI as columns
    (cdb_omp_batch_cols, tolerances rel * |y| on the device): results equal the
    rows ABI on fp32 rows with the reference's host tolerances."""
    from paper_1511_05174_b200 import device as D
    rel_tol(W.REL_TOL)
    ci = 1
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    p = 40_000
    ys = W.signals(ci, 0, p)
    tol = 0.05 if case == "fixed_tol" else None
    cols = np.ascontiguousarray(ys.T, dtype=np.float32 if case == "f32_input" else np.float64)
    assert D.cols_layout(cols)
    s = P.omp_many_arrays(np.ascontiguousarray(d.high_t.T), cols,
                          PU.PursuitConfig(w.k, residual_tolerance=tol))
    _check_batch(s, p, w.k)
    eps = np.full(p, tol) if tol else W.REL_TOL * np.sqrt(np.einsum("pn,pn->p", ys, ys))
    r = D.omp_batch_raw(D.device_dictionary(d.high_t), ys.astype(np.float32), p, w.k, eps)
    assert np.array_equal(s.sel, r["sel"]) and np.array_equal(s.counts, r["counts"])
    assert np.array_equal(s.scans, r["scans"])
    np.testing.assert_allclose(s.alpha, r["alpha"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(s.rnorm, r["rnorm"], rtol=1e-12, atol=1e-14)


def test_column_matrix_cache_follows_in_place_changes(rel_tol):
    """omp_many_arrays stages `columns` once per content: a second call on the
    same matrix reuses the device dictionary (no new staging), and a matrix
    changed in place -- the reference re-reads it on every call,
    pursuit.py:84-94 -- is staged again instead of served from the cache."""
    from paper_1511_05174_b200 import device as D
    rel_tol(1e-3)
    rng = np.random.default_rng(11)
    n, t, p, k = 64, 8192 + 512, 48, 4  # 4.4 MB: the threaded comparison path
    mat = rng.standard_normal((n, t))
    mat /= np.linalg.norm(mat, axis=0, keepdims=True)
    picks = rng.choice(t, size=p, replace=False)
    ys = np.ascontiguousarray(mat[:, picks])  # one-atom signals
    s1 = P.omp_many_arrays(mat, ys, PU.PursuitConfig(k))
    assert np.array_equal(s1.sel[:, 0], picks) and np.all(s1.counts == 1)
    dd1 = D.device_dictionary_cols(mat)
    assert D.device_dictionary_cols(mat) is dd1  # a hit: same handle
    # swap two atoms in place (the sampled entries 0, size/3, size/2, size-1 keep their values)
    a, b = int(picks[0]), int(picks[1])
    if {a, b} & {0, t - 1, (n * t // 3) % t, (n * t // 2) % t}:
        pytest.skip("sampled column touched")
    mat[:, [a, b]] = mat[:, [b, a]]
    s2 = P.omp_many_arrays(mat, ys, PU.PursuitConfig(k))
    assert s2.sel[0, 0] == b and s2.sel[1, 0] == a
    assert np.array_equal(s2.sel[2:, 0], picks[2:])
    assert D.device_dictionary_cols(mat) is not dd1
