"""K-SVD coding stage on the device against the reference's
own _code_stage outputs (tests/golden/learn_code_stage.npz): the ragged block
call reproduces the per-group results, with the parity contract."""

import os

import numpy as np
import pytest

from paper_1511_05174_b200.learn import code_stage

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                         "learn_code_stage.npz"))


def _check(results, prefix, k):
    for p, r in enumerate(results):
        sel = np.full(k, -1, np.int64)
        sel[:len(r.selected)] = r.selected
        assert np.array_equal(sel, G[f"{prefix}_sel"][p]), p
        assert r.iterations == G[f"{prefix}_iterations"][p]
        assert r.atom_scan_count == G[f"{prefix}_scans"][p]
        sup = np.asarray(r.code.support)
        assert np.array_equal(sup, G[f"{prefix}_support"][p][:len(sup)])
        np.testing.assert_allclose(np.asarray(r.code.coefficients), G[f"{prefix}_values"][p][:len(sup)],
                                   rtol=1e-9, atol=1e-12)
        assert r.residual_norm == pytest.approx(G[f"{prefix}_rnorm"][p], rel=1e-9, abs=1e-12)


def test_plain_coding_stage():
    k = int(G["k"])
    _check(code_stage(G["d"], G["y"], k, None, None), "plain", k)


def test_ragged_block_coding_stage_is_one_call_with_reference_results():
    k, q = int(G["k"]), int(G["q"])
    blocks_list = [[int(b) for b in row if b >= 0] for row in G["blocks_list"]]
    allowed = [set(b * q + c + 1 for b in bl for c in range(q)) for bl in blocks_list]
    _check(code_stage(G["d"], G["y"], k, allowed, (blocks_list, q)), "blocks", k)


def test_explicit_allowed_sets_coding_stage():
    k = int(G["k"])
    sets = [set(int(j) for j in row if j >= 0) for row in G["sets_list"]]
    _check(code_stage(G["d"], G["y"][:, :24], k, sets, None), "sets", k)


def test_code_stage_arbitrary_sets_batched():
    """Per-sample allowed sets without a block hint (learn.py:258-261: one
    scalar omp per sample in the reference) run as ONE ragged device call;
    each sample matches the oracle's restricted OMP over its sorted set."""
    import math

    import oracle as O
    from parity import compare
    from paper_1511_05174_b200.learn import code_stage
    rng = np.random.default_rng(17)
    n, t, m, k = 24, 60, 50, 5
    d = rng.standard_normal((n, t))
    d /= np.linalg.norm(d, axis=0)
    y = rng.standard_normal((n, m))
    sets = [frozenset((rng.choice(t, size=int(rng.integers(3, 30)), replace=False) + 1).tolist())
            for _ in range(m)]
    res = code_stage(d, y, k, sets, None)
    for p in range(m):
        allowed = np.array(sorted(sets[p]), dtype=np.int64)[None, :] - 1
        kp = min(k, len(sets[p]))
        eps = np.array([1e-6 * math.sqrt(y[:, p].dot(y[:, p]))])
        sel, coef, cnt, rn, sc, fl = O.omp_batch(np.ascontiguousarray(d.T), y[:, p][None, :], kp,
                                                 eps, allowed)
        got = res[p]
        assert list(got.selected) == (sel[0, :cnt[0]] + 1).tolist()
        assert got.atom_scan_count == int(sc[0])
        np.testing.assert_allclose(got.residual_norm, rn[0], rtol=1e-9)
