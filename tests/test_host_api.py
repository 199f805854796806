"""Host-side behaviour that needs no GPU: validation (raised before any
device call, with the reference's error classes), block map, cost model,
model invariants, scale maps -- ported from the reference's own tests
(pkg/tests/test_pursuit.py:142-155, test_crossscale.py:15-58, 458-482,
test_scaling.py:84-96)."""

import numpy as np
import pytest

from paper_1511_05174_b200 import (ConfigError, CrossScaleModel, DimensionError, DomainError,
                                   PursuitConfig, ScaleSpec, cross_scale_map, omp,
                                   omp_many_arrays, normalize_atoms, zero_tree_many_arrays)
from paper_1511_05174_b200.crossscale import omp_cost, predicted_speedup
from paper_1511_05174_b200.scaling import downsample_columns, upsample_columns


def test_validation_errors_match_reference():
    d = np.eye(4)
    with pytest.raises(ConfigError):
        omp(d, np.ones(4), PursuitConfig(5))
    with pytest.raises(ConfigError):
        omp(d, np.ones(4), PursuitConfig(3, allowed_support=frozenset({1, 2})))
    with pytest.raises(DomainError):
        omp(d, np.ones(4), PursuitConfig(1, allowed_support=frozenset({9})))
    with pytest.raises(DimensionError):
        omp(d, np.ones(3), PursuitConfig(1))
    with pytest.raises(ConfigError):
        PursuitConfig(0)
    with pytest.raises(ConfigError):
        PursuitConfig(1, residual_tolerance=-1.0)
    with pytest.raises(ConfigError):
        PursuitConfig(1, allowed_support=frozenset({0}))


def test_batched_validation():
    d = np.eye(4)
    with pytest.raises(DimensionError):
        omp_many_arrays(d, np.ones((3, 2)), PursuitConfig(1))
    with pytest.raises(ConfigError):
        omp_many_arrays(d, np.ones((4, 2)), PursuitConfig(5))
    with pytest.raises(ConfigError):
        omp_many_arrays(d, np.ones((4, 2)), PursuitConfig(1), allowed_blocks=np.zeros((2, 1)),
                        block_q=3)
    with pytest.raises(DimensionError):
        omp_many_arrays(d, np.ones((4, 2)), PursuitConfig(1), allowed_blocks=np.zeros((3, 1)),
                        block_q=2)
    with pytest.raises(DomainError):
        omp_many_arrays(d, np.ones((4, 2)), PursuitConfig(1),
                        allowed_blocks=np.full((2, 1), 2), block_q=2)


def test_empty_inputs_need_no_device():
    s = omp_many_arrays(np.eye(4), np.zeros((4, 0)), PursuitConfig(2))
    assert s.counts.shape == (0,) and s.sel.shape == (0, 2)
    res = omp(np.eye(4), np.ones(4), PursuitConfig(2, allowed_support=frozenset()))
    assert res.code.entries == () and res.residual_norm == pytest.approx(2.0)


def test_cross_scale_map_rules():
    assert cross_scale_map({1}, 16, 256) == frozenset(range(1, 17))
    assert cross_scale_map(set(), 4, 40) == frozenset()
    assert cross_scale_map({2, 5}, 4, 40) == frozenset({5, 6, 7, 8, 17, 18, 19, 20})
    rng = np.random.default_rng(0)
    for _ in range(50):
        q = int(rng.integers(1, 9))
        t_low = int(rng.integers(1, 30))
        omega = set(rng.choice(t_low, size=int(rng.integers(0, t_low + 1)), replace=False) + 1)
        assert len(cross_scale_map(omega, q, q * t_low)) == q * len(omega)
    for bad in (({0}, 4, 16), ({5}, 4, 16), ({1}, 3, 16)):
        with pytest.raises(DomainError):
            cross_scale_map(*bad)


def test_model_invariants():
    spec = ScaleSpec((8,), (2,))
    rng = np.random.default_rng(1)
    d_low = normalize_atoms(rng.standard_normal((4, 4)))
    d_high = normalize_atoms(rng.standard_normal((8, 8)))
    model = CrossScaleModel(d_low, d_high, spec, 2, 3)
    assert model.q == 2 and model.t_low == 4 and model.t_high == 8
    with pytest.raises(ConfigError):
        CrossScaleModel(d_low, normalize_atoms(rng.standard_normal((8, 6))), spec, 2, 3)
    with pytest.raises(ConfigError):
        CrossScaleModel(d_low, d_high, spec, 3, 2)
    with pytest.raises(ConfigError):
        CrossScaleModel(d_low, d_high, spec, 1, 3)
    with pytest.raises(DimensionError):
        CrossScaleModel(d_low, d_high, ScaleSpec((16,), (2,)), 2, 3)
    with pytest.raises(DimensionError):
        zero_tree_many_arrays(model, np.ones((7, 3)))


def test_cost_model():
    assert omp_cost(1, 1, 1) == 4.0
    assert omp_cost(2, 3, 4) == 2 * 3 * 4 + 3 * 4 + 4**4 + 4**3 * 2
    assert predicted_speedup(1024, 64, 8, 16) == pytest.approx(1024 / 192)
    assert predicted_speedup(100, 100, 0, 7) == 1.0
    with pytest.raises(DomainError):
        predicted_speedup(0, 1, 1, 1)
    with pytest.raises(DomainError):
        omp_cost(0, 1, 1)


def test_scale_maps_round_trip():
    rng = np.random.default_rng(3)
    spec = ScaleSpec((4, 4, 2), (2, 2, 2))
    z = rng.standard_normal((spec.coarse_size, 5))
    assert np.allclose(downsample_columns(upsample_columns(z, spec), spec), z)
    with pytest.raises(DimensionError):
        ScaleSpec((5, 4), (2, 2))
