"""install(): the reference's entry points are rebound to this package, its
result/error types are used, and uninstall() restores everything.  Needs the
reference importable (build container only); no device call is made."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture
def crossdict():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    import crossdict as cd
    yield cd
    sys.path.remove(REF)


def test_install_rebinds_and_restores(crossdict):
    import paper_1511_05174_b200 as b200
    orig = crossdict.pursuit.omp_many_arrays
    patched = b200.install()
    try:
        assert "crossdict.pursuit.omp_many_arrays" in patched
        assert "crossdict.pipelines.zero_tree_many_arrays" in patched
        # K-SVD coding stage and the patch pipeline ends
        assert "crossdict.learn._code_stage" in patched
        assert "crossdict.learn._update_stage" in patched
        assert "crossdict.learn._ksvd_core" in patched
        # .csd loading through the native reader, reference types out
        assert "crossdict.fileio.load_model" in patched
        gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
        m = crossdict.fileio.load_model(os.path.join(gold, "csd_cross.csd"))
        assert isinstance(m, crossdict.crossscale.CrossScaleModel)
        assert isinstance(m.d_high, crossdict.tensor.Dictionary)
        m1 = crossdict.fileio.load_model(os.path.join(gold, "csd_single.csd"))
        assert type(m1).__name__ == "SingleScaleModel" and type(m1).__module__.startswith("crossdict")
        assert "crossdict.patchwork.extract_patches" in patched
        assert "crossdict.pipelines.aggregate_patches" in patched
        # operator recovery
        assert "crossdict.pipelines._recover_operator" in patched
        import crossdict.learn as cl
        assert cl._code_stage is b200.learn.code_stage
        assert crossdict.pursuit.omp_many_arrays is b200.omp_many_arrays
        assert crossdict.crossscale.zero_tree_many_arrays is b200.zero_tree_many_arrays
        # validation happens on the host, with the reference's exception classes
        with pytest.raises(crossdict.errors.ConfigError):
            crossdict.pursuit.omp(np.eye(4), np.ones(4), crossdict.pursuit.PursuitConfig(5))
        with pytest.raises(crossdict.errors.DimensionError):
            crossdict.omp_many_arrays(np.eye(4), np.ones((3, 2)), crossdict.PursuitConfig(1))
        # empty batches need no device and come back as the reference's BatchSolve
        s = crossdict.omp_many_arrays(np.eye(4), np.zeros((4, 0)), crossdict.PursuitConfig(2))
        assert isinstance(s, crossdict.pursuit.BatchSolve)
        r = crossdict.omp(np.eye(4), np.ones(4),
                          crossdict.PursuitConfig(2, allowed_support=frozenset()))
        assert isinstance(r, crossdict.pursuit.PursuitResult)
        assert isinstance(r.code, crossdict.tensor.SparseCode)
    finally:
        b200.uninstall()
    assert crossdict.pursuit.omp_many_arrays is orig
    with pytest.raises(b200.errors.ConfigError):
        b200.omp(np.eye(4), np.ones(4), b200.PursuitConfig(5))
