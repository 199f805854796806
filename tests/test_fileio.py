""".csd model files: the native reader against the
reference's own files, parses and error messages (tests/golden/csd_*); the
writer against the reference's bytes.  Host code only -- runs without a GPU."""

import os

import numpy as np
import pytest

from paper_1511_05174_b200 import errors as E
from paper_1511_05174_b200.crossscale import CrossScaleModel
from paper_1511_05174_b200.fileio import SingleScaleModel, load_model, save_model

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EXP = np.load(os.path.join(GOLD, "csd_expect.npz"))


def test_single_scale_file_parses_like_the_reference():
    m = load_model(os.path.join(GOLD, "csd_single.csd"))
    assert isinstance(m, SingleScaleModel)
    assert np.array_equal(m.dictionary.atoms, EXP["single_atoms"])
    assert m.patch_shape == tuple(EXP["single_shape"]) and m.sparsity == int(EXP["single_k"])


def test_cross_scale_file_parses_like_the_reference():
    m = load_model(os.path.join(GOLD, "csd_cross.csd"))
    assert isinstance(m, CrossScaleModel)
    assert np.array_equal(m.d_low.atoms, EXP["low_atoms"])
    assert np.array_equal(m.d_high.atoms, EXP["high_atoms"])
    assert m.scale.fine_shape == tuple(EXP["fine_shape"])
    assert m.scale.factors == tuple(EXP["factors"])
    assert (m.k_low, m.k_high) == (int(EXP["k_low"]), int(EXP["k_high"]))


@pytest.mark.parametrize("name", ["single", "cross"])
def test_writer_reproduces_reference_bytes(name, tmp_path):
    src = os.path.join(GOLD, f"csd_{name}.csd")
    out = tmp_path / f"{name}.csd"
    save_model(out, load_model(src))
    assert out.read_bytes() == open(src, "rb").read()


def test_bare_dictionary_needs_geometry(tmp_path):
    m = load_model(os.path.join(GOLD, "csd_single.csd"))
    with pytest.raises(E.DimensionError):
        save_model(tmp_path / "x.csd", m.dictionary)
    save_model(tmp_path / "x.csd", m.dictionary, patch_shape=m.patch_shape, sparsity=m.sparsity)
    assert (tmp_path / "x.csd").read_bytes() == open(os.path.join(GOLD, "csd_single.csd"),
                                                      "rb").read()


ERR = np.load(os.path.join(GOLD, "csd_errors.npz"))


@pytest.mark.parametrize("i", range(len(ERR["names"])))
def test_malformed_files_fail_like_the_reference(i):
    name, cls, msg = str(ERR["names"][i]), str(ERR["classes"][i]), str(ERR["msgs"][i])
    path = os.path.join(GOLD, f"csd_bad_{name}.csd")
    with pytest.raises(getattr(E, cls)) as info:
        load_model(path)
    assert str(info.value) == msg.replace("{path}", path)


def test_missing_file():
    with pytest.raises(FileNotFoundError):
        load_model(os.path.join(GOLD, "no_such_model.csd"))


@pytest.mark.gpu
def test_staged_model_codes_like_in_memory_model():
    from paper_1511_05174_b200.crossscale import zero_tree_many_arrays
    m = load_model(os.path.join(GOLD, "csd_cross.csd"), stage=True)
    ys = np.random.default_rng(3).standard_normal((16, 40))
    low, high, _ = zero_tree_many_arrays(m, ys)
    m2 = CrossScaleModel(type(m.d_low)(EXP["low_atoms"]), type(m.d_high)(EXP["high_atoms"]),
                         m.scale, m.k_low, m.k_high)
    low2, high2, _ = zero_tree_many_arrays(m2, ys)
    assert np.array_equal(high.sel, high2.sel) and np.array_equal(high.alpha, high2.alpha)
