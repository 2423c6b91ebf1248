"""FHMT fixture files: the product's save/load
(fmha_tensor_save / fmha_tensor_load, C++ fmha_b200::save_tensor /
load_tensor) against the reference's save_tensor / load_tensor
(proj/src/tensor.cpp:30-84), and the reference's own I/O tests
(proj/tests/test_io.cpp:20-50) restated."""
import os

import numpy as np
import pytest

import paper_2312_11918_b200 as fm


def test_f32_round_trip_exact(tmp_path, oracle):
    """test_io.cpp:20-26."""
    t = oracle.gaussian(2, 16, 3, 8, 99)
    p = tmp_path / "t.fhmt"
    fm.save_tensor(t, p, "f32")
    np.testing.assert_array_equal(fm.load_tensor(p), t)


def test_f16_dump_rounds_to_nearest_even(tmp_path):
    """test_io.cpp:28-37."""
    t = np.array([0.1, 1.0], np.float32).reshape(1, 1, 1, 2)
    p = tmp_path / "h.fhmt"
    fm.save_tensor(t, p, "f16")
    r = fm.load_tensor(p)
    assert r[0, 0, 0, 0] == np.float32(0.0999755859375)
    assert r[0, 0, 0, 1] == 1.0


def test_header_and_precision_validation(tmp_path):
    """test_io.cpp:39-50."""
    t = np.zeros((1, 2, 1, 2), np.float32)
    with pytest.raises(ValueError):
        fm.save_tensor(t, tmp_path / "x.fhmt", "f64")
    bad = tmp_path / "bad.fhmt"
    bad.write_bytes(b"not a tensor")
    with pytest.raises(RuntimeError, match="bad magic"):
        fm.load_tensor(bad)
    with pytest.raises(RuntimeError, match="cannot open"):
        fm.load_tensor("/nonexistent/fmhasim.bin")
    trunc = tmp_path / "trunc.fhmt"
    fm.save_tensor(np.ones((1, 4, 1, 4), np.float32), trunc)
    trunc.write_bytes(trunc.read_bytes()[:-8])
    with pytest.raises(RuntimeError, match="truncated"):
        fm.load_tensor(trunc)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle",
                                                    "_ref", "libfmhasim_ref.so")), reason="oracle/_ref not built")
@pytest.mark.parametrize("f16", [False, True])
def test_cross_compatible_with_reference(tmp_path, oracle, f16):
    t = oracle.gaussian(2, 8, 3, 16, 5) * 3
    ours, theirs = str(tmp_path / "ours.fhmt"), str(tmp_path / "theirs.fhmt")
    fm.save_tensor(t, ours, "f16" if f16 else "f32")
    assert oracle.ref_save_tensor(theirs, t, f16) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()  # byte-identical files
    np.testing.assert_array_equal(oracle.ref_load_tensor(ours), fm.load_tensor(theirs))
