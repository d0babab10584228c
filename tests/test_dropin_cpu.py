"""Drop-in module surface (CPU, no compute on the device): every hot-path
name of the reference's moeinfer package exists, host-side helpers match the
reference's test_smoke.py anchors, and argument validation raises the same
exception types before any device work."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def mi():
    return pytest.importorskip("paper_2211_10017_b200.moeinfer")


def test_reference_names_present(mi):
    for name in mi.REFERENCE_HOT_PATH_NAMES:
        assert hasattr(mi, name), name


def test_half_and_magic_constants(mi):
    # proj/tests/python/test_smoke.py:18-30 (host-side helpers)
    assert mi.f32_to_half(1.0) == 0x3C00
    assert mi.f32_to_half(-2.0) == 0xC000
    assert mi.half_to_f32(0x3C00) == 1.0
    assert mi.compose_magic(0) == 0x6400
    assert mi.compose_magic(3) == 0x6403
    assert mi.half_to_f32(mi.compose_magic(3)) == 1027.0
    assert mi.half_to_f32(mi.debias_const_u8()) == 1152.0
    assert mi.half_to_f32(mi.debias_const_u4()) == 1032.0
    assert mi.half_add(0x3C00, 0x3C00) == mi.f32_to_half(2.0)
    assert mi.half_mul(0x4000, 0x4000) == mi.f32_to_half(4.0)


def test_validation_errors_before_device(mi):
    with pytest.raises(ValueError, match="float16"):
        mi.quantize(np.zeros((1, 2, 8), np.float32), bits=4)
    with pytest.raises(ValueError, match="dimensions"):
        mi.quantize(np.zeros((2, 8), np.float16), bits=4)
    with pytest.raises(ValueError, match="bits must be 4 or 8"):
        mi.quantize(np.zeros((1, 2, 8), np.float16), bits=3)
    with pytest.raises(ValueError, match="divisible by 8"):
        mi.quantize(np.zeros((1, 2, 7), np.float16), bits=4)
    with pytest.raises(ValueError, match="multiple of 8"):
        mi.pack_int4_interleaved(np.zeros(7, np.uint8))
    with pytest.raises(ValueError, match="gate_top1"):
        mi.gate_top1(np.zeros((0, 3), np.float32))
    with pytest.raises(ValueError, match="numerics"):
        mi.set_numerics("sloppy")
