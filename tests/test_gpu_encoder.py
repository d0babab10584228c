"""encoder_forward on the device (csrc/encoder.cu) against
the UNMODIFIED reference's encoder_forward (proj/src/model.cpp:351-398) over
the committed checkpoints (tests/golden/make_encoder_golden.py): EXACT mode
bit for bit, FAST mode within the layer tolerance."""
import os

import numpy as np
import pytest

from conftest import bits16

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
TOL_FAST = 1e-2


def _vectors():
    return np.load(os.path.join(GOLD, "encoder_vectors.npz"))


@pytest.mark.parametrize("name", ["model_int4", "model_f16"])
@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_encoder_matches_reference(cuda, name, case):
    from paper_2211_10017_b200.moec import MoecModel
    v = _vectors()
    tok, want = v[f"{name}_{case}_tok"], v[f"{name}_{case}_out"]
    m = MoecModel(os.path.join(GOLD, name + ".moec"))
    exact = m.encoder_forward(tok, mode=0).cpu().numpy().view(np.uint16)
    assert np.array_equal(exact, want), int((exact != want).sum())
    fast = m.encoder_forward(tok, mode=1).cpu().numpy().astype(np.float64)
    w = want.view(np.float16).astype(np.float64)
    err = np.abs(fast - w).max() / max(np.abs(w).max(), 1e-30)
    assert err <= TOL_FAST, err


def test_encoder_errors(cuda):
    from paper_2211_10017_b200.moec import MoecModel
    m = MoecModel(os.path.join(GOLD, "model_int4.moec"))
    with pytest.raises(ValueError, match="token id out of range"):
        m.encoder_forward(np.full((2, 3), 16, np.int32))
    with pytest.raises(ValueError, match="source length out of range"):
        m.encoder_forward(np.zeros((2, 9), np.int32))  # max_seq_len = 8
    with pytest.raises(ValueError, match="empty batch"):
        m.encoder_forward(np.zeros((0, 3), np.int32))
    # the same checkpoint without device layers has no encoder
    m2 = MoecModel(os.path.join(GOLD, "model_int4.moec"), create_layers=False)
    with pytest.raises(ValueError, match="without device layers"):
        m2.encoder_forward(np.zeros((1, 3), np.int32))


@pytest.mark.parametrize("bits", [4, 16])
def test_encoder_synthetic_checkpoint_matches_reference(cuda, tmp_path, bits):
    """A wider encoder (d=128, 8 heads of 16, 4 layers: two MoE, two dense,
    E=8) from moe_moec_write_synthetic: the reference's own loader and
    encoder_forward (oracle/_ref) against the device, EXACT bit for bit."""
    import ctypes as C
    from oracle.oracle import REF_SO
    from paper_2211_10017_b200 import abi
    from paper_2211_10017_b200.moec import MoecModel
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built")
    path = str(tmp_path / f"syn{bits}.moec")
    cfg = (C.c_uint32 * 9)(128, 256, 4, 1, 8, 8, 40, 2, 32)
    abi.call("moe_moec_write_synthetic", path.encode(), cfg, bits, 11)
    tok = np.random.default_rng(bits).integers(0, 40, (6, 16)).astype(np.int32)
    lib = C.CDLL(REF_SO)
    lib.ref_last_error.restype = C.c_char_p
    want = np.zeros((6 * 16, 128), np.uint16)
    st = lib.ref_encoder_forward(path.encode(), tok.ctypes.data_as(C.c_void_p), C.c_size_t(6),
                                 C.c_size_t(16), want.ctypes.data_as(C.c_void_p))
    assert st == 0, lib.ref_last_error()
    m = MoecModel(path)
    got = m.encoder_forward(tok, mode=0).cpu().numpy().view(np.uint16)
    assert np.array_equal(got, want), int((got != want).sum())


@pytest.mark.parametrize("length", [128, 100, 17])
def test_encoder_fast_attention_vs_exact(cuda, tmp_path, length):
    """FAST mode's tensor-core attention (mma.sync, flash-style in registers;
    64-wide heads, sentences up to 128 tokens, ragged lengths masked) against
    the bit-exact EXACT path on the same device, within the layer tolerance."""
    import ctypes as C
    from paper_2211_10017_b200 import abi
    from paper_2211_10017_b200.moec import MoecModel
    path = str(tmp_path / "syn_wide.moec")
    cfg = (C.c_uint32 * 9)(256, 512, 2, 1, 4, 4, 64, 2, 128)
    abi.call("moe_moec_write_synthetic", path.encode(), cfg, 4, 3)
    m = MoecModel(path)
    tok = np.random.default_rng(length).integers(0, 64, (3, length)).astype(np.int32)
    exact = m.encoder_forward(tok, mode=0).cpu().numpy().astype(np.float64)
    fast = m.encoder_forward(tok, mode=1).cpu().numpy().astype(np.float64)
    err = np.abs(fast - exact).max() / max(np.abs(exact).max(), 1e-30)
    assert err <= TOL_FAST, err
