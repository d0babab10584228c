"""`.moec` checkpoint loader (csrc/moec.cu) against files
written by the UNMODIFIED reference (tests/golden/make_moec_golden.py:
random_model -> quantize_model -> save_model, proj/src/checkpoint.cpp).

CPU: header / record validation and the reference's error messages
("checkpoint: ...", RuntimeError).  GPU: every MoE block loaded straight
from the int4 / fp16 payloads runs bit-identically to the reference's
moe_ffn_forward on that block in EXACT mode, within tolerance in FAST."""
import os
import struct

import numpy as np
import pytest

from conftest import ROOT, bits16, layer_err, to_dev, to_np

GOLD = os.path.join(ROOT, "tests", "golden")
CFG = dict(d_model=64, d_ffn=128, n_enc_layers=2, n_dec_layers=2, n_experts=4, n_heads=4,
           vocab_size=16, moe_every=2, max_seq_len=8)


def _fnv1a(b):
    h = 0xcbf29ce484222325
    for c in b:
        h = ((h ^ c) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def _resealed(raw):
    body = raw[:-8]
    return body + struct.pack("<Q", _fnv1a(body))


@pytest.mark.parametrize("name,prec", [("model_int4.moec", "int4"), ("model_f16.moec", "f16")])
def test_moec_parse(name, prec):
    from paper_2211_10017_b200.moec import MoecModel
    m = MoecModel(os.path.join(GOLD, name), create_layers=False)
    assert m.config == CFG
    assert m.precision == prec
    assert [n for n, _ in m.blocks] == ["enc.0.ffn", "dec.0.ffn"]


def test_moec_errors(tmp_path):
    from paper_2211_10017_b200.moec import MoecModel
    raw = open(os.path.join(GOLD, "model_int4.moec"), "rb").read()
    cases = {
        "checksum mismatch": raw[:100] + bytes([raw[100] ^ 1]) + raw[101:],
        "bad magic": _resealed(b"MOEX" + raw[4:]),
        "unsupported version": _resealed(raw[:4] + struct.pack("<I", 2) + raw[8:]),
        "truncated file": _resealed(raw[:200] + raw[-8:]),
        "trailing bytes": _resealed(raw[:-8] + b"\0" * 4 + raw[-8:]),
    }
    for want, data in cases.items():
        p = tmp_path / "bad.moec"
        p.write_bytes(data)
        with pytest.raises(RuntimeError, match="checkpoint: " + want):
            MoecModel(str(p), create_layers=False)
    with pytest.raises(RuntimeError, match="checkpoint: cannot open"):
        MoecModel(str(tmp_path / "missing.moec"), create_layers=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name,bits", [("model_int4.moec", 4), ("model_f16.moec", 16)])
def test_moec_blocks_match_reference(cuda, name, bits):
    from paper_2211_10017_b200.moec import MoecModel
    g = np.load(os.path.join(GOLD, "moec_vectors.npz"))
    m = MoecModel(os.path.join(GOLD, name))
    for b, (nm, layer) in enumerate(m.blocks):
        x = g[f"b{bits}_{b}_x"].view(np.float16)
        fin = g[f"b{bits}_{b}_fin"]
        want = g[f"b{bits}_{b}_out"].view(np.float16)
        got = to_np(layer.forward(to_dev(x), to_dev(fin), k=1, mode=0))
        assert np.array_equal(bits16(got), bits16(want)), nm
        fast = to_np(layer.forward(to_dev(x), to_dev(fin), k=1, mode=1))
        assert layer_err(fast, want, x) <= 1e-2, nm
