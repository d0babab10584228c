"""Golden vectors produced by the unmodified reference engine
(tests/golden/make_golden.py).  The oracle must reproduce every one bit for
bit on CPU; the CUDA path (EXACT mode) must too on the GPU, and FAST mode
must match routing bit for bit and outputs within TOL_FAST.  Nothing here
reads /root/reference, so it runs on the GPU box."""
import os

import numpy as np
import pytest

from conftest import bits16, norm_err, to_dev, to_np

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))
TOL_FAST = 1e-2  # max|out-x - ref-x| / max|ref-x|  (BASELINE north_star: 1e-2)


def f16(a):
    return np.ascontiguousarray(a).view(np.float16)


def _small(bits):
    from oracle.oracle import random_layer
    lw = random_layer(64, 128, 8, seed=5000 + bits)
    g = {k[len(f"small{bits}_"):]: GOLD[k] for k in GOLD.files if k.startswith(f"small{bits}_")}
    q = (g["q1"], f16(g["s1"]), g["q2"], f16(g["s2"])) if bits != 16 else None
    return lw, g, q


# ------------------------------------------------------------------------ CPU
@pytest.mark.parametrize("bits", [4, 8])
def test_oracle_quantizer_golden(oracle, bits):
    w = f16(GOLD["quant_w"])
    p, s = oracle.quantize(w, bits)
    assert np.array_equal(p, GOLD[f"quant{bits}_packed"])
    assert np.array_equal(bits16(s), GOLD[f"quant{bits}_scales"])
    deq = oracle.dequantize(p, s, w.shape, bits)
    assert np.array_equal(bits16(deq), GOLD[f"quant{bits}_deq"])


@pytest.mark.parametrize("bits", [16, 8, 4])
def test_oracle_layer_golden(oracle, bits):
    lw, g, q = _small(bits)
    x = f16(g["x"])
    got, diag = oracle.moe_forward(lw, x, g["fin"], k=1, bits=bits, q=q, diagnostics=True)
    assert np.array_equal(bits16(got), g["out"])
    assert np.array_equal(diag["expert"][:, 0], g["expert"])
    assert np.array_equal(diag["scale"][:, 0], g["scale"])
    for key in ("perm", "inv", "offsets"):
        assert np.array_equal(diag[key], g[key]), key
    assert diag["active"] == int(g["active"][0])
    if bits != 16:
        q1, s1 = oracle.quantize(lw.w1, bits)
        assert np.array_equal(q1, g["q1"]) and np.array_equal(bits16(s1), g["s1"])


@pytest.mark.parametrize("bits", [16, 4])
def test_oracle_config1_golden(oracle, bits):
    from oracle.oracle import random_layer
    lw = random_layer(512, 2048, 8, seed=1)
    got = oracle.moe_forward(lw, f16(GOLD["c1_x"]), None, k=1, bits=bits)
    assert np.array_equal(bits16(got), GOLD[f"c1_{bits}_out"])


# ------------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("bits", [16, 8, 4])
def test_gpu_layer_golden(cuda, bits):
    from paper_2211_10017_b200.ops import MoELayer
    lw, g, q = _small(bits)
    L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits)
    if bits != 16:  # quantized ON THE GPU: codes/scales bit-exact with the reference
        assert np.array_equal(to_np(L.quant[0]), g["q1"])
        assert np.array_equal(bits16(to_np(L.quant[1])), g["s1"])
        assert np.array_equal(to_np(L.quant[2]), g["q2"])
    x = f16(g["x"])
    T = x.shape[0]
    for mode in (0, 1):
        out = to_np(L.forward(to_dev(x), to_dev(g["fin"]), k=1, mode=mode))
        r = L.routing(T, 1)
        assert np.array_equal(r["expert"][:, 0], g["expert"])
        assert np.array_equal(r["scale"][:, 0], g["scale"])
        for key in ("perm", "inv", "offsets"):
            assert np.array_equal(r[key], g[key]), key
        if mode == 0:
            assert np.array_equal(bits16(out), g["out"])
        else:
            xf = x.astype(np.float64)
            err = norm_err(out.astype(np.float64) - xf, f16(g["out"]).astype(np.float64) - xf)
            assert err <= TOL_FAST, err


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [16, 4])
def test_gpu_config1_golden(cuda, bits):
    from oracle.oracle import random_layer
    from paper_2211_10017_b200.ops import MoELayer
    lw = random_layer(512, 2048, 8, seed=1)
    L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits)
    x = f16(GOLD["c1_x"])
    want = f16(GOLD[f"c1_{bits}_out"])
    exact = to_np(L.forward(to_dev(x), None, k=1, mode=0))
    assert np.array_equal(bits16(exact), bits16(want))
    fast = L.forward_host(x, None, k=1, mode=1)  # host-buffer (drop-in) path
    xf = x.astype(np.float64)
    err = norm_err(fast.astype(np.float64) - xf, want.astype(np.float64) - xf)
    assert err <= TOL_FAST, err
