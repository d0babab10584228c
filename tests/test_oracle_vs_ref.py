"""Pin the C oracle against the UNMODIFIED reference engine compiled from
/root/reference/proj/src (oracle/_ref/libmoeref.so, built by oracle/Makefile).
CPU only; skipped where the reference library was not built.  Bit-exact for
every output (codes, scales, LN, logits, decisions, plans, GEMM outputs,
traffic counters, whole-layer outputs)."""
import numpy as np
import pytest

from conftest import bits16


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("shape", [(1, 3, 8), (2, 17, 24), (3, 64, 128)])
def test_quantize_dequantize(oracle, ref, bits, shape):
    rng = np.random.default_rng(hash((bits,) + shape) & 0xFFFF)
    w = (rng.standard_normal(shape) * rng.uniform(0.01, 3)).astype(np.float16)
    w[0, 0, :] = 0  # a degenerate row (not channel) and a zero channel below
    w[:, :, 1] = 0
    po, so = oracle.quantize(w, bits)
    pr, sr = ref.quantize(w, bits)
    assert np.array_equal(po, pr)
    assert np.array_equal(bits16(so), bits16(sr))
    for fast in (True, False):
        a = oracle.dequantize(po, so, shape, bits, fast)
        b = ref.dequantize(pr, sr, shape, bits, fast)
        assert np.array_equal(bits16(a), bits16(b))


def test_quantize_thread_invariance(ref):
    rng = np.random.default_rng(5)
    w = rng.standard_normal((2, 40, 64)).astype(np.float16)
    a = ref.quantize(w, 4, threads=1)
    b = ref.quantize(w, 4, threads=7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(bits16(a[1]), bits16(b[1]))


@pytest.mark.parametrize("T,d,E", [(1, 8, 1), (37, 64, 8), (64, 512, 32)])
def test_layernorm_logits_gate_plan(oracle, ref, T, d, E):
    rng = np.random.default_rng(T * 1000 + d + E)
    x = (rng.standard_normal((T, d)) * 2).astype(np.float16)
    g = (1 + 0.1 * rng.standard_normal(d)).astype(np.float16)
    b = (0.05 * rng.standard_normal(d)).astype(np.float16)
    gw = (rng.standard_normal((d, E)) / np.sqrt(d)).astype(np.float16)
    gb = (0.02 * rng.standard_normal(E)).astype(np.float16)
    xn_o, xn_r = oracle.layer_norm(x, g, b), ref.layer_norm(x, g, b)
    assert np.array_equal(bits16(xn_o), bits16(xn_r))
    lo, lr = oracle.gate_logits(xn_o, gw, gb), ref.gate_logits(xn_r, gw, gb)
    assert np.array_equal(lo.view(np.uint32), lr.view(np.uint32))
    eo, so = oracle.gate_topk(lo, 1)
    er, sr = ref.gate_top1(lr)
    assert np.array_equal(eo[:, 0], er) and np.array_equal(so[:, 0], sr)
    fin = (rng.random(T) < 0.25).astype(np.uint8)
    assert all(np.array_equal(a, b) if isinstance(a, np.ndarray) else a == b
               for a, b in zip(oracle.routing_plan(eo, fin, E), ref.build_plan(er, fin, E)))


def test_gate_ties_and_extremes(oracle, ref):
    rows = np.array([[5, 5, 1, 5], [-3, -3, -3, -3], [80, -80, 0, 79.9], [0, 0, 0, 1e-30]],
                    np.float32)
    eo, so = oracle.gate_topk(rows, 1)
    er, sr = ref.gate_top1(rows)
    assert np.array_equal(eo[:, 0], er) and np.array_equal(so[:, 0], sr)


@pytest.mark.parametrize("bits", [16, 8, 4])
def test_grouped_gemm_and_traffic(oracle, ref, bits):
    rng = np.random.default_rng(77 + bits)
    E, m, n, rows = 5, 48, 40, 61
    x = rng.standard_normal((rows, m)).astype(np.float16)
    w = (rng.standard_normal((E, m, n)) / np.sqrt(m)).astype(np.float16)
    bias = (0.02 * rng.standard_normal((E, n))).astype(np.float16)
    probs = np.array([[0, 0, 10], [2, 10, 11], [3, 11, 50], [4, 50, 61]], np.uint32)
    kw = dict(E=E, n=n, bias=bias)
    if bits == 16:
        kw.update(w16=w)
    else:
        p, s = oracle.quantize(w, bits)
        kw.update(packed=p, scales=s)
    for relu in (False, True):
        for sep in ((False, True) if bits != 16 else (False,)):
            a, ta = oracle.grouped_gemm(x, probs, bits=bits, relu=relu, separate=sep, **kw)
            b, tb = ref.grouped_gemm(x, probs, bits=bits, relu=relu, separate=sep, **kw)
            assert np.array_equal(bits16(a), bits16(b))
            assert ta == tb


@pytest.mark.parametrize("bits", [16, 8, 4])
def test_moe_layer_forward(oracle, ref, bits):
    from oracle.oracle import random_layer
    d, f, E, T = 64, 128, 8, 45
    lw = random_layer(d, f, E, seed=900 + bits)
    rng = np.random.default_rng(bits)
    x = rng.standard_normal((T, d)).astype(np.float16)
    fin = (rng.random(T) < 0.2).astype(np.uint8)
    R = ref.layer(lw, bits)
    q = R.export_quant() if bits != 16 else None
    want = R.forward(x, fin)
    got = oracle.moe_forward(lw, x, fin, k=1, bits=bits, q=q)
    assert np.array_equal(bits16(got), bits16(want))
    assert np.array_equal(bits16(R.per_token(x, fin)), bits16(want))
    assert np.array_equal(bits16(oracle.moe_per_token(lw, x, fin, k=1, bits=bits, q=q)),
                          bits16(want))
    # threads never change results (test_model.cpp:332-340)
    assert np.array_equal(bits16(R.forward(x, fin, threads=5)), bits16(want))


def test_topk_extension_matches_reference_driver(oracle, ref):
    """k=2 (EXTENSION, SPEC.md:319 has top-1 only): the oracle's top-k layer
    equals the reference-function composition in oracle/ref_driver.cpp."""
    from oracle.oracle import random_layer
    lw = random_layer(64, 96, 8, seed=31)
    x = np.random.default_rng(1).standard_normal((29, 64)).astype(np.float16)
    fin = (np.arange(29) % 5 == 0).astype(np.uint8)
    R = ref.layer(lw, 4)
    q = R.export_quant()
    want = R.forward_topk(x, fin, k=2)
    got = oracle.moe_forward(lw, x, fin, k=2, bits=4, q=q)
    assert np.array_equal(bits16(got), bits16(want))
