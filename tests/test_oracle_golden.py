"""Pin the C oracle (oracle/moe_oracle.c) to the reference's own known-answer
tests.  CPU only.  Every case cites the reference test it restates
(paths relative to /root/reference/proj)."""
import numpy as np
import pytest

from conftest import bits16


def h(x):
    return np.float16(x).view(np.uint16).item()


# --- half (tests/unit/test_half.cpp:54-66, 68-86) -----------------------------
def test_half_anchor_patterns(oracle):
    assert oracle.lib.or_f64_to_half(1024.0) == 0x6400
    assert oracle.lib.or_f64_to_half(1027.0) == 0x6403
    assert oracle.lib.or_f64_to_half(1032.0) == 0x6408
    assert oracle.lib.or_f64_to_half(1152.0) == 0x6480
    # RNE ties: 2049 sits halfway between 2048 and 2050 -> even (2048)
    assert oracle.lib.or_f64_to_half(2049.0) == 0x6800
    assert oracle.lib.or_f64_to_half(2051.0) == 0x6802  # -> 2052 (even mantissa)
    assert oracle.lib.or_f64_to_half(65520.0) == 0x7C00  # overflow -> inf
    assert oracle.lib.or_f64_to_half(2.0 ** -25) == 0x0000  # tie to even (zero)
    assert oracle.lib.or_f64_to_half(3 * 2.0 ** -26) == 0x0001


def test_half_round_trip_exhaustive(oracle):
    # every non-NaN pattern survives half -> f32 -> half (test_half.cpp:34-52)
    for b in range(0, 1 << 16, 7):  # stride keeps the CPU suite fast
        if (b & 0x7C00) == 0x7C00 and (b & 0x3FF):
            continue
        assert oracle.lib.or_f32_to_half(oracle.lib.or_half_to_f32(b)) == b


def test_half_ops_single_rounding(oracle):
    # half_add/mul round the exact result once (test_half.cpp:150-172)
    rng = np.random.default_rng(3)
    a = rng.standard_normal(500).astype(np.float16)
    b = rng.standard_normal(500).astype(np.float16)
    for x, y in zip(a, b):
        want_add = np.float16(np.float64(x) + np.float64(y)).view(np.uint16)
        want_mul = np.float16(np.float64(x) * np.float64(y)).view(np.uint16)
        assert oracle.lib.or_half_add(h(x), h(y)) == want_add
        assert oracle.lib.or_half_mul(h(x), h(y)) == want_mul


# --- quantizer (tests/unit/test_quantize.cpp) ----------------------------------
def test_quantize_worked_8bit(oracle):
    # test_quantize.cpp:42-53
    w = np.array([1.0, -1.0, 0.5], np.float16).reshape(1, 3, 1)
    packed, scales = oracle.quantize(w, 8)
    assert bits16(scales)[0, 0] == 0x2008
    assert list(packed) == [255, 1, 192]


def test_quantize_worked_4bit(oracle):
    # test_quantize.cpp:55-61
    w = h(0.7)
    s = oracle.lib.or_quant_scale(oracle.half_to_f32(w), 7)
    assert s == 0x2E67
    assert oracle.lib.or_quant_encode(w, s, 4) == 15
    assert oracle.lib.or_quant_encode(h(-0.7), s, 4) == 1


def test_pack_anchor(oracle):
    # test_quantize.cpp:182-197
    assert list(oracle.pack_int4(np.arange(8, dtype=np.uint8))) == [0x20, 0x64, 0x31, 0x75]
    rng = np.random.default_rng(0x20A5)
    for _ in range(50):
        v = rng.integers(0, 16, 8 * int(rng.integers(1, 17))).astype(np.uint8)
        assert np.array_equal(oracle.unpack_int4(oracle.pack_int4(v), len(v)), v)


def test_quantize_degenerate_channels(oracle):
    # test_quantize.cpp:199-219
    w = np.zeros((1, 4, 8), np.float16)
    packed, scales = oracle.quantize(w, 4)
    assert (bits16(scales) == 0x3C00).all()
    assert (oracle.unpack_int4(packed, 32) == 8).all()
    w = np.full((1, 4, 8), np.uint16(1), np.uint16).view(np.float16)  # min subnormal
    packed, scales = oracle.quantize(w, 8)
    assert (bits16(scales) == 0x0001).all()
    assert (packed == 129).all()


def test_quantize_validation(oracle):
    # test_quantize.cpp:232-249; quantize.cpp:76-86
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        oracle.quantize(np.zeros((1, 2, 7), np.float16), 4)
    w = np.zeros((1, 2, 8), np.float16)
    w[0, 1, 3] = np.inf
    with pytest.raises(OracleError, match="non-finite"):
        oracle.quantize(w, 4)


# --- dequant (tests/unit/test_dequant.cpp) --------------------------------------
def test_dequant_anchors(oracle):
    # test_dequant.cpp:34-48
    assert oracle.lib.or_debias_u8() == 0x6480
    assert oracle.lib.or_debias_u4() == 0x6408


def test_dequant_worked_example(oracle):
    # test_dequant.cpp:92-106
    packed = np.array([255, 1, 192], np.uint8)
    scales = np.array([0x2008], np.uint16).view(np.float16).reshape(1, 1)
    for fast in (True, False):
        out = bits16(oracle.dequantize(packed, scales, (1, 3, 1), 8, fast=fast)).ravel()
        assert list(out) == [0x3C00, 0xBC00, 0x3808]


def test_dequant_fast_equals_naive_all_codes(oracle):
    # test_dequant.cpp:50-90 (all codes x positions, random positive scales)
    rng = np.random.default_rng(0x30C1)
    for bits, ncode in ((8, 256), (4, 16)):
        n = 8 * ncode if bits == 4 else ncode
        codes = np.tile(np.arange(ncode, dtype=np.uint8), n // ncode)
        for _ in range(20):
            s = np.abs(rng.standard_normal(n) * 0.05).astype(np.float16).reshape(1, n)
            s[s == 0] = np.float16(1e-3)
            packed = oracle.pack_int4(codes) if bits == 4 else codes
            a = oracle.dequantize(packed, s, (1, 1, n), bits, fast=True)
            b = oracle.dequantize(packed, s, (1, 1, n), bits, fast=False)
            assert np.array_equal(bits16(a), bits16(b))


# --- routing (tests/unit/test_routing.cpp) --------------------------------------
def test_gate_worked_rows(oracle):
    # test_routing.cpp:50-78
    ex, sc = oracle.gate_topk(np.array([[1.0, 2.0, 0.5]], np.float32))
    assert ex[0, 0] == 1
    assert abs(float(np.uint16(sc[0, 0]).view(np.float16)) - 0.62853) <= 0.62853 * 2e-4
    ex, sc = oracle.gate_topk(np.array([[10.0, 0.0, 0.0]], np.float32))
    assert ex[0, 0] == 0 and float(np.uint16(sc[0, 0]).view(np.float16)) >= 0.999
    ex, _ = oracle.gate_topk(np.array([[5.0, 5.0, 1.0]], np.float32))
    assert ex[0, 0] == 0  # ties -> lowest index
    ex, _ = oracle.gate_topk(np.array([[1.0, 2.0, 0.5], [9.0, 1.0, 1.0]], np.float32))
    assert list(ex[:, 0]) == [1, 0]


def test_gate_rejects_non_finite(oracle):
    from oracle.oracle import OracleError
    for bad in (np.nan, np.inf):
        with pytest.raises(OracleError):
            oracle.gate_topk(np.array([[1.0, bad, 0.0]], np.float32))


def test_worked_routing_plan(oracle):
    # test_routing.cpp:105-117
    perm, inv, offs, active = oracle.routing_plan(np.array([2, 0, 2, 1], np.uint32),
                                                  np.array([0, 0, 1, 0], np.uint8), 3)
    assert active == 3
    assert list(perm) == [1, 3, 0, 2]
    assert list(inv) == [2, 0, 3, 1]
    assert list(offs) == [0, 1, 2, 3]


def test_plan_matches_stable_sort(oracle):
    # test_routing.cpp:119-138 (ref::routing_plan = std::stable_sort by key)
    rng = np.random.default_rng(0x40D1)
    for _ in range(300):
        T, E = int(rng.integers(1, 60)), int(rng.integers(1, 9))
        ex = rng.integers(0, E, T).astype(np.uint32)
        fin = (rng.random(T) < 0.3).astype(np.uint8)
        perm, inv, offs, active = oracle.routing_plan(ex, fin, E)
        key = np.where(fin == 1, E, ex)
        assert np.array_equal(perm, np.argsort(key, kind="stable"))
        assert np.array_equal(inv[perm], np.arange(T))
        assert active == int((fin == 0).sum())
        assert np.array_equal(offs, np.searchsorted(np.sort(key), np.arange(E + 1)))


def test_gemm_k_sequential(oracle):
    # test_gemm.cpp:126-140: 65504*65504 + 1 - 65504*65504 in k order must give 0
    x = np.array([[65504.0, 1.0, -65504.0]], np.float16)
    w = np.array([[65504.0], [1.0], [65504.0]], np.float16).reshape(1, 3, 1)
    probs = np.array([[0, 0, 1]], np.uint32)
    out, _ = oracle.grouped_gemm(x, probs, bits=16, w16=w, E=1, n=1,
                                 bias=np.zeros((1, 1), np.float16), relu=False)
    assert bits16(out)[0, 0] == 0x0000
