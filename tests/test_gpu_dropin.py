"""The drop-in Python module (paper_2211_10017_b200.moeinfer == the
reference's moeinfer API for the hot path) on the GPU: the reference's own
smoke tests (proj/tests/python/test_smoke.py:33-114) plus bit-exact parity
with the compiled reference via the golden vectors, and the additive layer
API."""
import os

import numpy as np
import pytest

from conftest import bits16, layer_err

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))


@pytest.fixture(scope="module")
def mi(cuda):
    import paper_2211_10017_b200.moeinfer as m
    m.set_numerics("exact")
    return m


def bits(a):
    return a.view(np.uint16)


@pytest.mark.parametrize("bits_", [8, 4])
def test_dequantize_fast_matches_naive(mi, bits_):
    rng = np.random.default_rng(100 + bits_)
    w = rng.standard_normal((4, 16, 32)).astype(np.float16)
    qw = mi.quantize(w, bits=bits_)
    assert qw.bits == bits_ and qw.shape == (4, 16, 32)
    assert np.array_equal(bits(mi.dequantize_fast(qw)), bits(mi.dequantize_naive(qw)))
    codes = 4 * 16 * 32 if bits_ == 8 else 4 * 16 * 32 // 2
    assert qw.packed_bytes == codes and qw.scale_bytes == 4 * 32 * 2
    assert qw.payload_bytes == codes + 4 * 32 * 2


def test_int4_interleave_anchor(mi):
    packed = mi.pack_int4_interleaved(np.arange(8, dtype=np.uint8))
    assert list(packed) == [0x20, 0x64, 0x31, 0x75]
    assert list(mi.unpack_int4_interleaved(packed, 8)) == list(range(8))


def test_routing_plan_invariants(mi):
    rng = np.random.default_rng(7)
    rows, experts = 33, 5
    logits = rng.standard_normal((rows, experts)).astype(np.float32)
    decisions = mi.gate_top1(logits)
    assert [d.expert for d in decisions] == list(np.argmax(logits, axis=1))
    finished = (rng.random(rows) < 0.25).astype(np.uint8)
    plan = mi.build_routing_plan(decisions, finished, experts)
    assert sorted(plan.permutation) == list(range(rows))
    assert plan.active_rows == rows - int(finished.sum())
    offs = list(plan.expert_offsets)
    assert offs[0] == 0 and offs[-1] == plan.active_rows
    for e in range(experts):
        for i in range(offs[e], offs[e + 1]):
            r = plan.permutation[i]
            assert decisions[r].expert == e and not finished[r]
    inv = plan.inverse_permutation
    assert all(inv[plan.permutation[i]] == i for i in range(rows))


def test_grouped_gemm_paths_agree(mi):
    rng = np.random.default_rng(21)
    rows, m, n, experts = 24, 16, 32, 4
    x = rng.standard_normal((rows, m)).astype(np.float16)
    w = (rng.standard_normal((experts, m, n)) * 0.25).astype(np.float16)
    bias = (rng.standard_normal((experts, n)) * 0.05).astype(np.float16)
    decisions = mi.gate_top1(rng.standard_normal((rows, experts)).astype(np.float32))
    plan = mi.build_routing_plan(decisions, np.zeros(rows, np.uint8), experts)
    xs = mi.permute_rows(x, plan)
    y16, tc16 = mi.grouped_gemm(xs, plan, w, bias, relu=True)
    qw = mi.quantize(w, bits=8)
    y_fused, tc_fused = mi.grouped_gemm_quant(xs, plan, qw, bias, relu=True)
    y_sep, tc_sep = mi.grouped_gemm_quant(xs, plan, qw, bias, relu=True, fused=False)
    assert np.array_equal(bits(y_fused), bits(y_sep))
    y_ref, _ = mi.grouped_gemm(xs, plan, mi.dequantize_naive(qw), bias, relu=True)
    assert np.array_equal(bits(y_fused), bits(y_ref))
    assert tc_fused.total_read < tc_sep.total_read
    assert tc_fused.bytes_written < tc_sep.bytes_written
    _, tc4 = mi.grouped_gemm_quant(xs, plan, mi.quantize(w, bits=4), bias, relu=True)
    assert tc16.weight_bytes_read > tc_fused.weight_bytes_read > tc4.weight_bytes_read
    dense = np.zeros((rows, n), np.float64)
    for i, r in enumerate(plan.permutation):
        e = decisions[r].expert
        dense[i] = np.maximum(xs[i].astype(np.float64) @ w[e].astype(np.float64)
                              + bias[e].astype(np.float64), 0.0)
    assert np.allclose(y16.astype(np.float64), dense, atol=2e-2)


def test_quantize_matches_reference_golden(mi):
    w = GOLD["quant_w"].view(np.float16)
    for b in (4, 8):
        qw = mi.quantize(w, bits=b)
        assert np.array_equal(qw.packed, GOLD[f"quant{b}_packed"])
        assert np.array_equal(bits16(qw.scales), GOLD[f"quant{b}_scales"])
        assert np.array_equal(bits16(mi.dequantize_fast(qw)), GOLD[f"quant{b}_deq"])


@pytest.mark.parametrize("b", [16, 8, 4])
def test_moe_ffn_forward_bit_exact_with_reference(mi, b):
    """moe_ffn_forward (value API, exact numerics) == the compiled reference's
    output and traffic, for the golden small layers."""
    from oracle.oracle import random_layer
    lw = random_layer(64, 128, 8, seed=5000 + b)
    x = GOLD[f"small{b}_x"].view(np.float16)
    fin = GOLD[f"small{b}_fin"]
    if b == 16:
        w1, w2 = lw.w1, lw.w2
    else:
        w1, w2 = mi.quantize(lw.w1, bits=b), mi.quantize(lw.w2, bits=b)
        assert np.array_equal(w1.packed, GOLD[f"small{b}_q1"])
    out, tr = mi.moe_ffn_forward(x, lw.ln_g, lw.ln_b, lw.gw, lw.gb, w1, lw.b1, w2, lw.b2, fin)
    assert np.array_equal(bits16(out), GOLD[f"small{b}_out"])
    assert tr.expert.weight_bytes_read > 0 and tr.other.bytes_written > 0
    layer = mi.MoeLayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, w1, lw.b1, w2, lw.b2)
    assert np.array_equal(bits16(layer.forward(x, fin, numerics="exact")), GOLD[f"small{b}_out"])
    fast = layer.forward(x, fin, numerics="fast")
    assert layer_err(fast, GOLD[f"small{b}_out"].view(np.float16), x) <= 1e-2


def test_errors_map_like_the_reference(mi):
    with pytest.raises(ValueError, match="non-finite"):
        w = np.zeros((1, 4, 8), np.float16)
        w[0, 2, 3] = np.inf
        mi.quantize(w, bits=4)
    with pytest.raises(ValueError, match="non-finite logit"):
        mi.gate_top1(np.array([[1.0, np.nan]], np.float32))
    qw = mi.quantize(np.ones((2, 4, 8), np.float16), bits=4)
    with pytest.raises(IndexError):
        qw.unpack_expert(5)


def test_cpp_quantize_model(cuda, tmp_path):
    """C++ drop-in quantize_model (reference model.hpp:118): built with g++
    against libmoeinfer_b200.so and run (tests/native/dropin_quantize_model.cpp)."""
    import os
    import subprocess
    from conftest import ROOT
    pkg = os.path.join(ROOT, "paper_2211_10017_b200")
    exe = str(tmp_path / "dq")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "dropin_quantize_model.cpp"),
                    "-L", pkg, "-lmoeinfer_b200", "-lmoe_cuda", f"-Wl,-rpath,{pkg}"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
