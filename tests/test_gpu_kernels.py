"""GPU parity: each sm_100a kernel vs the C oracle (oracle/moe_oracle.c), on
the same seeded inputs.  Bit-exact for quantizer codes/scales, dequant,
LayerNorm, gate logits, top-k decisions/scales, routing plans and the
EXACT-mode GEMM; FAST-mode (tcgen05) GEMM within the stated tolerance
(TOL_FAST, normalized max error)."""
import numpy as np
import pytest

from conftest import bits16, norm_err, to_dev, to_np

pytestmark = pytest.mark.gpu

TOL_FAST = 1e-2  # max|gpu-ref| / max|ref|, f32-accumulated int4/int8/fp16 weights


def _ops():
    from paper_2211_10017_b200 import ops
    return ops


# --------------------------------------------------------------------- quantize
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("shape", [(1, 3, 8), (2, 16, 8), (8, 64, 16), (3, 7, 24), (4, 33, 136),
                                   (3, 301, 264), (2, 1024, 520)])
def test_quantize_matches_oracle(cuda, oracle, bits, shape):
    rng = np.random.default_rng(hash((bits,) + shape) % 2**32)
    w = rng.uniform(-4, 4, shape).astype(np.float16)
    p_ref, s_ref = oracle.quantize(w, bits)
    p, s = _ops().quantize(to_dev(w), bits)
    assert np.array_equal(to_np(p), p_ref)
    assert np.array_equal(bits16(to_np(s)), bits16(s_ref))


def test_quantize_int8_ragged_columns(cuda, oracle):
    """int8 with n % 8 != 0 (the scalar per-column kernel)."""
    rng = np.random.default_rng(12)
    for shape in [(2, 17, 12), (1, 5, 3), (3, 40, 100)]:
        w = rng.uniform(-3, 3, shape).astype(np.float16)
        p_ref, s_ref = oracle.quantize(w, 8)
        p, s = _ops().quantize(to_dev(w), 8)
        assert np.array_equal(to_np(p), p_ref)
        assert np.array_equal(bits16(to_np(s)), bits16(s_ref))


def test_quantize_half_integer_quotients(cuda, oracle):
    """Weights placed exactly on and one ulp around code boundaries (w = (j +
    0.5) * s): round-half-away must match llround(f64 w / f64 s)."""
    rng = np.random.default_rng(5)
    for bits, qmax in ((4, 7), (8, 127)):
        s = np.float16(2.0 ** -6)  # qmax * s and (j + 0.5) * s are exact in fp16
        m, n = 64, 16
        w = np.zeros((1, m, n), np.float16)
        w[0, 0, :] = np.float16(qmax) * s  # pins maxabs -> the scale s
        j = rng.integers(-qmax, qmax, (m - 1, n)).astype(np.float64) + 0.5
        v = (j * np.float64(s)).astype(np.float16)
        bump = rng.integers(-1, 2, v.shape).astype(np.int16)
        v = (v.view(np.int16) + bump).view(np.float16)
        w[0, 1:, :] = v
        p_ref, s_ref = oracle.quantize(w, bits)
        p, sc = _ops().quantize(to_dev(w), bits)
        assert np.array_equal(to_np(p), p_ref)
        assert np.array_equal(bits16(to_np(sc)), bits16(s_ref))


@pytest.mark.parametrize("bits", [8, 4])
def test_quantize_degenerate_and_subnormal(cuda, oracle, bits):
    w = np.zeros((2, 24, 8), np.float16)
    w[0, :, 1] = np.float16(2.0**-24)            # smallest subnormals
    w[0, :, 2] = np.float16(6e-8) * np.arange(24)  # tiny, scale toward subnormal
    w[1] = (np.random.default_rng(3).standard_normal((24, 8)) * 2.0**-18).astype(np.float16)
    w[1, :, 5] = -0.0
    p_ref, s_ref = oracle.quantize(w, bits)
    p, s = _ops().quantize(to_dev(w), bits)
    assert np.array_equal(to_np(p), p_ref)
    assert np.array_equal(bits16(to_np(s)), bits16(s_ref))


def test_quantize_rejects_non_finite_like_reference(cuda):
    w = np.zeros((1, 2, 8), np.float16)
    w[0, 1, 2] = np.inf
    w[0, 1, 5] = np.nan
    with pytest.raises(ValueError, match="non-finite weight at flat index 10"):
        _ops().quantize(to_dev(w), 8)
    with pytest.raises(ValueError, match="divisible by 8"):
        _ops().quantize(to_dev(np.zeros((1, 2, 6), np.float16)), 4)


def test_pack_unpack_int4_anchor(cuda, oracle):
    import torch
    v = torch.arange(8, dtype=torch.uint8, device="cuda")
    p = _ops().pack_int4(v)
    assert list(to_np(p)) == [0x20, 0x64, 0x31, 0x75]
    assert list(to_np(_ops().unpack_int4(p, 8))) == list(range(8))
    rng = np.random.default_rng(5)
    vals = rng.integers(0, 16, 8 * 97).astype(np.uint8)
    assert np.array_equal(to_np(_ops().pack_int4(to_dev(vals))), oracle.pack_int4(vals))
    with pytest.raises(ValueError, match="nibble"):
        _ops().pack_int4(to_dev(np.full(8, 16, np.uint8)))


# ------------------------------------------------------------------ dequantize
@pytest.mark.parametrize("fast", [True, False])
def test_dequant_exhaustive_codes_and_scales(cuda, oracle, fast):
    """Acceptance C1 domain (acceptance_main.cpp:88-128): every int8 code,
    every int4 code in every lane, 1000 random positive FP16 scales incl.
    subnormals -- bit-exact vs the oracle."""
    rng = np.random.default_rng(0xACC0001)
    scales = (1 + rng.integers(0, 0x7BFF, 1000)).astype(np.uint16).view(np.float16)
    # int8: 1000 experts of a 16x16 slab holding all 256 codes
    E = 1000
    p8 = np.tile(np.arange(256, dtype=np.uint8), E)
    s8 = np.repeat(scales[:, None], 16, axis=1)
    got8 = to_np(_ops().dequantize(to_dev(p8), to_dev(s8), (E, 16, 16), 8, fast))
    want8 = oracle.dequantize(p8, s8, (E, 16, 16), 8, fast)
    assert np.array_equal(bits16(got8), bits16(want8))
    # int4: code mi in lane ni, m=16 x n=8
    logical = np.repeat(np.arange(16, dtype=np.uint8)[:, None], 8, axis=1).reshape(-1)
    p4 = np.tile(oracle.pack_int4(logical), E)
    s4 = np.repeat(scales[:, None], 8, axis=1)
    got4 = to_np(_ops().dequantize(to_dev(p4), to_dev(s4), (E, 16, 8), 4, fast))
    want4 = oracle.dequantize(p4, s4, (E, 16, 8), 4, fast)
    assert np.array_equal(bits16(got4), bits16(want4))


def test_dequant_worked_example(cuda):
    # test_dequant.cpp:92-106: codes {255,1,192}, scale 0x2008
    out = to_np(_ops().dequantize(to_dev(np.array([255, 1, 192], np.uint8)),
                                  to_dev(np.array([[0x2008]], np.uint16).view(np.float16)),
                                  (1, 3, 1), 8, True))
    assert list(bits16(out).reshape(-1)) == [0x3C00, 0xBC00, 0x3808]


# ---------------------------------------------------------------------- gating
@pytest.mark.parametrize("T,d,E", [(1, 8, 1), (33, 64, 8), (257, 512, 8), (64, 1024, 64),
                                   (130, 2048, 128), (5, 40, 3)])
def test_layer_norm_and_logits_bit_exact(cuda, oracle, T, d, E):
    rng = np.random.default_rng(T * 1000 + d + E)
    x = rng.standard_normal((T, d)).astype(np.float16)
    g = (1 + 0.1 * rng.standard_normal(d)).astype(np.float16)
    b = (0.05 * rng.standard_normal(d)).astype(np.float16)
    gw = (rng.standard_normal((d, E)) / np.sqrt(d)).astype(np.float16)
    gb = (0.02 * rng.standard_normal(E)).astype(np.float16)
    xn_ref = oracle.layer_norm(x, g, b)
    xn = _ops().layer_norm(to_dev(x), to_dev(g), to_dev(b))
    assert np.array_equal(bits16(to_np(xn)), bits16(xn_ref))
    lg_ref = oracle.gate_logits(xn_ref, gw, gb)
    lg = to_np(_ops().gate_logits(xn, to_dev(gw), to_dev(gb)))
    assert np.array_equal(lg.view(np.uint32), lg_ref.view(np.uint32))


@pytest.mark.parametrize("k", [1, 2, 3])
def test_gate_topk_bit_exact(cuda, oracle, k):
    rng = np.random.default_rng(40 + k)
    for E in (k, 3, 8, 64, 128):
        if E < k:
            continue
        lg = (rng.standard_normal((500, E)) * 8).astype(np.float32)
        lg[::7, : min(E, 3)] = lg[::7, :1]  # ties -> lowest index
        lg[3] = -90.0                        # expf underflow region
        lg[4, 0] = 0.0
        ex_ref, sc_ref = oracle.gate_topk(lg, k)
        ex, sc = _ops().gate_topk(to_dev(lg), k)
        assert np.array_equal(to_np(ex), ex_ref)
        assert np.array_equal(bits16(to_np(sc)), sc_ref)


def test_gate_worked_rows_and_rejection(cuda):
    ex, sc = _ops().gate_topk(to_dev(np.array([[1, 2, 0.5], [5, 5, 1], [10, 0, 0]], np.float32)))
    e = to_np(ex).reshape(-1)
    s = to_np(sc).astype(np.float64).reshape(-1)
    assert list(e) == [1, 0, 0]
    assert abs(s[0] - 0.62853) < 0.62853 * 2e-4
    assert s[2] >= 0.999
    with pytest.raises(ValueError, match="non-finite logit at row 1"):
        _ops().gate_topk(to_dev(np.array([[1, 2], [np.nan, 0], [np.inf, 0]], np.float32)))


# --------------------------------------------------------------------- routing
@pytest.mark.parametrize("k", [1, 2])
def test_routing_plan_bit_exact_many(cuda, oracle, k):
    """10^3 random instances (test_routing.cpp:119-138 style) + big ones."""
    rng = np.random.default_rng(0x40D1 + k)
    cases = [(int(rng.integers(1, 65)), int(rng.integers(max(1, k), 17)), i % 3)
             for i in range(300)]
    cases += [(4096, 8, 0), (16384, 64, 1), (5000, 128, 1), (1, 1, 0), (3, 5, 2)]
    for T, E, mode in cases:
        if E < k:
            continue
        ex = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.uint32)
        fin = np.zeros(T, np.uint8) if mode == 0 else (
            np.ones(T, np.uint8) if mode == 2 else (rng.random(T) < 0.3).astype(np.uint8))
        perm_r, inv_r, off_r, act_r = oracle.routing_plan(ex, fin, E)
        perm, inv, off, probs, act = _ops().routing_plan(to_dev(ex), to_dev(fin), E)
        assert np.array_equal(to_np(perm), perm_r)
        assert np.array_equal(to_np(inv), inv_r)
        assert np.array_equal(to_np(off), off_r)
        assert int(to_np(act)[0]) == act_r
        pr = to_np(probs).reshape(-1, 3)
        assert np.array_equal(pr[:, 1], off_r[:-1]) and np.array_equal(pr[:, 2], off_r[1:])


def test_routing_worked_plan_and_validation(cuda):
    ex = np.array([[2], [0], [2], [1]], np.uint32)
    perm, inv, off, _, act = _ops().routing_plan(to_dev(ex), to_dev(np.array([0, 0, 1, 0],
                                                                              np.uint8)), 3)
    assert list(to_np(perm)) == [1, 3, 0, 2]
    assert list(to_np(inv)) == [2, 0, 3, 1]
    assert list(to_np(off)) == [0, 1, 2, 3]
    with pytest.raises(ValueError, match="expert out of range"):
        _ops().routing_plan(to_dev(np.array([[5]], np.uint32)), None, 3)


def test_permute_unpermute_combine(cuda, oracle):
    rng = np.random.default_rng(0x40D3)
    T, cols, E = 37, 24, 4
    x = rng.standard_normal((T, cols)).astype(np.float16)
    ex = rng.integers(0, E, (T, 1)).astype(np.uint32)
    sc = (0.25 + 0.5 * rng.random((T, 1))).astype(np.float16)
    fin = np.zeros(T, np.uint8)
    fin[[3, 7]] = 1
    perm_r, inv_r, off_r, act_r = oracle.routing_plan(ex, fin, E)
    perm, inv, off, probs, act = _ops().routing_plan(to_dev(ex), to_dev(fin), E)
    xp = _ops().permute_rows(to_dev(x), perm)
    assert np.array_equal(bits16(to_np(xp)), bits16(x[perm_r]))
    back = _ops().unpermute_scale(xp, perm, act, to_dev(sc.reshape(-1)))
    # fp16 x fp16 is exact in f32, so this is the single RN16 of half_mul
    want = (x.astype(np.float32) * sc.astype(np.float32)).astype(np.float16)
    want[fin == 1] = 0
    assert np.array_equal(bits16(to_np(back)), bits16(want))
    # combine (k=1): out = finished ? x : x (+) y*s, with y = the permuted x
    out = _ops().combine(to_dev(x), xp, inv, to_dev(sc), to_dev(fin))
    cw = (x.astype(np.float32) + want.astype(np.float32)).astype(np.float16)
    cw[fin == 1] = x[fin == 1]
    assert np.array_equal(bits16(to_np(out)), bits16(cw))


# ----------------------------------------------------------------- grouped GEMM
def _gemm_case(rng, rows, E, m, n, bits, fin_frac=0.1):
    ex = rng.integers(0, E, (rows, 1)).astype(np.uint32)
    fin = (rng.random(rows) < fin_frac).astype(np.uint8)
    x = rng.standard_normal((rows, m)).astype(np.float16)
    w = (0.25 * rng.standard_normal((E, m, n))).astype(np.float16)
    bias = (0.05 * rng.standard_normal((E, n))).astype(np.float16)
    return ex, fin, x, w, bias


def _run_gemm(oracle, ex, fin, x, w, bias, bits, relu, mode, sample=None):
    """GPU grouped GEMM over the plan-sorted rows vs the oracle.  sample=N:
    the oracle computes only N random live rows (large shapes); returns
    (got rows, want rows) for those rows."""
    ops = _ops()
    E, m, n = w.shape
    perm_r, inv_r, off_r, act_r = oracle.routing_plan(ex, fin, E)
    probs = oracle.make_problems(off_r)
    xs = x[perm_r]
    sel = None
    if sample is not None and act_r > sample:
        sel = np.sort(np.random.default_rng(act_r).choice(act_r, size=sample, replace=False))
        key = np.searchsorted(off_r[1:], sel, side="right")  # expert of each sampled row
        o_probs = np.array([[e, np.searchsorted(key, e), np.searchsorted(key, e, "right")]
                            for e in np.unique(key)], np.uint32)
        o_x = xs[sel]
    else:
        o_probs, o_x = probs, xs
    if bits == 16:
        want, _ = oracle.grouped_gemm(o_x, o_probs, bits=16, w16=w, E=E, n=n, bias=bias,
                                      relu=relu)
        tiled = ops.tile_weights(to_dev(w), E, m, n, 16)
        sc = None
    else:
        packed, scales = oracle.quantize(w, bits)
        want, _ = oracle.grouped_gemm(o_x, o_probs, bits=bits, packed=packed, scales=scales,
                                      E=E, n=n, bias=bias, relu=relu)
        tiled = ops.tile_weights(to_dev(packed), E, m, n, bits)
        sc = to_dev(scales)
    pr = to_dev(probs.astype(np.uint32)) if len(probs) else to_dev(np.zeros((0, 3), np.uint32))
    got = to_np(ops.grouped_gemm(to_dev(xs), pr, tiled, sc, bits, E, n, to_dev(bias), relu, mode))
    if sel is not None:
        return got[sel], want
    return got, want


@pytest.mark.parametrize("bits", [16, 8, 4])
def test_gemm_exact_bit_exact(cuda, oracle, bits):
    rng = np.random.default_rng(0x50E0 + bits)
    for trial in range(25):
        rows = int(rng.integers(1, 70))
        E = int(rng.integers(1, 7))
        m = int(rng.integers(1, 150))
        n = 8 * int(rng.integers(1, 40)) if bits == 4 else int(rng.integers(1, 300))
        ex, fin, x, w, bias = _gemm_case(rng, rows, E, m, n, bits)
        got, want = _run_gemm(oracle, ex, fin, x, w, bias, bits, trial % 2 == 0, _ops().MODE_EXACT)
        assert np.array_equal(bits16(got), bits16(want)), (trial, rows, E, m, n)


def test_gemm_exact_k_sequential(cuda):
    """test_gemm.cpp:126-140: 65504^2 + 1 - 65504^2 must give exactly +0."""
    ops = _ops()
    x = np.array([[65504.0, 1.0, 65504.0]], np.float16)
    w = np.array([[[65504.0], [1.0], [-65504.0]]], np.float16)
    tiled = ops.tile_weights(to_dev(w), 1, 3, 1, 16)
    got = ops.grouped_gemm(to_dev(x), to_dev(np.array([[0, 0, 1]], np.uint32)), tiled, None, 16,
                           1, 1, to_dev(np.zeros((1, 1), np.float16)), False, ops.MODE_EXACT)
    assert bits16(to_np(got))[0, 0] == 0x0000


@pytest.mark.parametrize("bits", [4, 8, 16])
@pytest.mark.parametrize("shape", [(300, 8, 512, 2048), (40, 4, 128, 256), (2000, 8, 2048, 512),
                                   (7, 3, 64, 128), (5000, 64, 1024, 256), (3000, 8, 512, 136),
                                   (3000, 8, 512, 200), (800, 4, 256, 72)])
def test_gemm_fast_tcgen05_within_tolerance(cuda, oracle, bits, shape):
    rows, E, m, n = shape
    rng = np.random.default_rng(rows + E + m + n + bits)
    ex, fin, x, w, bias = _gemm_case(rng, rows, E, m, n, bits, fin_frac=0.05)
    # large shapes: the scalar oracle computes 256 sampled rows (every row of
    # the GPU output is still produced by the full launch)
    sample = 256 if rows * m * n > 600e6 else None
    got, want = _run_gemm(oracle, ex, fin, x, w, bias, bits, True, _ops().MODE_FAST,
                          sample=sample)
    if sample is None:
        active = int((fin == 0).sum())
        got, want = got[:active], want[:active]
    err = norm_err(got, want)
    assert err <= TOL_FAST, err


def test_gemm_fast_equals_exact_semantics_large(cuda, oracle):
    """Full C2-size FFN1 (8192 slots x 512 -> 2048, int4): fast vs exact on
    the GPU (exact is bit-identical to the oracle at every size tested)."""
    ops = _ops()
    rng = np.random.default_rng(77)
    E, m, n, rows = 8, 512, 2048, 8192
    ex, fin, x, w, bias = _gemm_case(rng, rows, E, m, n, 4, fin_frac=0.0)
    perm_r, inv_r, off_r, act_r = oracle.routing_plan(ex, fin, E)
    probs = to_dev(oracle.make_problems(off_r))
    packed, scales = ops.quantize(to_dev(w), 4)
    tiled = ops.tile_weights(packed, E, m, n, 4)
    xs = to_dev(x[perm_r])
    a = ops.grouped_gemm(xs, probs, tiled, scales, 4, E, n, to_dev(bias), True, ops.MODE_EXACT)
    b = ops.grouped_gemm(xs, probs, tiled, scales, 4, E, n, to_dev(bias), True, ops.MODE_FAST)
    assert norm_err(to_np(b), to_np(a)) <= TOL_FAST


@pytest.mark.parametrize("bits", [4, 8, 16])
@pytest.mark.parametrize("sizes,m,n", [
    ([1000, 17, 1, 1500, 257, 999, 2048, 2182], 512, 2048),   # CTA pairs, 256-token SS tiles
    ([672] * 8, 512, 2048),                                   # CTA pairs, 224-token TS tiles
    ([300, 15, 33, 224, 225, 480, 600, 0, 431], 520, 1024),   # pairs, ragged + K tail
    ([64, 70, 33, 95, 1, 0, 80, 50, 96, 17], 512, 1024),      # pairs, 96-token tiles (C5-like)
    ([64] * 16, 1024, 2048),                                  # pairs, 96-token tiles, 64 rows
])
def test_gemm_fast_cta_pair_ragged(cuda, sizes, m, n, bits):
    """cta_group::2 tiles (M = 256 over two SMs, each CTA holding half of the
    token tile): problem sizes that leave every kind of partial last tile
    (1..255 rows, empty problems, a K tail), fast vs exact on the GPU."""
    ops = _ops()
    rng = np.random.default_rng(sum(sizes) + m + n + bits)
    E = len(sizes)
    rows = sum(sizes)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    probs = np.stack([np.arange(E, dtype=np.uint32), off[:-1], off[1:]], 1)
    x = rng.standard_normal((rows, m)).astype(np.float16)
    w = (0.25 * rng.standard_normal((E, m, n))).astype(np.float16)
    bias = (0.05 * rng.standard_normal((E, n))).astype(np.float16)
    if bits == 16:
        tiled, sc = ops.tile_weights(to_dev(w), E, m, n, 16), None
    else:
        packed, sc = ops.quantize(to_dev(w), bits)
        tiled = ops.tile_weights(packed, E, m, n, bits)
    xs, pr, bd = to_dev(x), to_dev(probs), to_dev(bias)
    a = ops.grouped_gemm(xs, pr, tiled, sc, bits, E, n, bd, True, ops.MODE_EXACT)
    b = ops.grouped_gemm(xs, pr, tiled, sc, bits, E, n, bd, True, ops.MODE_FAST)
    got, want = to_np(b), to_np(a)
    assert np.isfinite(got.astype(np.float32)).all()
    for e in range(E):  # every problem on its own: a missed tail tile cannot hide
        lo, hi = int(off[e]), int(off[e + 1])
        if hi > lo:
            assert norm_err(got[lo:hi], want[lo:hi]) <= TOL_FAST, (e, lo, hi)


@pytest.mark.parametrize("bits", [4, 8, 16])
@pytest.mark.parametrize("shape", [(1, 1, 1024, 4096), (8, 4, 1024, 512), (64, 32, 256, 1024),
                                   (40, 3, 4096, 256), (3, 5, 72, 136), (200, 8, 512, 2048)])
def test_gemm_gemv_decode_within_tolerance(cuda, oracle, bits, shape):
    """K5 decode kernel (mma.sync over the tcgen05 weight tiles, split-K with a
    fixed-order reduction) vs the oracle: any rows per expert, ragged m/n."""
    rows, E, m, n = shape
    if bits == 4 and n % 8:
        pytest.skip("int4 needs n % 8 == 0")
    rng = np.random.default_rng(rows * 7 + E + m + n + bits)
    ex, fin, x, w, bias = _gemm_case(rng, rows, E, m, n, bits, fin_frac=0.1)
    got, want = _run_gemm(oracle, ex, fin, x, w, bias, bits, bits != 8, _ops().MODE_GEMV)
    active = int((fin == 0).sum())
    if active:
        assert norm_err(got[:active], want[:active]) <= TOL_FAST


def test_gemm_gemv_deterministic(cuda, oracle):
    rng = np.random.default_rng(5)
    ex, fin, x, w, bias = _gemm_case(rng, 16, 2, 2048, 512, 4, fin_frac=0.0)
    a, _ = _run_gemm(oracle, ex, fin, x, w, bias, 4, False, _ops().MODE_GEMV)
    b, _ = _run_gemm(oracle, ex, fin, x, w, bias, 4, False, _ops().MODE_GEMV)
    assert np.array_equal(bits16(a), bits16(b))
