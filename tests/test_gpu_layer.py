"""GPU parity for the whole MoE layer (moe_ffn_forward replacement).

EXACT mode must equal the oracle's batched forward AND the per-token oracle
bit for bit (test_model.cpp:303-330 contract), at fp16/int8/int4 and top-1/
top-2, with finished rows.  FAST mode: routing (expert indices, scales,
perm, inv, offsets) bit-exact, outputs within TOL_FAST (normalized max error
of the MoE contribution out - x)."""
import numpy as np
import pytest

from conftest import bits16, layer_err, norm_err, to_dev, to_np

pytestmark = pytest.mark.gpu

TOL_FAST = 1e-2


def _layer(lw, bits, q=None):
    from paper_2211_10017_b200.ops import MoELayer
    return MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits, q=q)


def _case(d, f, E, T, seed, fin_frac=0.25):
    from oracle.oracle import random_layer
    lw = random_layer(d, f, E, seed=seed)
    rng = np.random.default_rng(seed + 1)
    x = rng.standard_normal((T, d)).astype(np.float16)
    fin = (rng.random(T) < fin_frac).astype(np.uint8)
    return lw, x, fin


@pytest.mark.parametrize("bits", [16, 8, 4])
@pytest.mark.parametrize("k", [1, 2])
def test_layer_exact_bit_exact(cuda, oracle, bits, k):
    lw, x, fin = _case(64, 96, 8, 33, seed=404 + bits + k)
    L = _layer(lw, bits)
    q = tuple(to_np(t) for t in L.quant) if bits != 16 else None
    want, diag = oracle.moe_forward(lw, x, fin, k=k, bits=bits, q=q, diagnostics=True)
    got = to_np(L.forward(to_dev(x), to_dev(fin), k=k, mode=0))
    assert np.array_equal(bits16(got), bits16(want))
    per_tok = oracle.moe_per_token(lw, x, fin, k=k, bits=bits, q=q)
    assert np.array_equal(bits16(got), bits16(per_tok))
    r = L.routing(33, k)
    for key in ("expert", "perm", "inv", "offsets"):
        assert np.array_equal(r[key].reshape(-1), diag[key].reshape(-1)), key
    assert np.array_equal(r["scale"].reshape(-1), diag["scale"].reshape(-1))
    assert r["active"] == diag["active"]
    # finished rows pass through exactly
    assert np.array_equal(bits16(got)[fin == 1], bits16(x)[fin == 1])


def test_layer_quantized_on_gpu_matches_oracle_quantizer(cuda, oracle):
    lw, x, fin = _case(128, 256, 8, 20, seed=7)
    L = _layer(lw, 4)
    q1, s1 = oracle.quantize(lw.w1, 4)
    assert np.array_equal(to_np(L.quant[0]), q1)
    assert np.array_equal(bits16(to_np(L.quant[1])), bits16(s1))


@pytest.mark.parametrize("bits", [4, 8, 16])
@pytest.mark.parametrize("k", [1, 2])
def test_layer_fast_routing_exact_output_tolerance(cuda, oracle, bits, k):
    lw, x, fin = _case(256, 512, 8, 200, seed=11 + bits + k, fin_frac=0.1)
    L = _layer(lw, bits)
    q = tuple(to_np(t) for t in L.quant) if bits != 16 else None
    want, diag = oracle.moe_forward(lw, x, fin, k=k, bits=bits, q=q, diagnostics=True)
    got = to_np(L.forward(to_dev(x), to_dev(fin), k=k, mode=1))
    r = L.routing(200, k)
    for key in ("expert", "perm", "inv", "offsets", "scale"):
        assert np.array_equal(r[key].reshape(-1), diag[key].reshape(-1)), key
    xf = x.astype(np.float64)
    err = norm_err(got.astype(np.float64) - xf, want.astype(np.float64) - xf)
    assert err <= TOL_FAST, err
    assert np.array_equal(bits16(got)[fin == 1], bits16(x)[fin == 1])


def test_layer_host_path_equals_device_path(cuda):
    lw, x, fin = _case(128, 256, 16, 77, seed=21)
    L = _layer(lw, 4)
    for mode in (0, 1):
        a = to_np(L.forward(to_dev(x), to_dev(fin), k=2, mode=mode))
        b = L.forward_host(x, fin, k=2, mode=mode)
        assert np.array_equal(bits16(a), bits16(b))


def test_layer_rejects_non_finite(cuda):
    lw, x, fin = _case(64, 64, 4, 8, seed=3)
    L = _layer(lw, 4)
    x[5, 3] = np.inf
    with pytest.raises(ValueError, match="non-finite logit at row 5"):
        L.forward_host(x, fin, k=1, mode=1)


def test_layer_traffic_matches_reference_accounting(cuda, oracle):
    lw, x, fin = _case(64, 96, 8, 40, seed=5)
    L = _layer(lw, 4)
    L.forward(to_dev(x), to_dev(fin), k=1, mode=0)
    t = L.traffic()
    _, diag = oracle.moe_forward(lw, x, fin, k=1, bits=4,
                                 q=tuple(to_np(a) for a in L.quant), diagnostics=True)
    off = diag["offsets"]
    d, f, E, T = 64, 96, 8, 40
    active = [e for e in range(E) if off[e + 1] > off[e]]
    rows = [int(off[e + 1] - off[e]) for e in active]
    ew = sum((d * f // 2 + f * 2) + (f * d // 2 + d * 2) for _ in active)
    ea = sum((r * d + f) * 2 + (r * f + d) * 2 for r in rows)
    eo = sum(r * f * 2 + r * d * 2 for r in rows)
    assert t["expert"] == (ew, ea, eo)


@pytest.mark.parametrize("T,k", [(4096, 2), (1, 1), (64, 1)])
def test_c2_c3_shapes_fast_vs_exact_and_per_token_rows(cuda, oracle, T, k):
    """BASELINE config 2 (E=8, d=512, f=2048, int4, top-2, T=4096) and
    decode-shaped rows at the same width: fast within tolerance of exact
    (exact == reference semantics); 16 sampled rows vs the per-token oracle."""
    lw, x, fin = _case(512, 2048, 8, T, seed=1234, fin_frac=0.0)
    L = _layer(lw, 4)
    q = tuple(to_np(a) for a in L.quant)
    xd = to_dev(x)
    ex = to_np(L.forward(xd, None, k=k, mode=0))
    fa = to_np(L.forward(xd, None, k=k, mode=1))
    xf = x.astype(np.float64)
    assert norm_err(fa.astype(np.float64) - xf, ex.astype(np.float64) - xf) <= TOL_FAST
    rows = np.random.default_rng(0).choice(T, size=min(T, 16), replace=False)
    want = oracle.moe_per_token(lw, x[rows], None, k=k, bits=4, q=q)
    assert np.array_equal(bits16(ex[rows]), bits16(want))


@pytest.mark.parametrize("T", [1, 2, 8, 64, 256])
def test_layer_decode_shapes(cuda, oracle, T):
    """Decode-shaped layers (C3 family, reduced d/f): fused gate + K5 GEMV
    (T*k <= 256) -- routing bit-exact, outputs within tolerance, and the same
    layer object reused across T (workspace growth)."""
    lw, x, fin = _case(256, 1024, 32, T, seed=300 + T, fin_frac=0.2 if T > 1 else 0.0)
    L = _layer(lw, 4)
    q = tuple(to_np(t) for t in L.quant)
    for k in (1, 2):
        want, diag = oracle.moe_forward(lw, x, fin, k=k, bits=4, q=q, diagnostics=True)
        got = to_np(L.forward(to_dev(x), to_dev(fin), k=k, mode=1))
        r = L.routing(T, k)
        for key in ("expert", "perm", "inv", "offsets", "scale"):
            assert np.array_equal(r[key].reshape(-1), diag[key].reshape(-1)), key
        if (want != x).any():
            err = layer_err(got, want, x)
            assert err <= TOL_FAST, err
        assert np.array_equal(bits16(got)[fin == 1], bits16(x)[fin == 1])


@pytest.mark.parametrize("E,d,T,k", [(8, 512, 4096, 2), (64, 1024, 600, 1), (128, 256, 300, 2),
                                     (3, 40, 50, 3), (130, 64, 20, 1), (300, 32, 40, 2),
                                     (32, 1024, 4096, 2), (64, 1024, 16384, 1), (8, 512, 1, 1),
                                     (256, 2048, 700, 8), (128, 512, 4100, 2), (64, 1024, 5000, 3),
                                     (64, 256, 9000, 1), (128, 2048, 2100, 1)])
def test_layer_fused_gate_routing_exact(cuda, oracle, E, d, T, k):
    """Fused LN+logits+top-k+histogram kernel (and the unfused fallback for
    E > 256): routing identical to the oracle at BASELINE-like shapes --
    f32-widened and fp16 LN chain forms, one and two waves of row blocks,
    chunked and resident gate weights, E <= 16 and warp-per-row selection."""
    from oracle.oracle import random_layer
    lw = random_layer(d, 64, E, seed=E + d + T)
    rng = np.random.default_rng(T)
    x = rng.standard_normal((T, d)).astype(np.float16)
    fin = (rng.random(T) < 0.1).astype(np.uint8)
    L = _layer(lw, 16)
    L.forward(to_dev(x), to_dev(fin), k=k, mode=1)
    r = L.routing(T, k)
    xn = oracle.layer_norm(x, lw.ln_g, lw.ln_b)
    lg = oracle.gate_logits(xn, lw.gw, lw.gb)
    ex, sc = oracle.gate_topk(lg, k)
    perm, inv, offs, act = oracle.routing_plan(ex, fin, E)
    assert np.array_equal(r["expert"], ex)
    assert np.array_equal(r["scale"], sc)
    assert np.array_equal(r["perm"], perm) and np.array_equal(r["inv"], inv)
    assert np.array_equal(r["offsets"], offs) and r["active"] == act


@pytest.mark.parametrize("bits,f", [(16, 64), (4, 64), (4, 4096)])
def test_layer_fast_repeat_bitwise_deterministic(cuda, bits, f):
    """Repeated FAST forwards of one layer give identical bits (catches
    pipeline races: with odd TMA stage counts fp16-weight layers at this
    shape faulted or drifted within ~20 repeats)."""
    import torch
    from oracle.oracle import random_layer
    d, E, T = 1024, 64, 16384
    lw = random_layer(d, f, E, seed=5)
    L = _layer(lw, bits)
    rng = np.random.default_rng(9)
    x = to_dev(rng.standard_normal((T, d)).astype(np.float16))
    fin = to_dev((rng.random(T) < 0.1).astype(np.uint8))
    ref = to_np(L.forward(x, fin, k=1, mode=1))
    for _ in range(25):
        got = to_np(L.forward(x, fin, k=1, mode=1))
        assert np.array_equal(bits16(got), bits16(ref))



def _pinned_like(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.int16 if a.dtype == np.float16 else torch.uint8,
                    pin_memory=True)
    v = t.numpy().view(a.dtype)
    v[...] = a
    return t, v


@pytest.mark.parametrize("k", [1, 2])
def test_layer_host_pinned_chunked_pipeline(cuda, oracle, k):
    """Pinned host buffers: moe_layer_forward_host pipelines copy-in / compute
    / copy-out over token chunks on three streams (C2 shape, 4 chunks).
    EXACT: bit-identical to the device path and the per-token oracle; FAST:
    identical to the device path (rows are independent), finished rows pass
    through; a non-finite token in a late chunk is reported by its global row."""
    lw, x, fin = _case(512, 2048, 8, 4096, seed=77 + k, fin_frac=0.1)
    L = _layer(lw, 4)
    q = tuple(to_np(t) for t in L.quant)
    xt, xh = _pinned_like(x)
    ft, fh = _pinned_like(fin)
    ot, oh = _pinned_like(np.zeros_like(x))
    for mode in (0, 1):
        L.forward_host(xh, fh, k=k, mode=mode, out_host=oh)
        dev = to_np(L.forward(to_dev(x), to_dev(fin), k=k, mode=mode))
        if mode == 0:
            assert np.array_equal(bits16(oh), bits16(dev))
            rows = np.arange(0, 4096, 97)
            want = oracle.moe_per_token(lw, x[rows], fin[rows], k=k, bits=4, q=q)
            assert np.array_equal(bits16(oh[rows]), bits16(want))
        else:
            assert layer_err(oh, dev, x) <= TOL_FAST
        assert np.array_equal(bits16(oh)[fin == 1], bits16(x)[fin == 1])
    xh[3500, 7] = np.inf
    with pytest.raises(ValueError, match="non-finite logit at row 3500"):
        L.forward_host(xh, fh, k=k, mode=1, out_host=oh)


@pytest.mark.parametrize("cf", [1.0, 1.25])
def test_layer_load_report(cuda, cf):
    """moe_layer_load_report (expert-capacity bookkeeping, north_star item 1):
    per-expert live loads from the last plan, capacity ceil(cf * live / E),
    max load, experts / rows over capacity -- against numpy on the routing."""
    import math
    lw, x, fin = _case(128, 256, 16, 700, seed=31, fin_frac=0.2)
    L = _layer(lw, 4)
    L.forward(to_dev(x), to_dev(fin), k=2, mode=1)
    rep = L.load_report(cf)
    off = L.routing(700, 2)["offsets"].astype(np.int64)
    load = np.diff(off[:17])
    live = int(off[16] - off[0])
    cap = math.ceil(cf * live / 16)
    assert rep["load"].tolist() == load.tolist()
    assert rep["live_slots"] == live == 2 * int((fin == 0).sum())
    assert rep["capacity"] == cap and rep["max_load"] == load.max()
    assert rep["experts_over"] == int((load > cap).sum())
    assert rep["overflow_rows"] == int(np.maximum(load - cap, 0).sum())
    assert rep["active_experts"] == int((load > 0).sum())


@pytest.mark.parametrize("bits", [16, 8, 4])
@pytest.mark.parametrize("T,k", [(1, 1), (37, 2), (200, 1)])
def test_layer_decode_pair_repeat(cuda, oracle, bits, T, k):
    """Decode-shaped layers at 16/8/4 bits: within tolerance of the oracle
    on the first forward (fresh workspace) and bitwise identical over
    repeated forwards (split-K tickets self-reset; no stale state)."""
    lw, x, fin = _case(256, 1024, 32, T, seed=900 + T + bits, fin_frac=0.1 if T > 1 else 0.0)
    L = _layer(lw, bits)
    q = tuple(to_np(t) for t in L.quant) if bits != 16 else None
    want = oracle.moe_forward(lw, x, fin, k=k, bits=bits, q=q)
    xd, fd = to_dev(x), to_dev(fin)
    first = to_np(L.forward(xd, fd, k=k, mode=1))
    if (want != x).any():
        assert layer_err(first, want, x) <= TOL_FAST
    for _ in range(6):
        assert np.array_equal(bits16(to_np(L.forward(xd, fd, k=k, mode=1))), bits16(first))
