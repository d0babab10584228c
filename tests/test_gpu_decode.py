"""Decode with batch pruning (moe_decode_run, csrc/decode.cu; reference
proj/src/decode.cpp:104-345): per step, a stack of MoE blocks over the
batch x beam rows with the finished rows as routing mask when pruning.

* EXACT: every step's output equals the oracle chain of moe_ffn_forward
  calls with the same mask (bit for bit);
* pruning is output-transparent: live rows are identical with and without
  pruning, and finished rows pass through every block unchanged;
* FAST (decode GEMV / tcgen05 paths): within tolerance of the oracle."""
import numpy as np
import pytest

from conftest import bits16, layer_err, to_dev, to_np

pytestmark = pytest.mark.gpu


def _stack(n, d, f, E, seed):
    from oracle.oracle import random_layer
    from paper_2211_10017_b200.ops import MoELayer
    lws = [random_layer(d, f, E, seed=seed + i) for i in range(n)]
    Ls = [MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4) for lw in lws]
    qs = [tuple(to_np(t) for t in L.quant) for L in Ls]
    return lws, Ls, qs


@pytest.mark.parametrize("k", [1, 2])
def test_decode_pruning_exact_and_transparent(cuda, oracle, k):
    from paper_2211_10017_b200.decode import decode_run, finished_schedule
    d, f, E, batch, beam, steps, nl = 128, 256, 8, 6, 4, 5, 3
    rows = batch * beam
    lws, Ls, qs = _stack(nl, d, f, E, seed=90 + k)
    rng = np.random.default_rng(k)
    xs = rng.standard_normal((steps, rows, d)).astype(np.float16)
    fin = finished_schedule(batch, beam, steps, [1, 5, 3, 2, 4, 5])
    on = to_np(decode_run(Ls, to_dev(xs), to_dev(fin), k=k, mode=0, prune=True))
    off = to_np(decode_run(Ls, to_dev(xs), to_dev(fin), k=k, mode=0, prune=False))
    for s in range(steps):
        a, b = xs[s], xs[s]
        for lw, q in zip(lws, qs):
            a = oracle.moe_forward(lw, a, fin[s], k=k, bits=4, q=q)
            b = oracle.moe_forward(lw, b, None, k=k, bits=4, q=q)
        assert np.array_equal(bits16(on[s]), bits16(a)), s
        assert np.array_equal(bits16(off[s]), bits16(b)), s
        live = fin[s] == 0
        assert np.array_equal(bits16(on[s])[live], bits16(off[s])[live]), s
        assert np.array_equal(bits16(on[s])[~live], bits16(xs[s])[~live]), s


def test_decode_pruning_fast_decode_shapes(cuda, oracle):
    """C3/C4-like decode: E=32, d=1024, f=4096 blocks, 64 x 4 rows (GEMV path
    as rows finish), FAST within tolerance of the oracle per step."""
    from paper_2211_10017_b200.decode import decode_run, finished_schedule
    d, f, E, batch, beam, steps, nl = 1024, 4096, 32, 16, 4, 4, 2
    rows = batch * beam
    lws, Ls, qs = _stack(nl, d, f, E, seed=7)
    rng = np.random.default_rng(3)
    xs = rng.standard_normal((steps, rows, d)).astype(np.float16)
    lens = rng.integers(1, steps + 1, batch)
    fin = finished_schedule(batch, beam, steps, lens)
    got = to_np(decode_run(Ls, to_dev(xs), to_dev(fin), k=1, mode=1, prune=True))
    for s in range(steps):
        a = xs[s]
        for lw, q in zip(lws, qs):
            a = oracle.moe_forward(lw, a, fin[s], k=1, bits=4, q=q)
        if (a != xs[s]).any():
            assert layer_err(got[s], a, xs[s]) <= 1e-2, s
        assert np.array_equal(bits16(got[s])[fin[s] == 1], bits16(xs[s])[fin[s] == 1])
