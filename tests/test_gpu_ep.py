"""Expert parallelism on the device: G simulated ranks on one B200 through
the loopback transport (same ep_forward code as the NCCL path), and the real
NCCL transport at world size 1.  EXACT numerics: every rank's output is
bit-identical to the single-GPU layer on its tokens (and to the oracle);
FAST: within tolerance."""
import os
import socket

import numpy as np
import pytest

from conftest import bits16, layer_err, to_dev, to_np

pytestmark = pytest.mark.gpu


def _ranks(lw, G, bits=4):
    from paper_2211_10017_b200.ep import CudaRank, owner_range
    from paper_2211_10017_b200.ops import MoELayer
    out = []
    for g in range(G):
        e0, el = owner_range(lw.E, G, g)
        sl = slice(e0, e0 + el)
        out.append(CudaRank(MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1[sl], lw.b1[sl],
                                     lw.w2[sl], lw.b2[sl], bits=bits, expert_range=(e0, el))))
    return out


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("k", [1, 2])
def test_ep_loopback_bit_identical_to_single_gpu(cuda, oracle, G, k):
    from oracle.oracle import random_layer
    from paper_2211_10017_b200.ep import LoopbackComm, ep_forward
    from paper_2211_10017_b200.ops import MoELayer
    lw = random_layer(128, 256, 8, seed=40 + G)
    full = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4)
    q = tuple(to_np(t) for t in full.quant)
    rng = np.random.default_rng(G * 10 + k)
    Ts = [int(rng.integers(1, 300)) for _ in range(G)]
    xs = [rng.standard_normal((T, 128)).astype(np.float16) for T in Ts]
    fins = [(rng.random(T) < 0.15).astype(np.uint8) for T in Ts]
    ranks = _ranks(lw, G)
    for mode in (0, 1):
        outs = ep_forward(ranks, LoopbackComm(G), [to_dev(x) for x in xs],
                          [to_dev(f) for f in fins], k=k, mode=mode)
        for g in range(G):
            got = to_np(outs[g])
            if mode == 0:
                want = to_np(full.forward(to_dev(xs[g]), to_dev(fins[g]), k=k, mode=0))
                assert np.array_equal(bits16(got), bits16(want)), g
                orc = oracle.moe_forward(lw, xs[g], fins[g], k=k, bits=4, q=q)
                assert np.array_equal(bits16(got), bits16(orc)), g
            else:
                want = oracle.moe_forward(lw, xs[g], fins[g], k=k, bits=4, q=q)
                assert layer_err(got, want, xs[g]) <= 1e-2


def test_ep_nccl_world1(cuda, oracle):
    import torch.distributed as dist
    from oracle.oracle import random_layer
    from paper_2211_10017_b200.ep import EPMoELayer
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        lw = random_layer(64, 128, 4, seed=3)
        L = EPMoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4)
        x = np.random.default_rng(0).standard_normal((50, 64)).astype(np.float16)
        got = to_np(L.forward(to_dev(x), None, k=2, mode=0))
        q = tuple(to_np(t) for t in (L.rank.L.quant))
        want = oracle.moe_forward(lw, x, None, k=2, bits=4, q=q)
        assert np.array_equal(bits16(got), bits16(want))
    finally:
        dist.destroy_process_group()
