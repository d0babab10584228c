"""Expert parallelism on the device through the C-ABI (moe_ep_forward,
csrc/ep.cu): G ranks held in one process on one B200 via the loopback
transport (the same C++ orchestration as the NCCL path, segments moved by
device-to-device copies), and the real NCCL transport at world size 1 (one
GPU per gpurun box).  EXACT numerics: every rank's output is bit-identical
to the single-GPU layer on its tokens and to the oracle; FAST: routing is
shared with the single-GPU layer, outputs within tolerance.  A world-2 NCCL
run (scripts/ep_nccl_check.py under torchrun) is skipped below 2 GPUs."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, bits16, layer_err, to_dev, to_np

pytestmark = pytest.mark.gpu


def _rank_layers(lw, G, q, bits=4):
    from paper_2211_10017_b200.ep import owner_range
    from paper_2211_10017_b200.ops import MoELayer
    out = []
    E = lw.E
    for g in range(G):
        e0, el = owner_range(E, G, g)
        sl = slice(e0, e0 + el)
        qs = None
        if q is not None:
            nb1, nb2 = q[0].size // E, q[2].size // E
            qs = (q[0][e0 * nb1:(e0 + el) * nb1], q[1][sl], q[2][e0 * nb2:(e0 + el) * nb2], q[3][sl])
        out.append(MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1[sl], lw.b1[sl], lw.w2[sl],
                            lw.b2[sl], bits=bits, expert_range=(e0, el), q=qs))
    return out


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("k", [1, 2])
def test_ep_loopback_bit_identical_to_single_gpu(cuda, oracle, G, k):
    from oracle.oracle import random_layer
    from paper_2211_10017_b200.ep import LoopbackEP
    from paper_2211_10017_b200.ops import MoELayer
    lw = random_layer(128, 256, 8, seed=40 + G)
    full = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4)
    q = tuple(to_np(t) for t in full.quant)
    rng = np.random.default_rng(G * 10 + k)
    Ts = [int(rng.integers(1, 300)) for _ in range(G)]
    xs = [rng.standard_normal((T, 128)).astype(np.float16) for T in Ts]
    fins = [(rng.random(T) < 0.15).astype(np.uint8) for T in Ts]
    ep = LoopbackEP(_rank_layers(lw, G, q))
    for mode in (0, 1):
        outs = ep.forward([to_dev(x) for x in xs], [to_dev(f) for f in fins], k=k, mode=mode)
        for g in range(G):
            got = to_np(outs[g])
            want = oracle.moe_forward(lw, xs[g], fins[g], k=k, bits=4, q=q)
            if mode == 0:
                single = to_np(full.forward(to_dev(xs[g]), to_dev(fins[g]), k=k, mode=0))
                assert np.array_equal(bits16(got), bits16(single)), g
                assert np.array_equal(bits16(got), bits16(want)), g
            else:
                assert layer_err(got, want, xs[g]) <= 1e-2
            assert np.array_equal(bits16(got)[fins[g] == 1], bits16(xs[g])[fins[g] == 1])
    # counts: what rank s sent to rank p is what p received from s
    sent = [ep.counts(g)[0] for g in range(G)]
    recv = [ep.counts(g)[1] for g in range(G)]
    for s in range(G):
        for p in range(G):
            assert np.array_equal(sent[s][p], recv[p][s])


def test_ep_loopback_c5_shape_fast(cuda, oracle):
    """C5's layer shape (E=128, d=2048, f=8192, int4, top-2) sharded 8 ways in
    loopback, 512 tokens per rank: routing-derived counts consistent, FAST
    outputs of sampled rows within tolerance of the per-token oracle."""
    import torch
    from paper_2211_10017_b200.ep import LoopbackEP, owner_range
    from paper_2211_10017_b200.ops import MoELayer
    from test_gpu_parity_configs import gpu_layer
    G, T, k = 8, 512, 2
    lw, full, q = gpu_layer(2048, 8192, 128, seed=55)
    layers = []
    E = 128
    for g in range(G):
        e0, el = owner_range(E, G, g)
        nb1, nb2 = q[0].size // E, q[2].size // E
        qs = (q[0][e0 * nb1:(e0 + el) * nb1], q[1][e0:e0 + el], q[2][e0 * nb2:(e0 + el) * nb2],
              q[3][e0:e0 + el])
        layers.append(MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, None, lw.b1[e0:e0 + el], None,
                               lw.b2[e0:e0 + el], bits=4, expert_range=(e0, el), q=qs))
    del full
    torch.cuda.empty_cache()
    rng = np.random.default_rng(7)
    xs = [rng.standard_normal((T, 2048)).astype(np.float16) for _ in range(G)]
    ep = LoopbackEP(layers)
    outs = ep.forward([to_dev(x) for x in xs], None, k=k, mode=1)
    total = sum(int(ep.counts(g)[2]) for g in range(G))
    assert total == G * T * k
    for g in (0, 5):
        rows = np.sort(rng.choice(T, 8, replace=False))
        want = oracle.moe_per_token(lw, xs[g][rows], None, k=k, bits=4, q=q)
        assert layer_err(to_np(outs[g])[rows], want, xs[g][rows]) <= 1e-2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_ep_nccl_world1(cuda, oracle):
    """The NCCL transport itself (ncclSend/ncclRecv to self) at world size 1."""
    import torch.distributed as dist
    from oracle.oracle import random_layer
    from paper_2211_10017_b200.ep import EPMoELayer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        lw = random_layer(64, 128, 4, seed=3)
        L = EPMoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4)
        x = np.random.default_rng(0).standard_normal((50, 64)).astype(np.float16)
        fin = (np.arange(50) % 7 == 0).astype(np.uint8)
        q = tuple(to_np(t) for t in L.layer.quant)
        want = oracle.moe_forward(lw, x, fin, k=2, bits=4, q=q)
        for _ in range(3):  # repeated forwards reuse the exchange buffers
            got = to_np(L.forward(to_dev(x), to_dev(fin), k=2, mode=0))
            assert np.array_equal(bits16(got), bits16(want))
    finally:
        dist.destroy_process_group()


def test_ep_nccl_world2(cuda):
    """Two processes, two GPUs, NCCL: each rank bit-identical to the
    single-GPU EXACT layer on its tokens (scripts/ep_nccl_check.py)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun grants one)")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1",
                        f"--master-port={_free_port()}",
                        os.path.join(ROOT, "scripts", "ep_nccl_check.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "ep_nccl_check ok" in r.stdout
