"""Expert-parallel orchestration (paper_2211_10017_b200/ep.py) on CPU with
gloo, world_size 2 and 4: every rank's output must equal the single-process
oracle layer on that rank's tokens bit for bit (rows are independent), for
top-1/top-2, int4/fp16 experts, ragged token counts and finished rows.  The
local compute is the oracle (tests/ep_oracle_rank.py); the transport, counts,
splits and regroup logic are the product code."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, results):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    from ep_oracle_rank import OracleRank
    from oracle.oracle import Oracle, random_layer
    from paper_2211_10017_b200.ep import DistComm, ep_forward, owner_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, f, E, k, bits = cfg["d"], cfg["f"], cfg["E"], cfg["k"], cfg["bits"]
    lw = random_layer(d, f, E, seed=17)
    orc = Oracle()
    q = None if bits == 16 else (*orc.quantize(lw.w1, bits), *orc.quantize(lw.w2, bits))
    T = cfg["T"][rank]
    rng = np.random.default_rng(100 + rank)
    x = rng.standard_normal((T, d)).astype(np.float16)
    fin = (rng.random(T) < 0.2).astype(np.uint8)
    e0, el = owner_range(E, world, rank)
    R = OracleRank(lw, e0, el, bits=bits, q=q)
    out = ep_forward([R], DistComm(), [torch.from_numpy(x.copy())],
                     [torch.from_numpy(fin)], k=k, mode=0)[0].numpy().view(np.uint16)
    want = orc.moe_forward(lw, x, fin, k=k, bits=bits, q=q).view(np.uint16)
    results[rank] = bool(np.array_equal(out, want))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [
    (2, dict(d=32, f=64, E=4, k=1, bits=4, T=[9, 14])),
    (2, dict(d=32, f=64, E=8, k=2, bits=4, T=[17, 3])),
    (2, dict(d=24, f=40, E=2, k=1, bits=16, T=[5, 0 + 6])),
    (4, dict(d=32, f=48, E=8, k=2, bits=8, T=[4, 11, 1, 7])),
])
def test_ep_matches_single_process_oracle(world, cfg):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert dict(results) == {r: True for r in range(world)}


def test_regroup_and_counts():
    from paper_2211_10017_b200.ep import inverse, regroup, send_counts
    offs = np.array([0, 2, 2, 5, 9, 9, 12])  # E = 5, finished tail from 9
    sc = send_counts(offs[:6].tolist() + [12], 4, 2)  # E=4 -> (2, 2)
    assert sc.tolist() == [[2, 0], [3, 4]]
    rc = np.array([[1, 2], [3, 0], [0, 4]])  # from 3 sources, 2 local experts
    perm, probs = regroup(rc)
    # received: src0 e0(0) e1(1,2) | src1 e0(3,4,5) | src2 e1(6,7,8,9)
    assert perm.tolist() == [0, 3, 4, 5, 1, 2, 6, 7, 8, 9]
    assert probs.tolist() == [[0, 0, 4], [1, 4, 10]]
    assert inverse(perm)[perm].tolist() == list(range(10))
