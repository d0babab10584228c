"""Expert-parallel host logic on CPU, world_size 2 and 4 over gloo.

The exchange protocol of csrc/ep.cu (moe_ep_forward) is replayed with gloo
point-to-point transfers -- one message per rank pair in the same issue
order as its NCCL transport, the staging -> expert-major segment copies of
its regroup kernel -- and the product's C++ segment arithmetic
(moe_ep_segments, called through the C-ABI -- pure host code, no GPU)
places every row.  The local compute (LN,
gate, plan, expert FFNs, combine) is the C oracle.  Every rank's output must
equal the single-process oracle layer on its tokens bit for bit (rows are
independent), for top-1/top-2, int4/int8/fp16 experts, ragged and empty
token counts and finished rows."""
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


def _exchange(dist, torch, sends, recvs, rank):
    """sends / recvs: [(peer, array)] in issue order (ep.cu run_xfer);
    self segments are local copies, the rest gloo isend / irecv (matched in
    order per peer, like NCCL point-to-point)."""
    mine = [a for p, a in sends if p == rank]
    into = [a for p, a in recvs if p == rank]
    for a, b in zip(mine, into):
        b[...] = a
    reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(a)), p) for p, a in sends if p != rank]
    bufs = [(torch.empty(a.shape, dtype=torch.int16), a) for p, a in recvs if p != rank]
    reqs += [dist.irecv(t, p) for (t, _), (p, _) in zip(bufs, [r for r in recvs if r[0] != rank])]
    for r in reqs:
        r.wait()
    for t, a in bufs:
        a[...] = t.numpy()


def _worker(rank, world, port, cfg, results):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle, random_layer
    from paper_2211_10017_b200.ep import owner_range, segments

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, f, E, k, bits = cfg["d"], cfg["f"], cfg["E"], cfg["k"], cfg["bits"]
    G = world
    lw = random_layer(d, f, E, seed=17)
    orc = Oracle()
    q = None if bits == 16 else (*orc.quantize(lw.w1, bits), *orc.quantize(lw.w2, bits))
    T = cfg["T"][rank]
    rng = np.random.default_rng(100 + rank)
    x = rng.standard_normal((max(T, 1), d)).astype(np.float16)[:T]
    fin = (rng.random(T) < 0.2).astype(np.uint8)
    e0, el = owner_range(E, G, rank)
    # 1. route (oracle): plan-sorted rows
    if T:
        xn = orc.layer_norm(x, lw.ln_g, lw.ln_b)
        ex, sc = orc.gate_topk(orc.gate_logits(xn, lw.gw, lw.gb), k)
        perm, inv, offs, act = orc.routing_plan(ex, fin, E)
        xp = xn[perm // k].view(np.int16)
    else:
        offs = np.zeros(E + 1, np.uint32)
        xp = np.zeros((0, d), np.int16)
    # 2. counts exchange
    send_cnt = np.diff(offs[:E + 1].astype(np.int64)).reshape(G, el)
    rc = torch.zeros(G * el, dtype=torch.int64)
    dist.all_to_all_single(rc, torch.from_numpy(send_cnt.reshape(-1).copy()))
    recv_cnt = rc.numpy().reshape(G, el)
    # 3. the product's segment arithmetic (C++)
    so, rd, probs, rows = segments(G, el, send_cnt, recv_cnt)
    so, rd = so.reshape(G, el), rd.reshape(G, el)
    # 4. dispatch, same messages as ep.cu: one per rank pair into the
    # (source, expert)-major staging buffer, then the regroup segment copies
    base = np.concatenate([[0], np.cumsum(recv_cnt.sum(1))]).astype(np.int64)
    segs = []  # (staging row, expert-major row, rows)
    for s in range(G):
        pos = base[s]
        for j in range(el):
            if recv_cnt[s, j]:
                segs.append((pos, rd[s, j], recv_cnt[s, j]))
                pos += recv_cnt[s, j]
    xr = np.zeros((rows, d), np.int16)
    sends = [(p, xp[so[p, 0]:so[p, 0] + send_cnt[p].sum()]) for p in range(G) if send_cnt[p].sum()]
    recvs = [(s, xr[base[s]:base[s + 1]]) for s in range(G) if base[s + 1] > base[s]]
    _exchange(dist, torch, sends, recvs, rank)
    xe = np.zeros((rows, d), np.int16)
    for a, b, c in segs:
        xe[b:b + c] = xr[a:a + c]
    # 5. local experts (oracle grouped GEMMs over the expert-major rows)
    sl = slice(e0, e0 + el)
    ye = np.zeros((rows, d), np.int16)
    if rows:
        xe16 = xe.view(np.float16)
        if bits == 16:
            h, _ = orc.grouped_gemm(xe16, probs, bits=16, w16=lw.w1[sl], E=el, n=f, bias=lw.b1[sl],
                                    relu=True)
            y, _ = orc.grouped_gemm(h, probs, bits=16, w16=lw.w2[sl], E=el, n=d, bias=lw.b2[sl],
                                    relu=False)
        else:
            per = lambda a, m, n: a[e0 * (m * n // (2 if bits == 4 else 1)):
                                    (e0 + el) * (m * n // (2 if bits == 4 else 1))]
            h, _ = orc.grouped_gemm(xe16, probs, bits=bits, packed=per(q[0], d, f),
                                    scales=q[1][sl], E=el, n=f, bias=lw.b1[sl], relu=True)
            y, _ = orc.grouped_gemm(h, probs, bits=bits, packed=per(q[2], f, d), scales=q[3][sl],
                                    E=el, n=d, bias=lw.b2[sl], relu=False)
        ye[...] = y.view(np.int16)
    # 6. inverse regroup, one message per rank pair back into the sorted y,
    # then the residual combine
    for a, b, c in segs:
        xr[a:a + c] = ye[b:b + c]
    ys = np.zeros((int(offs[E]) if T else 0, d), np.int16)
    sends = [(s, xr[base[s]:base[s + 1]]) for s in range(G) if base[s + 1] > base[s]]
    recvs = [(p, ys[so[p, 0]:so[p, 0] + send_cnt[p].sum()]) for p in range(G) if send_cnt[p].sum()]
    _exchange(dist, torch, sends, recvs, rank)
    if T:
        out = x.copy()
        y16 = ys.view(np.float16)
        for r in range(T):
            if fin[r]:
                continue
            acc = x[r]
            for s in range(k):
                prod = (y16[inv[r * k + s]].astype(np.float64) *
                        np.float64(sc.view(np.float16)[r, s])).astype(np.float16)
                acc = (acc.astype(np.float64) + prod.astype(np.float64)).astype(np.float16)
            out[r] = acc
        want = orc.moe_forward(lw, x, fin, k=k, bits=bits, q=q)
        results[rank] = bool(np.array_equal(out.view(np.uint16), want.view(np.uint16)))
    else:
        results[rank] = True  # no tokens: the rank still served its experts
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [
    (2, dict(d=32, f=64, E=4, k=1, bits=4, T=[9, 14])),
    (2, dict(d=32, f=64, E=8, k=2, bits=4, T=[17, 3])),
    (2, dict(d=24, f=40, E=2, k=1, bits=16, T=[5, 6])),
    (4, dict(d=32, f=48, E=8, k=2, bits=8, T=[4, 11, 1, 7])),
    (4, dict(d=32, f=48, E=8, k=2, bits=4, T=[0, 23, 5, 9])),
])
def test_ep_protocol_matches_single_process_oracle(world, cfg):
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


def test_ep_segments_host_logic():
    """moe_ep_segments on a hand-worked case: 3 ranks, 2 experts per rank."""
    from paper_2211_10017_b200.ep import segments
    sc = np.array([[2, 0], [3, 4], [0, 0]])   # to rank 0: e0 2 rows; to rank 1: e0 3, e1 4
    rc = np.array([[1, 2], [3, 0], [0, 4]])   # from 3 sources, 2 local experts
    so, rd, pr, rows = segments(3, 2, sc, rc)
    assert so.tolist() == [0, 2, 2, 5, 9, 9]
    # expert-major: e0 <- src0(1) src1(3) src2(0); e1 <- src0(2) src1(0) src2(4)
    assert rd.reshape(3, 2).tolist() == [[0, 4], [1, 6], [4, 6]]
    assert pr.tolist() == [[0, 0, 4], [1, 4, 10]] and rows == 10
    with pytest.raises(ValueError):
        segments(0, 2, sc, rc)
