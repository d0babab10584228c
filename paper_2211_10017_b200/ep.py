"""Expert parallelism for the MoE layer.

G ranks (one process per GPU); rank g owns experts [g*E/G, (g+1)*E/G) and a
contiguous range of tokens.  One forward:

  1. route     -- local LN -> gate -> top-k -> plan -> gather (moe_layer_route);
                  the plan is sorted by expert, hence by owner rank
  2. counts    -- per (destination rank, local expert) row counts from the
                  plan offsets; all-to-all of G x E/G counts
  3. dispatch  -- all-to-all-v of the expert-sorted rows (NCCL over NVLink)
  4. regroup   -- received rows are (source, expert)-major; one gather puts
                  them expert-major for the grouped GEMMs
  5. experts   -- FFN1 + FFN2 of the local experts (moe_layer_experts)
  6. combine   -- inverse gather, reverse all-to-all-v, then the local
                  residual + gate-scaled un-permute (moe_layer_combine)

Every compute step is a libmoe_cuda.so kernel; torch.distributed (NCCL) is
the transport.  Rows are independent in every kernel, so in EXACT numerics
an EP forward is bit-identical to the single-GPU layer on the same tokens
(tests/test_ep_*.py).  The orchestration is written over a list of rank
states and a `Comm`, so the same code runs (a) distributed, one state per
process, and (b) as an in-process loopback of G ranks on one device (tests;
and the gloo CPU tests drive it with the oracle as the local compute).
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------- host bookkeeping
def owner_range(E: int, G: int, g: int):
    """(first expert, count) owned by rank g (E % G == 0)."""
    if E % G != 0:
        raise ValueError("ep: n_experts must be divisible by the world size")
    el = E // G
    return g * el, el


def send_counts(offsets, E: int, G: int) -> np.ndarray:
    """(G, E/G) rows this rank sends to each (owner rank, local expert);
    offsets = the plan's expert_offsets (E+1), finished rows excluded."""
    off = np.asarray(offsets, np.int64)
    return np.diff(off[: E + 1]).reshape(G, E // G)


def regroup(recv_counts: np.ndarray):
    """Received rows arrive (source rank, local expert)-major.  Returns
    perm (gather: expert-major position -> received position) and the
    grouped-GEMM problems (local expert, row_begin, row_end)."""
    rc = np.asarray(recv_counts, np.int64)
    G, el = rc.shape
    base = np.concatenate([[0], np.cumsum(rc.reshape(-1))])[:-1].reshape(G, el)
    perm = np.empty(int(rc.sum()), np.int64)
    problems = np.zeros((el, 3), np.int64)
    pos = 0
    for e in range(el):
        start = pos
        for src in range(G):
            c = int(rc[src, e])
            perm[pos:pos + c] = np.arange(base[src, e], base[src, e] + c)
            pos += c
        problems[e] = (e, start, pos)
    return perm, problems


def inverse(perm: np.ndarray) -> np.ndarray:
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm), dtype=perm.dtype)
    return inv


# ------------------------------------------------------------------ transports
class DistComm:
    """torch.distributed all-to-all-v (NCCL on GPUs, gloo on CPU); one local
    rank state per process."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)

    def all_to_all(self, sends, send_splits, recv_splits, outs=None):
        """sends: [tensor (sum(send_splits), ...)] for the one local rank;
        outs (optional): [preallocated receive tensor] (e.g. a layer buffer)."""
        import torch
        (x,), (ss,), (rs,) = sends, send_splits, recv_splits
        out = outs[0] if outs is not None else torch.empty(
            (int(sum(rs)),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        self.dist.all_to_all_single(out, x.contiguous(), [int(v) for v in rs],
                                    [int(v) for v in ss], group=self.group)
        return [out]


class LoopbackComm:
    """All G ranks in this process (one device): the all-to-all is a
    reshuffle of row segments between the rank states."""

    def __init__(self, world):
        self.world = world

    def all_to_all(self, sends, send_splits, recv_splits, outs=None):
        import torch
        G = self.world
        seg = []
        for g in range(G):
            cuts = np.concatenate([[0], np.cumsum(send_splits[g])]).astype(np.int64)
            seg.append([sends[g][int(cuts[j]):int(cuts[j + 1])] for j in range(G)])
        res = [torch.cat([seg[src][dst] for src in range(G)], 0) for dst in range(G)]
        if outs is not None:
            for o, r in zip(outs, res):
                if o is not None and r.shape[0]:
                    o.copy_(r)
            return outs
        return res


# ------------------------------------------------------------------ compute
class CudaRank:
    """Local compute of one rank over libmoe_cuda.so (a MoELayer holding the
    full gate and only this rank's experts)."""

    def __init__(self, layer):
        self.L = layer
        self.E = layer.E

    def route(self, x, fin, k):
        self.L.route(x, fin, k)
        import torch
        off = torch.empty(self.L.E + 1, dtype=torch.int32)
        from . import abi
        import ctypes as C
        abi.call("moe_cuda_memcpy", C.c_void_p(off.data_ptr()), C.c_void_p(self.L.offsets_device()),
                 (self.L.E + 1) * 4, 1, None)
        return off.numpy().view(np.uint32).astype(np.int64)

    def sorted_rows(self, n):
        return _dev_view(self.L.buffers()[0], n, self.L.d)

    def y_rows(self, n):
        return _dev_view(self.L.buffers()[1], n, self.L.d)

    def gather(self, x, idx):
        from . import ops
        import torch
        if x.shape[0] == 0:
            return x.clone()
        p = torch.as_tensor(idx.astype(np.int32), device=x.device)
        return ops.permute_rows(x, p)

    def experts(self, xe, problems, mode):
        import torch
        if xe.shape[0] == 0:
            return torch.empty_like(xe)
        pr = torch.as_tensor(problems.astype(np.int32), device=xe.device)
        return self.L.experts(xe, pr, mode=mode)

    def combine(self, x, fin, k, y_sorted):
        return self.L.combine(x, self.L.buffers()[1], fin, k)


class _CAI:
    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f2", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _dev_view(ptr, rows, cols):
    """torch view (no copy) of rows x cols fp16 at a device pointer."""
    import torch
    if rows == 0:
        return torch.empty((0, cols), dtype=torch.float16, device="cuda")
    return torch.as_tensor(_CAI(ptr, (rows, cols)), device="cuda")


# ------------------------------------------------------------------ forward
def ep_forward(ranks, comm, xs, fins, k=1, mode=1):
    """One expert-parallel MoE layer forward.

    ranks: local compute per rank state (CudaRank or a test double);
    xs / fins: per-state input rows / finished flags (None = none finished).
    Returns the per-state outputs (same shapes as xs)."""
    n = len(ranks)
    G = comm.world
    E = ranks[0].E
    el = E // G
    offs = [ranks[i].route(xs[i], fins[i], k) for i in range(n)]
    # 2. counts (G, el) -> exchanged
    sc = [send_counts(o, E, G) for o in offs]
    import torch
    cnt_dev = "cpu" if not xs[0].is_cuda else xs[0].device
    sends = [torch.as_tensor(c.reshape(-1), dtype=torch.int64, device=cnt_dev) for c in sc]
    recv = comm.all_to_all(sends, [[el] * G] * n, [[el] * G] * n)
    rc = [r.cpu().numpy().reshape(G, el) for r in recv]
    send_rows = [c.sum(1) for c in sc]
    recv_rows = [c.sum(1) for c in rc]
    active = [int(o[E]) for o in offs]
    # 3. dispatch
    xsend = [ranks[i].sorted_rows(active[i]) for i in range(n)]
    xrecv = comm.all_to_all(xsend, send_rows, recv_rows)
    # 4./5. regroup + experts
    yrecv = []
    for i in range(n):
        perm, probs = regroup(rc[i])
        xe = ranks[i].gather(xrecv[i], perm)
        ye = ranks[i].experts(xe, probs, mode)
        yrecv.append(ranks[i].gather(ye, inverse(perm)))
    # 6. reverse all-to-all straight into each rank's sorted y, then local combine
    ys = [ranks[i].y_rows(active[i]) for i in range(n)]
    comm.all_to_all(yrecv, recv_rows, send_rows, outs=ys)
    return [ranks[i].combine(xs[i], fins[i], k, ys[i]) for i in range(n)]


class EPMoELayer:
    """Distributed EP layer for this process's rank: the full gate plus the
    owned experts on this GPU, NCCL transport."""

    def __init__(self, ln_g, ln_b, gate_w, gate_b, w1, b1, w2, b2, bits=4, group=None,
                 device="cuda"):
        import torch.distributed as dist
        from .ops import MoELayer
        self.comm = DistComm(group)
        G, g = self.comm.world, dist.get_rank(group)
        E = gate_w.shape[1]
        e0, el = owner_range(E, G, g)
        sl = slice(e0, e0 + el)
        layer = MoELayer(ln_g, ln_b, gate_w, gate_b, w1[sl], b1[sl], w2[sl], b2[sl], bits=bits,
                         device=device, expert_range=(e0, el))
        self.rank = CudaRank(layer)

    def forward(self, x, finished=None, k=1, mode=1):
        return ep_forward([self.rank], self.comm, [x], [finished], k=k, mode=mode)[0]
