"""Expert parallelism for the MoE layer.

A thin wrapper over the C-ABI (include/moe_cuda.h `moe_ep_*`,
csrc/ep.cu): G ranks, one process per GPU; rank g owns experts
[g*E/G, (g+1)*E/G) and brings its own tokens.  The whole forward -- route,
device-side count exchange, per-(peer, expert) NCCL send/recv dispatch into
expert-major order, local grouped GEMMs, reverse exchange, combine -- runs
in C++/CUDA; Python only creates the communicator (the NCCL unique id is
broadcast over torch.distributed) and passes pointers.

`LoopbackEP` holds all G ranks in one process on one device (the same
orchestration with device-to-device copies as the transport): the G > 1
test path on a single GPU.  `segments` is the pure host arithmetic of the
exchange (moe_ep_segments), callable without a GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi

ID_BYTES = 128


def owner_range(E: int, G: int, g: int):
    """(first expert, count) owned by rank g (E % G == 0)."""
    if E % G != 0:
        raise ValueError("ep: n_experts must be divisible by the world size")
    el = E // G
    return g * el, el


def segments(G: int, el: int, send_cnt, recv_cnt):
    """moe_ep_segments: (send_off [G*el], recv_dst [G*el], problems (el, 3),
    rows received) from the per-(peer, local expert) sent / received counts."""
    sc = np.ascontiguousarray(send_cnt, np.uint32).reshape(-1)
    rc = np.ascontiguousarray(recv_cnt, np.uint32).reshape(-1)
    so = np.zeros(G * el, np.int64)
    rd = np.zeros(G * el, np.int64)
    pr = np.zeros((el, 3), np.uint32)
    rows = C.c_int64()
    abi.call("moe_ep_segments", G, el, C.c_void_p(sc.ctypes.data), C.c_void_p(rc.ctypes.data),
             C.c_void_p(so.ctypes.data), C.c_void_p(rd.ctypes.data), C.c_void_p(pr.ctypes.data),
             C.byref(rows))
    return so, rd, pr, rows.value


def _ptrs(ts, ctype=C.c_void_p):
    arr = (ctype * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = None if t is None else t.data_ptr()
    return arr


class _EP:
    """Owner of a moe_ep handle."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                abi.lib().moe_ep_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def world(self):
        g, r, n = C.c_int(), C.c_int(), C.c_int()
        abi.call("moe_ep_world", self._h, C.byref(g), C.byref(r), C.byref(n))
        return g.value, r.value, n.value

    def _forward(self, layers, xs, fins, k, mode, outs, stream):
        import torch
        n = len(layers)
        Ls = (C.c_void_p * n)(*[L._h.value for L in layers])
        Ts = (C.c_int64 * n)(*[x.shape[0] for x in xs])
        s = stream if stream is not None else torch.cuda.current_stream()
        fin_arr = None if all(f is None for f in fins) else _ptrs(fins)
        abi.call("moe_ep_forward", self._h, Ls, _ptrs(xs), fin_arr, Ts, k, mode, _ptrs(outs),
                 C.c_void_p(s.cuda_stream))
        return outs

    def counts(self, local=0):
        """(sent (G, el), received (G, el), rows received) of the last forward."""
        G, _, _ = self.world()
        E = self._E
        sc = np.zeros(E, np.uint32)
        rc = np.zeros(E, np.uint32)
        rows = C.c_int64()
        abi.call("moe_ep_counts", self._h, local, C.c_void_p(sc.ctypes.data),
                 C.c_void_p(rc.ctypes.data), C.byref(rows))
        return sc.reshape(G, -1), rc.reshape(G, -1), rows.value


class EPMoELayer(_EP):
    """This process's rank of an EP layer: the full gate plus the owned
    experts on the current GPU, NCCL transport.  torch.distributed must be
    initialised (any backend: it only carries the 128-byte NCCL id)."""

    def __init__(self, ln_g, ln_b, gate_w, gate_b, w1, b1, w2, b2, bits=4, group=None,
                 device="cuda", q=None, sliced=False):
        """w1/b1/w2/b2 (and q): all E experts, or (sliced=True) only this
        rank's E/G experts."""
        import torch
        import torch.distributed as dist
        from .ops import MoELayer
        G, g = dist.get_world_size(group), dist.get_rank(group)
        E = gate_w.shape[1]
        e0, el = owner_range(E, G, g)
        sl = slice(0, el) if sliced else slice(e0, e0 + el)
        if q is not None and not sliced:
            raise ValueError("EPMoELayer: pass q payloads already sliced to this rank (sliced=True)")
        self.layer = MoELayer(ln_g, ln_b, gate_w, gate_b, None if w1 is None else w1[sl], b1[sl],
                              None if w2 is None else w2[sl], b2[sl], bits=bits, device=device,
                              expert_range=(e0, el), q=q)
        idb = torch.zeros(ID_BYTES, dtype=torch.uint8)
        if g == 0:
            raw = (C.c_uint8 * ID_BYTES)()
            abi.call("moe_ep_unique_id", raw)
            idb = torch.tensor(list(bytes(raw)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            idb = idb.to(device)
        dist.broadcast(idb, src=dist.get_global_rank(group, 0) if group is not None else 0,
                       group=group)
        raw = (C.c_uint8 * ID_BYTES)(*idb.cpu().tolist())
        h = C.c_void_p()
        abi.call("moe_ep_create", raw, G, g, C.byref(h))
        super().__init__(h)
        self._E = E
        self.E, self.rank, self.world_size = E, g, G

    def forward(self, x, finished=None, k=1, mode=abi.MODE_FAST, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty_like(x)
        self._forward([self.layer], [x], [finished], k, mode, [out], stream)
        return out


class LoopbackEP(_EP):
    """All G ranks of an EP layer in this process on one device (test path):
    layers[g] holds rank g's experts (MoELayer(..., expert_range=(g*el, el)))."""

    def __init__(self, layers):
        G = len(layers)
        h = C.c_void_p()
        abi.call("moe_ep_create_loopback", G, C.byref(h))
        super().__init__(h)
        self.layers = layers
        self._E = layers[0].E

    def forward(self, xs, fins=None, k=1, mode=abi.MODE_FAST, outs=None, stream=None):
        import torch
        if fins is None:
            fins = [None] * len(xs)
        if outs is None:
            outs = [torch.empty_like(x) for x in xs]
        return self._forward(self.layers, xs, fins, k, mode, outs, stream)
