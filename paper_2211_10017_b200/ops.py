"""Device-side operators over the C-ABI, on torch CUDA tensors.

torch supplies device memory and streams only (plumbing); every computation
is one of libmoe_cuda.so's sm_100a kernels.  Names follow the reference's
hot-path API (proj/include/moeinfer/*.hpp); each wrapper cites the entry
point it calls.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import abi

MODE_EXACT, MODE_FAST, MODE_GEMV = abi.MODE_EXACT, abi.MODE_FAST, abi.MODE_GEMV


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _chk_cuda(*ts):
    for t in ts:
        if t is not None:
            assert t.is_cuda and t.is_contiguous(), "expected contiguous CUDA tensors"


def quantize(w: torch.Tensor, bits: int, stream=None):
    """moe_quantize (replaces moe::quantize, proj/src/quantize.cpp:74-122).

    w: (E, m, n) float16 CUDA tensor -> (packed uint8, scales float16 (E, n))."""
    _chk_cuda(w)
    E, m, n = w.shape
    nbytes = E * m * n // 2 if bits == 4 else E * m * n
    packed = torch.empty(nbytes, dtype=torch.uint8, device=w.device)
    scales = torch.empty((E, n), dtype=torch.float16, device=w.device)
    abi.call("moe_quantize", _p(w), E, m, n, bits, _p(packed), _p(scales), _stream(stream))
    return packed, scales


def dequantize(packed, scales, shape, bits, fast=True, stream=None):
    """moe_dequantize (dequantize_fast / dequantize_naive, proj/src/dequant.cpp:55-112)."""
    E, m, n = shape
    out = torch.empty((E, m, n), dtype=torch.float16, device=packed.device)
    abi.call("moe_dequantize", _p(packed), _p(scales), E, m, n, bits, int(fast), _p(out),
             _stream(stream))
    return out


def pack_int4(values, stream=None):
    out = torch.empty(values.numel() // 2, dtype=torch.uint8, device=values.device)
    abi.call("moe_pack_int4", _p(values), values.numel(), _p(out), _stream(stream))
    return out


def unpack_int4(packed, count, stream=None):
    out = torch.empty(count, dtype=torch.uint8, device=packed.device)
    abi.call("moe_unpack_int4", _p(packed), count, _p(out), _stream(stream))
    return out


def tile_weights(src, E, m, n, bits, stream=None):
    nbytes = abi.lib().moe_tiled_bytes(E, m, n, bits)
    out = torch.empty(nbytes, dtype=torch.uint8, device=src.device)
    abi.call("moe_tile_weights", _p(src), E, m, n, bits, _p(out), _stream(stream))
    return out


def layer_norm(x, gamma, beta, stream=None):
    """moe_layer_norm (proj/src/model.cpp:175-205)."""
    T, d = x.shape
    out = torch.empty_like(x)
    abi.call("moe_layer_norm", _p(x), T, d, _p(gamma), _p(beta), _p(out), _stream(stream))
    return out


def gate_logits(xn, gw, gb, stream=None):
    """moe_gate_logits (proj/src/model.cpp:273-297)."""
    T, d = xn.shape
    E = gw.shape[1]
    out = torch.empty((T, E), dtype=torch.float32, device=xn.device)
    abi.call("moe_gate_logits", _p(xn), T, d, _p(gw), _p(gb), E, _p(out), _stream(stream))
    return out


def gate_topk(logits, k=1, stream=None):
    """moe_gate_topk (gate_top1, proj/src/routing.cpp:11-41, top-k extension)."""
    T, E = logits.shape
    ex = torch.empty((T, k), dtype=torch.int32, device=logits.device)
    sc = torch.empty((T, k), dtype=torch.float16, device=logits.device)
    abi.call("moe_gate_topk", _p(logits), T, E, k, _p(ex), _p(sc), _stream(stream))
    return ex, sc


def routing_plan(expert, finished, E, stream=None):
    """moe_routing_plan (build_routing_plan, proj/src/routing.cpp:43-87)."""
    T, k = expert.shape
    S = T * k
    dev = expert.device
    perm = torch.empty(S, dtype=torch.int32, device=dev)
    inv = torch.empty(S, dtype=torch.int32, device=dev)
    offs = torch.empty(E + 1, dtype=torch.int32, device=dev)
    probs = torch.empty((E, 3), dtype=torch.int32, device=dev)
    active = torch.empty(1, dtype=torch.int32, device=dev)
    abi.call("moe_routing_plan", _p(expert), _p(finished), T, k, E, _p(perm), _p(inv), _p(offs),
             _p(probs), _p(active), _stream(stream))
    return perm, inv, offs, probs, active


def permute_rows(x, perm, k=1, stream=None):
    S = perm.numel()
    out = torch.empty((S, x.shape[1]), dtype=x.dtype, device=x.device)
    abi.call("moe_permute_rows", _p(x), x.shape[1], _p(perm), S, k, _p(out), _stream(stream))
    return out


def unpermute_scale(y, perm, active, scale, stream=None):
    T, cols = y.shape
    out = torch.empty_like(y)
    abi.call("moe_unpermute_scale", _p(y), T, cols, _p(perm), _p(active), _p(scale), _p(out),
             _stream(stream))
    return out


def combine(x, y, inv, scale, finished, k=1, stream=None):
    """moe_combine (residual + gate-scaled un-permute, proj/src/model.cpp:334-346)."""
    T, d = x.shape
    out = torch.empty_like(x)
    abi.call("moe_combine", _p(x), _p(y), _p(inv), _p(scale), _p(finished), T, d, k, _p(out),
             _stream(stream))
    return out


def grouped_gemm(x, problems, tiled, scales, bits, E, n, bias, relu, mode, out=None,
                 stream=None):
    """moe_grouped_gemm (grouped_gemm_f16 / grouped_gemm_quant,
    proj/src/grouped_gemm.cpp:140-214).  problems: (np, 3) int32 CUDA tensor."""
    rows, m = x.shape
    if out is None:
        out = torch.zeros((rows, n), dtype=torch.float16, device=x.device)
    abi.call("moe_grouped_gemm", _p(x), rows, m, _p(problems), problems.shape[0], _p(tiled),
             _p(scales), bits, E, n, _p(bias), int(relu), mode, _p(out), _stream(stream))
    return out


class MoELayer:
    """Device-resident MoE FFN block (replaces moe::moe_ffn_forward,
    proj/src/model.cpp:299-349).  Weights are uploaded and tiled once.

    Construct from FP16 master weights (numpy or torch) with ``bits`` 16/8/4;
    for 8/4 the experts are quantized ON THE GPU by moe_quantize unless
    ``q=(q1, s1, q2, s2)`` payloads (reference layout) are given.
    """

    def __init__(self, ln_g, ln_b, gate_w, gate_b, w1, b1, w2, b2, bits=4, q=None,
                 device="cuda", expert_range=None):
        """expert_range=(e_begin, e_count): w1/w2/b1/b2 (and q) hold only those
        experts (expert parallelism); the gate always covers all E."""
        def T(a):
            if isinstance(a, torch.Tensor):
                return a.to(device).contiguous()
            import numpy as np
            a = np.ascontiguousarray(a)
            t = torch.from_numpy(a.view(np.int16) if a.dtype == np.float16 else a)
            t = t.to(device)
            return t.view(torch.float16) if a.dtype == np.float16 else t

        self.bits = bits
        d, E = gate_w.shape
        f = (w1.shape[2] if w1 is not None else q[1].shape[1])
        self.d, self.f, self.E = d, f, E
        self.e_begin, self.e_count = expert_range if expert_range else (0, E)
        keep = dict(ln_g=T(ln_g), ln_b=T(ln_b), gate_w=T(gate_w), gate_b=T(gate_b), b1=T(b1),
                    b2=T(b2))
        if bits == 16:
            keep.update(w1=T(w1), w2=T(w2))
        else:
            if q is None:
                q1, s1 = quantize(T(w1), bits)
                q2, s2 = quantize(T(w2), bits)
            else:
                q1, s1, q2, s2 = (T(a) for a in q)
            keep.update(q1=q1, s1=s1, q2=q2, s2=s2)
        desc = abi.LayerDesc(d, f, E, bits, *[
            keep[nm].data_ptr() if nm in keep else None
            for nm in ("ln_g", "ln_b", "gate_w", "gate_b", "b1", "b2", "w1", "w2", "q1", "q2",
                       "s1", "s2")], *((self.e_begin, self.e_count) if expert_range else (0, 0)))
        h = C.c_void_p()
        torch.cuda.synchronize()
        abi.call("moe_layer_create_device", C.byref(desc), C.byref(h))
        self._h = h
        self.quant = (keep.get("q1"), keep.get("s1"), keep.get("q2"), keep.get("s2"))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                abi.lib().moe_layer_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def reserve(self, T, k=1):
        abi.call("moe_layer_reserve", self._h, T, k)

    def forward(self, x, finished=None, k=1, mode=MODE_FAST, out=None, stream=None,
                graph=False):
        """Device-resident forward (no host sync, graph-capturable).  graph=True
        replays a cached CUDA graph of this argument set (moe_layer_forward_graph)."""
        T = x.shape[0]
        if out is None:
            out = torch.empty_like(x)
        abi.call("moe_layer_forward_graph" if graph else "moe_layer_forward", self._h, _p(x),
                 _p(finished), T, k, mode, _p(out), _stream(stream))
        return out

    def forward_host(self, x_host, finished_host=None, k=1, mode=MODE_FAST, out_host=None,
                     stream=None):
        """Host-buffer forward (numpy in, numpy out): the drop-in / e2e path."""
        import numpy as np
        x_host = np.ascontiguousarray(x_host)
        T = x_host.shape[0]
        if out_host is None:
            out_host = np.empty_like(x_host)
        fin = None if finished_host is None else np.ascontiguousarray(finished_host, np.uint8)
        abi.call("moe_layer_forward_host", self._h, C.c_void_p(x_host.ctypes.data),
                 None if fin is None else C.c_void_p(fin.ctypes.data), T, k, mode,
                 C.c_void_p(out_host.ctypes.data), _stream(stream))
        return out_host

    def status(self, stream=None):
        abi.call("moe_layer_status", self._h, _stream(stream))

    def routing(self, T, k=1):
        """Copies of the last forward's routing (host numpy)."""
        import numpy as np
        ptrs = [C.c_void_p() for _ in range(6)]
        abi.call("moe_layer_routing", self._h, *[C.byref(p) for p in ptrs])
        S, E = T * k, self.E

        def get(ptr, count, dt):
            a = np.empty(count, dt)
            abi.call("moe_cuda_memcpy", C.c_void_p(a.ctypes.data), ptr, a.nbytes, 1, None)
            return a

        torch.cuda.synchronize()
        return dict(expert=get(ptrs[0], S, np.uint32).reshape(T, k),
                    scale=get(ptrs[1], S, np.uint16).reshape(T, k),
                    perm=get(ptrs[2], S, np.uint32), inv=get(ptrs[3], S, np.uint32),
                    offsets=get(ptrs[4], E + 1, np.uint32),
                    active=int(get(ptrs[5], 1, np.uint32)[0]))

    # ---- expert-parallel building blocks (moe_layer_route / _experts / _combine)
    def route(self, x, finished=None, k=1, stream=None):
        """LN -> gate -> top-k -> plan -> gather into the layer workspace."""
        abi.call("moe_layer_route", self._h, _p(x), _p(finished), x.shape[0], k, _stream(stream))

    def buffers(self):
        """(xp, y) device pointers of the layer workspace (expert-sorted rows)."""
        xp, y = C.c_void_p(), C.c_void_p()
        abi.call("moe_layer_buffers", self._h, C.byref(xp), C.byref(y))
        return xp.value, y.value

    def experts(self, xin, problems, mode=MODE_FAST, out=None, stream=None):
        """FFN1+FFN2 of the LOCAL experts over expert-sorted rows; problems:
        (np, 3) int32 device tensor with local expert ids."""
        rows = xin.shape[0]
        if out is None:
            out = torch.empty((rows, self.d), dtype=torch.float16, device=xin.device)
        abi.call("moe_layer_experts", self._h, _p(xin), rows, _p(problems), problems.shape[0],
                 mode, _p(out), _stream(stream))
        return out

    def combine(self, x, y_ptr, finished=None, k=1, out=None, stream=None):
        """out = finished ? x : x + sum_s y[inv[r,s]] * scale[r,s] (last route's plan)."""
        if out is None:
            out = torch.empty_like(x)
        abi.call("moe_layer_combine", self._h, _p(x), C.c_void_p(y_ptr), _p(finished),
                 x.shape[0], k, _p(out), _stream(stream))
        return out

    def ffn(self, mode=MODE_FAST, stream=None):
        """Re-run FFN1 + FFN2 on the last forward's routed rows (moe_layer_ffn)."""
        abi.call("moe_layer_ffn", self._h, mode, _stream(stream))

    def offsets_device(self):
        """(E+1) int32 device view of the last plan's expert offsets."""
        ptrs = [C.c_void_p() for _ in range(6)]
        abi.call("moe_layer_routing", self._h, *[C.byref(p) for p in ptrs])
        return ptrs[4].value

    STAGES = ("layer_norm", "gate_logits", "gate_topk", "routing_plan", "ffn1", "ffn2",
              "combine")

    def profile(self, enable=True):
        """Start (reset) / stop CUDA-event timing (moe_layer_profile): 1 / True =
        grouped-GEMM boundaries only, 2 = every stage, 0 / False = off."""
        abi.call("moe_layer_profile", self._h, int(enable))

    def profile_read(self):
        """(summed ms per stage, forwards recorded) (moe_layer_profile_read)."""
        import numpy as np
        ms = np.zeros(len(self.STAGES), np.float64)
        n = C.c_int()
        abi.call("moe_layer_profile_read", self._h, C.c_void_p(ms.ctypes.data), C.byref(n))
        return dict(zip(self.STAGES, ms.tolist())), n.value

    def traffic(self, stream=None):
        import numpy as np
        t = np.zeros(6, np.uint64)
        abi.call("moe_layer_traffic", self._h, C.c_void_p(t.ctypes.data), _stream(stream))
        return dict(expert=tuple(int(v) for v in t[:3]), other=tuple(int(v) for v in t[3:]))

    def load_report(self, capacity_factor=1.0, stream=None):
        """Expert-capacity bookkeeping of the last routed forward
        (moe_layer_load_report): per-expert live rows, the capacity
        ceil(cf * live / E), max load, experts / rows over capacity.  Nothing
        is dropped (the reference routes every live slot)."""
        import numpy as np
        E = self.E
        rep = torch.empty(E + 8, dtype=torch.int32, device="cuda")
        abi.call("moe_layer_load_report", self._h, C.c_float(capacity_factor), _p(rep),
                 _stream(stream))
        r = rep.cpu().numpy().view(np.uint32)
        load = r[:E].astype(np.int64)
        live = int(r[E + 2])
        return dict(load=load, capacity=int(r[E]), max_load=int(r[E + 1]), live_slots=live,
                    experts_over=int(r[E + 3]), overflow_rows=int(r[E + 4]),
                    active_experts=int(r[E + 5]),
                    imbalance=float(r[E + 1]) / (live / E) if live else 0.0,
                    capacity_factor=capacity_factor)


class HostBuffer:
    """Pinned host memory from the library (moe_cuda_host_alloc, or
    write-combined moe_cuda_host_alloc_wc for streaming inputs the host only
    writes) exposed as a numpy array; freed with the object."""

    def __init__(self, shape, dtype, write_combined=False):
        import numpy as np
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        p = C.c_void_p()
        abi.call("moe_cuda_host_alloc_wc" if write_combined else "moe_cuda_host_alloc", C.byref(p), n)
        self._p = p
        buf = (C.c_uint8 * n).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dt).reshape(shape)

    def __del__(self):
        p = getattr(self, "_p", None)
        if p:
            try:
                abi.lib().moe_cuda_host_free(p)
            except Exception:
                pass
            self._p = None
