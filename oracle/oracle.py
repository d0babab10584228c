"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes faces over the two CHECKERS:

* ``Oracle``    -- oracle/liboracle.so, the plain-C restatement
                   (oracle/moe_oracle.c) of the reference hot path;
* ``Reference`` -- oracle/_ref/libmoeref.so, the unmodified reference engine
                   built from /root/reference/proj/src by oracle/Makefile
                   (absent when the reference was not available at build time).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  FP16 tensors are numpy
float16 arrays (bit patterns viewed as uint16 at the boundary).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoeref.so")

_p = C.c_void_p
_sz = C.c_size_t


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _u16(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.float16:
        return a.view(np.uint16)
    assert a.dtype == np.uint16, a.dtype
    return a


class OracleError(ValueError):
    pass


@dataclass
class LayerWeights:
    """One MoE FFN block (model.hpp:73-84), FP16 master weights."""

    ln_g: np.ndarray
    ln_b: np.ndarray
    gw: np.ndarray  # (d, E)
    gb: np.ndarray  # (E,)
    w1: np.ndarray  # (E, d, f)
    b1: np.ndarray  # (E, f)
    w2: np.ndarray  # (E, f, d)
    b2: np.ndarray  # (E, d)

    @property
    def d(self):
        return self.gw.shape[0]

    @property
    def E(self):
        return self.gw.shape[1]

    @property
    def f(self):
        return self.w1.shape[2]


def random_layer(d, f, E, seed=1234, dtype=np.float16):
    """Synthetic weights with random_model's MoE init (model.cpp:87-114)."""
    rng = np.random.default_rng(seed)
    s1, s2 = 1.0 / np.sqrt(d), 1.0 / np.sqrt(f)
    n = lambda shape, s: (rng.standard_normal(shape) * s).astype(dtype)
    return LayerWeights(
        ln_g=(1.0 + 0.1 * rng.standard_normal(d)).astype(dtype),
        ln_b=(0.05 * rng.standard_normal(d)).astype(dtype),
        gw=n((d, E), s1),
        gb=n((E,), 0.02),
        w1=n((E, d, f), s1),
        b1=n((E, f), 0.02),
        w2=n((E, f, d), s2),
        b2=n((E, d), 0.02),
    )


class Oracle:
    """The C restatement (oracle/moe_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_last_error.restype = C.c_char_p
        L.or_half_to_f32.restype = C.c_float
        L.or_half_to_f32.argtypes = [C.c_uint16]
        for nm in ("or_f32_to_half",):
            getattr(L, nm).restype = C.c_uint16
            getattr(L, nm).argtypes = [C.c_float]
        L.or_f64_to_half.restype = C.c_uint16
        L.or_f64_to_half.argtypes = [C.c_double]
        for nm in ("or_half_add", "or_half_sub", "or_half_mul"):
            getattr(L, nm).restype = C.c_uint16
            getattr(L, nm).argtypes = [C.c_uint16, C.c_uint16]
        L.or_quant_scale.restype = C.c_uint16
        L.or_quant_scale.argtypes = [C.c_float, C.c_int]
        L.or_quant_encode.restype = C.c_uint8
        L.or_quant_encode.argtypes = [C.c_uint16, C.c_uint16, C.c_int]
        L.or_expf.restype = C.c_float
        L.or_expf.argtypes = [C.c_float]
        L.or_debias_u8.restype = C.c_uint16
        L.or_debias_u4.restype = C.c_uint16
        L.or_make_problems.restype = _sz
        L.or_make_problems.argtypes = [_p, _sz, _p]

    def _chk(self, st):
        if st != 0:
            raise OracleError(self.lib.or_last_error().decode())

    # scalar helpers -------------------------------------------------------
    def f32_to_half(self, x):
        return self.lib.or_f32_to_half(float(x))

    def half_to_f32(self, h):
        return self.lib.or_half_to_f32(int(h))

    # quantizer -------------------------------------------------------------
    def quantize(self, w, bits):
        w = _u16(w)
        e, m, n = w.shape
        nb = e * m * n // 2 if bits == 4 else e * m * n
        packed = np.zeros(nb, np.uint8)
        scales = np.zeros((e, n), np.uint16)
        self._chk(self.lib.or_quantize(_ptr(w), _sz(e), _sz(m), _sz(n), C.c_int(bits),
                                       _ptr(packed), _ptr(scales)))
        return packed, scales.view(np.float16)

    def pack_int4(self, v):
        v = np.ascontiguousarray(v, np.uint8)
        out = np.zeros(len(v) // 2, np.uint8)
        self._chk(self.lib.or_pack_int4(_ptr(v), _sz(len(v)), _ptr(out)))
        return out

    def unpack_int4(self, p, count):
        p = np.ascontiguousarray(p, np.uint8)
        out = np.zeros(count, np.uint8)
        self._chk(self.lib.or_unpack_int4(_ptr(p), _sz(count), _ptr(out)))
        return out

    def dequantize(self, packed, scales, shape, bits, fast=True):
        e, m, n = shape
        out = np.zeros(shape, np.uint16)
        self._chk(self.lib.or_dequantize(_ptr(np.ascontiguousarray(packed, np.uint8)),
                                         _ptr(_u16(scales)), _sz(e), _sz(m), _sz(n),
                                         C.c_int(bits), C.c_int(int(fast)), _ptr(out)))
        return out.view(np.float16)

    # gate / routing ----------------------------------------------------------
    def layer_norm(self, x, g, b):
        x = _u16(x)
        T, d = x.shape
        out = np.zeros_like(x)
        self._chk(self.lib.or_layer_norm(_ptr(x), _sz(T), _sz(d), _ptr(_u16(g)), _ptr(_u16(b)),
                                         _ptr(out)))
        return out.view(np.float16)

    def gate_logits(self, xn, gw, gb):
        xn = _u16(xn)
        T, d = xn.shape
        E = gw.shape[1]
        out = np.zeros((T, E), np.float32)
        self._chk(self.lib.or_gate_logits(_ptr(xn), _sz(T), _sz(d), _ptr(_u16(gw)),
                                          _ptr(_u16(gb)), _sz(E), _ptr(out)))
        return out

    def gate_topk(self, logits, k=1):
        logits = np.ascontiguousarray(logits, np.float32)
        T, E = logits.shape
        ex = np.zeros((T, k), np.uint32)
        sc = np.zeros((T, k), np.uint16)
        self._chk(self.lib.or_gate_topk(_ptr(logits), _sz(T), _sz(E), C.c_int(k), _ptr(ex),
                                        _ptr(sc)))
        return ex, sc

    def routing_plan(self, expert, finished, E):
        expert = np.ascontiguousarray(expert, np.uint32)
        if expert.ndim == 1:
            expert = expert[:, None]
        T, k = expert.shape
        fin = np.ascontiguousarray(finished, np.uint8)
        S = T * k
        perm = np.zeros(S, np.uint32)
        inv = np.zeros(S, np.uint32)
        offs = np.zeros(E + 1, np.uint32)
        act = C.c_uint32(0)
        self._chk(self.lib.or_routing_plan(_ptr(expert), _ptr(fin), _sz(T), C.c_int(k), _sz(E),
                                           _ptr(perm), _ptr(inv), _ptr(offs), C.byref(act)))
        return perm, inv, offs, act.value

    def make_problems(self, offsets):
        offsets = np.ascontiguousarray(offsets, np.uint32)
        E = len(offsets) - 1
        out = np.zeros((E, 3), np.uint32)
        npb = self.lib.or_make_problems(_ptr(offsets), _sz(E), _ptr(out))
        return out[:npb].copy()

    def grouped_gemm(self, x, problems, *, bits, w16=None, packed=None, scales=None, E, n,
                     bias, relu, separate=False):
        x = _u16(x)
        rows, m = x.shape
        problems = np.ascontiguousarray(problems, np.uint32).reshape(-1, 3)
        out = np.zeros((rows, n), np.uint16)
        tr = np.zeros(3, np.uint64)
        self._chk(self.lib.or_grouped_gemm(
            _ptr(x), _sz(rows), _sz(m), _ptr(problems), _sz(len(problems)), C.c_int(bits),
            _ptr(None if w16 is None else _u16(w16)),
            _ptr(None if packed is None else np.ascontiguousarray(packed, np.uint8)),
            _ptr(None if scales is None else _u16(scales)), _sz(E), _sz(n), _ptr(_u16(bias)),
            C.c_int(int(relu)), C.c_int(int(separate)), _ptr(out), _ptr(tr)))
        return out.view(np.float16), tuple(int(t) for t in tr)

    # whole layer ---------------------------------------------------------------
    def _layer_struct(self, lw: LayerWeights, bits, q=None):
        class OrLayer(C.Structure):
            _fields_ = [("d", _sz), ("f", _sz), ("E", _sz), ("bits", C.c_int)] + [
                (nm, _p) for nm in ("ln_g", "ln_b", "gw", "gb", "b1", "b2", "w1", "w2", "q1",
                                    "q2", "s1", "s2")]

        keep = []

        def P(a):
            if a is None:
                return None
            a = np.ascontiguousarray(a)
            if a.dtype == np.float16:
                a = a.view(np.uint16)
            keep.append(a)
            return a.ctypes.data

        if bits != 16 and q is None:
            q = (*self.quantize(lw.w1, bits), *self.quantize(lw.w2, bits))
        s = OrLayer(lw.d, lw.f, lw.E, bits, P(lw.ln_g), P(lw.ln_b), P(lw.gw), P(lw.gb),
                    P(lw.b1), P(lw.b2), P(lw.w1 if bits == 16 else None),
                    P(lw.w2 if bits == 16 else None), P(q[0] if q else None),
                    P(q[2] if q else None), P(q[1] if q else None), P(q[3] if q else None))
        return s, keep

    def moe_forward(self, lw: LayerWeights, x, finished=None, k=1, bits=16, q=None,
                    diagnostics=False):
        x = _u16(x)
        T, d = x.shape
        fin = np.zeros(T, np.uint8) if finished is None else np.ascontiguousarray(finished,
                                                                                  np.uint8)
        s, keep = self._layer_struct(lw, bits, q)
        out = np.zeros_like(x)
        S, E = T * k, lw.E
        ex = np.zeros((T, k), np.uint32)
        sc = np.zeros((T, k), np.uint16)
        perm = np.zeros(S, np.uint32)
        inv = np.zeros(S, np.uint32)
        offs = np.zeros(E + 1, np.uint32)
        act = C.c_uint32(0)
        self._chk(self.lib.or_moe_forward(C.byref(s), _ptr(x), _sz(T), _ptr(fin), C.c_int(k),
                                          _ptr(out), _ptr(ex), _ptr(sc), _ptr(perm), _ptr(inv),
                                          _ptr(offs), C.byref(act)))
        if diagnostics:
            return out.view(np.float16), dict(expert=ex, scale=sc, perm=perm, inv=inv,
                                             offsets=offs, active=act.value)
        return out.view(np.float16)

    def moe_per_token(self, lw: LayerWeights, x, finished=None, k=1, bits=16, q=None):
        x = _u16(x)
        T, d = x.shape
        fin = np.zeros(T, np.uint8) if finished is None else np.ascontiguousarray(finished,
                                                                                  np.uint8)
        s, keep = self._layer_struct(lw, bits, q)
        out = np.zeros_like(x)
        self._chk(self.lib.or_moe_per_token(C.byref(s), _ptr(x), _sz(T), _ptr(fin), C.c_int(k),
                                            _ptr(out)))
        return out.view(np.float16)


def reference_available():
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference engine (oracle/_ref/libmoeref.so)."""

    def __init__(self, path=REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_layer_create.restype = _p
        L.ref_layer_create.argtypes = [_sz, _sz, _sz] + [_p] * 8 + [C.c_int, C.c_int]
        L.ref_layer_create_quant.restype = _p
        L.ref_layer_create_quant.argtypes = [_sz, _sz, _sz] + [_p] * 10 + [C.c_int]
        L.ref_layer_destroy.argtypes = [_p]
        L.ref_layer_forward.argtypes = [_p, _p, _sz, _sz, _p, C.c_int, _p, _p]
        L.ref_layer_forward_topk.argtypes = [_p, _p, _sz, _sz, _p, C.c_int, C.c_int, _p]
        L.ref_layer_per_token.argtypes = [_p, _p, _sz, _sz, _p, _p]
        L.ref_layer_export_quant.argtypes = [_p, _p, _p, _p, _p]

    def _chk(self, st):
        if st != 0:
            raise OracleError(self.lib.ref_last_error().decode())

    def quantize(self, w, bits, threads=1):
        w = _u16(w)
        e, m, n = w.shape
        packed = np.zeros(e * m * n // 2 if bits == 4 else e * m * n, np.uint8)
        scales = np.zeros((e, n), np.uint16)
        self._chk(self.lib.ref_quantize(_ptr(w), _sz(e), _sz(m), _sz(n), C.c_int(bits),
                                        C.c_int(threads), _ptr(packed), _ptr(scales)))
        return packed, scales.view(np.float16)

    def ref_quantize(self, w, bits):
        w = _u16(w)
        e, m, n = w.shape
        stored = np.zeros(e * m * n, np.uint8)
        scales = np.zeros(e * n, np.float64)
        self._chk(self.lib.ref_ref_quantize(_ptr(w), _sz(e), _sz(m), _sz(n), C.c_int(bits),
                                            _ptr(stored), _ptr(scales)))
        return stored, scales

    def dequantize(self, packed, scales, shape, bits, fast=True):
        e, m, n = shape
        out = np.zeros(shape, np.uint16)
        self._chk(self.lib.ref_dequantize(_ptr(np.ascontiguousarray(packed, np.uint8)),
                                          _ptr(_u16(scales)), _sz(e), _sz(m), _sz(n),
                                          C.c_int(bits), C.c_int(int(fast)), _ptr(out)))
        return out.view(np.float16)

    def gate_top1(self, logits):
        logits = np.ascontiguousarray(logits, np.float32)
        T, E = logits.shape
        ex = np.zeros(T, np.uint32)
        sc = np.zeros(T, np.uint16)
        self._chk(self.lib.ref_gate_top1(_ptr(logits), _sz(T), _sz(E), _ptr(ex), _ptr(sc)))
        return ex, sc

    def build_plan(self, expert, finished, E):
        expert = np.ascontiguousarray(expert, np.uint32)
        T = len(expert)
        fin = np.ascontiguousarray(finished, np.uint8)
        perm = np.zeros(T, np.uint32)
        inv = np.zeros(T, np.uint32)
        offs = np.zeros(E + 1, np.uint32)
        act = C.c_uint32(0)
        self._chk(self.lib.ref_build_plan(_ptr(expert), _ptr(fin), _sz(T), _sz(E), _ptr(perm),
                                          _ptr(inv), _ptr(offs), C.byref(act)))
        return perm, inv, offs, act.value

    def layer_norm(self, x, g, b):
        x = _u16(x)
        T, d = x.shape
        out = np.zeros_like(x)
        self._chk(self.lib.ref_layer_norm(_ptr(x), _sz(T), _sz(d), _ptr(_u16(g)), _ptr(_u16(b)),
                                          _ptr(out)))
        return out.view(np.float16)

    def gate_logits(self, xn, gw, gb):
        xn = _u16(xn)
        T, d = xn.shape
        E = gw.shape[1]
        out = np.zeros((T, E), np.float32)
        self._chk(self.lib.ref_gate_logits(_ptr(xn), _sz(T), _sz(d), _ptr(_u16(gw)),
                                           _ptr(_u16(gb)), _sz(E), _ptr(out)))
        return out

    def grouped_gemm(self, x, problems, *, bits, w16=None, packed=None, scales=None, E, n,
                     bias, relu, separate=False, threads=1):
        x = _u16(x)
        rows, m = x.shape
        problems = np.ascontiguousarray(problems, np.uint32).reshape(-1, 3)
        out = np.zeros((rows, n), np.uint16)
        tr = np.zeros(3, np.uint64)
        if bits == 16:
            st = self.lib.ref_grouped_gemm_f16(
                _ptr(x), _sz(rows), _sz(m), _ptr(problems), _sz(len(problems)), _ptr(_u16(w16)),
                _sz(E), _sz(n), _ptr(_u16(bias)), C.c_int(int(relu)), C.c_int(threads),
                _ptr(out), _ptr(tr))
        else:
            st = self.lib.ref_grouped_gemm_quant(
                _ptr(x), _sz(rows), _sz(m), _ptr(problems), _sz(len(problems)),
                _ptr(np.ascontiguousarray(packed, np.uint8)), _ptr(_u16(scales)), C.c_int(bits),
                _sz(E), _sz(n), _ptr(_u16(bias)), C.c_int(int(relu)), C.c_int(int(not separate)),
                C.c_int(threads), _ptr(out), _ptr(tr))
        self._chk(st)
        return out.view(np.float16), tuple(int(t) for t in tr)

    def layer(self, lw: LayerWeights, bits=16, threads=1, q=None):
        return RefLayer(self, lw, bits, threads, q)


class RefLayer:
    def __init__(self, ref: Reference, lw: LayerWeights, bits, threads, q=None):
        self.ref, self.lw, self.bits = ref, lw, bits
        P = lambda a: _u16(a).ctypes.data
        # fp16 expert masters only when the reference quantizes them itself
        masters = (lw.w1, lw.w2) if q is None else ()
        self._keep = [_u16(a) for a in (lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.b1, lw.b2) + masters]
        if q is not None:
            q1, s1, q2, s2 = [np.ascontiguousarray(a) for a in q]
            self._keep += [q1, _u16(s1), q2, _u16(s2)]
            self.h = ref.lib.ref_layer_create_quant(
                lw.d, lw.f, lw.E, P(lw.ln_g), P(lw.ln_b), P(lw.gw), P(lw.gb), q1.ctypes.data,
                P(s1), P(lw.b1), q2.ctypes.data, P(s2), P(lw.b2), bits)
        else:
            self.h = ref.lib.ref_layer_create(lw.d, lw.f, lw.E, P(lw.ln_g), P(lw.ln_b),
                                              P(lw.gw), P(lw.gb), P(lw.w1), P(lw.b1), P(lw.w2),
                                              P(lw.b2), bits, threads)
        if not self.h:
            raise OracleError(ref.lib.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_layer_destroy(self.h)
            self.h = None

    def export_quant(self):
        lw = self.lw
        nb = lambda m, n: lw.E * m * n // (2 if self.bits == 4 else 1)
        q1 = np.zeros(nb(lw.d, lw.f), np.uint8)
        q2 = np.zeros(nb(lw.f, lw.d), np.uint8)
        s1 = np.zeros((lw.E, lw.f), np.uint16)
        s2 = np.zeros((lw.E, lw.d), np.uint16)
        self.ref._chk(self.ref.lib.ref_layer_export_quant(self.h, _ptr(q1), _ptr(s1), _ptr(q2),
                                                          _ptr(s2)))
        return q1, s1.view(np.float16), q2, s2.view(np.float16)

    def forward(self, x, finished=None, threads=1, k=1):
        x = _u16(x)
        T, d = x.shape
        fin = np.zeros(T, np.uint8) if finished is None else np.ascontiguousarray(finished,
                                                                                  np.uint8)
        out = np.zeros_like(x)
        if k == 1:
            st = self.ref.lib.ref_layer_forward(self.h, _ptr(x), T, d, _ptr(fin), threads,
                                                _ptr(out), None)
        else:
            st = self.ref.lib.ref_layer_forward_topk(self.h, _ptr(x), T, d, _ptr(fin), k,
                                                     threads, _ptr(out))
        self.ref._chk(st)
        return out.view(np.float16)

    def forward_topk(self, x, finished=None, k=1, threads=1):
        x = _u16(x)
        T, d = x.shape
        fin = np.zeros(T, np.uint8) if finished is None else np.ascontiguousarray(finished,
                                                                                  np.uint8)
        out = np.zeros_like(x)
        self.ref._chk(self.ref.lib.ref_layer_forward_topk(self.h, _ptr(x), T, d, _ptr(fin), k,
                                                          threads, _ptr(out)))
        return out.view(np.float16)

    def per_token(self, x, finished=None):
        x = _u16(x)
        T, d = x.shape
        fin = np.zeros(T, np.uint8) if finished is None else np.ascontiguousarray(finished,
                                                                                  np.uint8)
        out = np.zeros_like(x)
        self.ref._chk(self.ref.lib.ref_layer_per_token(self.h, _ptr(x), T, d, _ptr(fin),
                                                       _ptr(out)))
        return out.view(np.float16)
