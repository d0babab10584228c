"""ctypes binding of include/moe_cuda.h (libmoe_cuda.so, sm_100a).

This is the Python-side face of the C-ABI: plain pointers (ints), int64
sizes, a cudaStream_t as an int.  It fails loudly when the CUDA library is
missing -- there is no CPU fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmoe_cuda.so")

MOE_OK, MOE_EINVAL, MOE_ECUDA, MOE_ENCCL, MOE_ERANGE, MOE_EIO = 0, 1, 2, 3, 4, 5
MODE_EXACT, MODE_FAST, MODE_GEMV = 0, 1, 2

_vp, _i64, _int, _u16, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_uint16, C.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "moe_cuda_last_error": (C.c_char_p, []),
    "moe_cuda_device_info": (_int, [_vp, _vp, _vp]),
    "moe_cuda_launch_count": (C.c_uint64, []),
    "moe_cuda_malloc": (_int, [_vp, _sz]),
    "moe_cuda_free": (_int, [_vp]),
    "moe_cuda_host_alloc": (_int, [_vp, _sz]),
    "moe_cuda_host_free": (_int, [_vp]),
    "moe_cuda_host_alloc_wc": (_int, [_vp, _sz]),
    "moe_cuda_memcpy": (_int, [_vp, _vp, _sz, _int, _vp]),
    "moe_cuda_memset": (_int, [_vp, _int, _sz, _vp]),
    "moe_cuda_sync": (_int, [_vp]),
    "moe_cuda_debias": (None, [_vp, _vp]),
    "moe_cuda_set_debias": (None, [_u16, _u16]),
    "moe_quantize": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _vp, _vp]),
    "moe_pack_int4": (_int, [_vp, _i64, _vp, _vp]),
    "moe_unpack_int4": (_int, [_vp, _i64, _vp, _vp]),
    "moe_dequantize": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp]),
    "moe_tiled_bytes": (_i64, [_i64, _i64, _i64, _int]),
    "moe_tile_weights": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _vp]),
    "moe_layer_norm": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "moe_gate_logits": (_int, [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp]),
    "moe_gate_topk": (_int, [_vp, _i64, _i64, _int, _vp, _vp, _vp]),
    "moe_routing_plan": (_int, [_vp, _vp, _i64, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "moe_permute_rows": (_int, [_vp, _i64, _vp, _i64, _int, _vp, _vp]),
    "moe_unpermute_scale": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "moe_combine": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _int, _vp, _vp]),
    "moe_grouped_gemm": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _int, _i64, _i64, _vp,
                                _int, _int, _vp, _vp]),
    "moe_layer_create": (_int, [_vp, _vp]),
    "moe_layer_create_device": (_int, [_vp, _vp]),
    "moe_layer_destroy": (_int, [_vp]),
    "moe_layer_reserve": (_int, [_vp, _i64, _int]),
    "moe_layer_forward": (_int, [_vp, _vp, _vp, _i64, _int, _int, _vp, _vp]),
    "moe_layer_forward_host": (_int, [_vp, _vp, _vp, _i64, _int, _int, _vp, _vp]),
    "moe_layer_forward_graph": (_int, [_vp, _vp, _vp, _i64, _int, _int, _vp, _vp]),
    "moe_layer_status": (_int, [_vp, _vp]),
    "moe_layer_routing": (_int, [_vp] + [_vp] * 6),
    "moe_layer_traffic": (_int, [_vp, _vp, _vp]),
    "moe_layer_profile": (_int, [_vp, _int]),
    "moe_layer_profile_read": (_int, [_vp, _vp, _vp]),
    "moe_ep_rank_counts": (_int, [_vp, _i64, _int, _vp, _vp]),
    "moe_layer_route": (_int, [_vp, _vp, _vp, _i64, _int, _vp]),
    "moe_layer_buffers": (_int, [_vp, _vp, _vp]),
    "moe_layer_ffn": (_int, [_vp, _int, _vp]),
    "moe_layer_experts": (_int, [_vp, _vp, _i64, _vp, _i64, _int, _vp, _vp]),
    "moe_layer_combine": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp, _vp]),
    "moe_layer_load_report": (_int, [_vp, C.c_float, _vp, _vp]),
    "moe_ep_unique_id": (_int, [_vp]),
    "moe_ep_create": (_int, [_vp, _int, _int, _vp]),
    "moe_ep_create_loopback": (_int, [_int, _vp]),
    "moe_ep_destroy": (_int, [_vp]),
    "moe_ep_world": (_int, [_vp, _vp, _vp, _vp]),
    "moe_ep_forward": (_int, [_vp, _vp, _vp, _vp, _vp, _int, _int, _vp, _vp]),
    "moe_ep_counts": (_int, [_vp, _int, _vp, _vp, _vp]),
    "moe_ep_segments": (_int, [_int, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "moe_moec_load": (_int, [C.c_char_p, _int, _vp]),
    "moe_moec_info": (_int, [_vp, _vp, _vp, _vp]),
    "moe_moec_block": (_int, [_vp, _int, _vp, _vp, _sz]),
    "moe_moec_destroy": (_int, [_vp]),
    "moe_encoder_forward": (_int, [_vp, _vp, _i64, _i64, _int, _vp, _vp]),
    "moe_moec_write_synthetic": (_int, [C.c_char_p, _vp, _int, C.c_uint64]),
    "moe_decode_run": (_int, [_vp, _int, _vp, _vp, _int, _i64, _int, _int, _int, _vp, _vp, _vp]),
}


class LayerDesc(C.Structure):
    """moe_layer_desc (include/moe_cuda.h)."""

    _fields_ = [("d", _i64), ("f", _i64), ("E", _i64), ("bits", _int)] + [
        (nm, _vp) for nm in ("ln_g", "ln_b", "gate_w", "gate_b", "b1", "b2", "w1", "w2", "q1",
                             "q2", "s1", "s2")] + [("e_begin", _i64), ("e_count", _i64)]


_lib = None


def lib():
    """Load libmoe_cuda.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().moe_cuda_last_error().decode(errors="replace")


def check(status: int):
    if status == MOE_OK:
        return
    msg = last_error()
    if status == MOE_EINVAL:
        raise ValueError(msg)
    if status == MOE_ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().moe_cuda_launch_count())


def device_info():
    sm, ma, mi = C.c_int(), C.c_int(), C.c_int()
    call("moe_cuda_device_info", C.byref(sm), C.byref(ma), C.byref(mi))
    return sm.value, (ma.value, mi.value)
