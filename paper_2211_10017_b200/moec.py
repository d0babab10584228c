"""`.moec` checkpoint -> device MoE layers, over the C-ABI
moe_moec_* (csrc/moec.cu): the reference's file format
(proj/src/checkpoint.cpp) parsed and validated in C++, every MoE block's
int4 / int8 / fp16 payload uploaded as stored (no host dequantization) and
re-tiled on the device."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .ops import MoELayer

CONFIG_KEYS = ("d_model", "d_ffn", "n_enc_layers", "n_dec_layers", "n_experts", "n_heads",
               "vocab_size", "moe_every", "max_seq_len")
PRECISION = {0: "f16", 1: "int8", 2: "int4"}


class _BlockLayer(MoELayer):
    """A MoE block owned by its MoecModel (not destroyed on its own)."""

    def __init__(self, handle, owner, d, f, E, bits):
        self._owner = owner  # keeps the checkpoint (which owns the layer) alive
        self.d, self.f, self.E, self.bits = d, f, E, bits
        self.e_begin, self.e_count = 0, E
        self.quant = (None, None, None, None)
        self._h = handle

    def __del__(self):  # the MoecModel frees its layers
        self._h = None


class MoecModel:
    """load_model's MoE side: `blocks` = [(name, layer)] in file order."""

    def __init__(self, path: str, create_layers: bool = True):
        h = C.c_void_p()
        abi.call("moe_moec_load", str(path).encode(), int(create_layers), C.byref(h))
        self._h = h
        cfg = (C.c_uint32 * 9)()
        prec, n = C.c_int(), C.c_int()
        abi.call("moe_moec_info", h, cfg, C.byref(prec), C.byref(n))
        self.config = dict(zip(CONFIG_KEYS, [int(v) for v in cfg]))
        self.precision = PRECISION[prec.value]
        bits = {"f16": 16, "int8": 8, "int4": 4}[self.precision]
        self.blocks = []
        for i in range(n.value):
            L, name = C.c_void_p(), C.create_string_buffer(64)
            abi.call("moe_moec_block", h, i, C.byref(L), name, 64)
            layer = None
            if L.value:
                c = self.config
                layer = _BlockLayer(L, self, c["d_model"], c["d_ffn"], c["n_experts"], bits)
            self.blocks.append((name.value.decode(), layer))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                abi.lib().moe_moec_destroy(h)
            except Exception:
                pass
            self._h = None

    def encoder_forward(self, tokens, mode: int = 1, stream=None):
        """encoder_forward (proj/src/model.cpp:351-398) on the device:
        tokens int32 [batch, len] (host) -> fp16 (batch * len, d_model)
        torch tensor on the current device.  mode 0 EXACT (bit-identical to
        the reference), 1 FAST."""
        import torch
        from .ops import _stream
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        if tok.ndim != 2:
            raise ValueError("encoder: tokens must be [batch, len]")
        batch, length = tok.shape
        out = torch.empty((batch * length, self.config["d_model"]), dtype=torch.float16,
                          device="cuda")
        abi.call("moe_encoder_forward", self._h, C.c_void_p(tok.ctypes.data), batch, length, mode,
                 C.c_void_p(out.data_ptr()), _stream(stream))
        return out
