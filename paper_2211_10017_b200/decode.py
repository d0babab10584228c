"""Decode with batch pruning: the MoE blocks of
beam-search decoding (proj/src/decode.cpp:104-345) on the device, through
the C-ABI moe_decode_run (csrc/decode.cu).

Rows are batch x beam (row r = sentence r // beam, beam r % beam, fixed for
the whole decode, decode.cpp:5-9).  At every step each MoE block runs
moe_ffn_forward with the finished rows as the routing mask when pruning
(decode.cpp:167-169, 216); a sentence's rows stay finished from the step
its top candidate is EOS (decode.cpp:283-294).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import abi
from .ops import _p, _stream


def finished_schedule(batch: int, beam: int, steps: int, lengths) -> np.ndarray:
    """(steps, batch*beam) uint8: the rows of sentence s are finished from
    step lengths[s] on (its EOS step), as finished_rows evolves in
    decode.cpp (all beams of a sentence finish together)."""
    lengths = np.asarray(lengths, np.int64)
    if lengths.shape != (batch,):
        raise ValueError("decode: one length per sentence")
    fin = np.zeros((steps, batch * beam), np.uint8)
    for s in range(batch):
        fin[lengths[s]:, s * beam:(s + 1) * beam] = 1
    return fin


def decode_run(layers, x_steps, finished_steps=None, k=1, mode=abi.MODE_FAST, prune=True,
               out=None, work=None, stream=None):
    """Run the MoE blocks `layers` (MoELayer list, block l feeds block l+1)
    over every step: x_steps (steps, rows, d) fp16 device, finished_steps
    (steps, rows) uint8 device or None.  Returns out (steps, rows, d): the
    last block's output per step."""
    steps, rows, d = x_steps.shape
    if out is None:
        out = torch.empty_like(x_steps)
    if work is None:
        work = torch.empty((rows, d), dtype=x_steps.dtype, device=x_steps.device)
    arr = (C.c_void_p * len(layers))(*[L._h.value for L in layers])
    abi.call("moe_decode_run", arr, len(layers), _p(x_steps), _p(finished_steps), steps, rows, k,
             mode, int(bool(prune)), _p(out), _p(work), _stream(stream))
    return out
