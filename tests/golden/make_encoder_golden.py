"""Generate encoder_forward fixtures from the UNMODIFIED reference engine
(oracle/_ref/libmoeref.so: load_model + encoder_forward, model.cpp:351-398)
over the committed checkpoints model_int4.moec / model_f16.moec.  Run here,
where /root/reference exists:

    make oracle && python tests/golden/make_encoder_golden.py

Writes tests/golden/encoder_vectors.npz (per case: tokens, reference out)."""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import REF_SO  # noqa: E402

CASES = [(3, 8), (5, 5), (1, 1), (4, 7)]  # (batch, len); max_seq_len = 8, vocab = 16


def main():
    lib = C.CDLL(REF_SO)
    lib.ref_last_error.restype = C.c_char_p
    out = {}
    for name in ("model_int4", "model_f16"):
        path = os.path.join(HERE, name + ".moec")
        for i, (batch, length) in enumerate(CASES):
            rng = np.random.default_rng(500 + 10 * i + len(name))
            tok = rng.integers(0, 16, size=(batch, length)).astype(np.int32)
            y = np.zeros((batch * length, 64), np.uint16)
            st = lib.ref_encoder_forward(path.encode(), tok.ctypes.data_as(C.c_void_p),
                                         C.c_size_t(batch), C.c_size_t(length),
                                         y.ctypes.data_as(C.c_void_p))
            if st != 0:
                raise SystemExit(lib.ref_last_error().decode())
            out[f"{name}_{i}_tok"], out[f"{name}_{i}_out"] = tok, y
    np.savez_compressed(os.path.join(HERE, "encoder_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
