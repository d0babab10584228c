"""Generate the .moec loader fixtures from the UNMODIFIED reference engine
(oracle/_ref/libmoeref.so: random_model -> quantize_model -> save_model, and
moe_ffn_forward of every MoE block of load_model).  Run here, where
/root/reference exists:

    make oracle && python tests/golden/make_moec_golden.py

Writes tests/golden/model_int4.moec, model_f16.moec and moec_vectors.npz
(per block: input rows, finished flags, reference outputs)."""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import REF_SO  # noqa: E402

# d_model, d_ffn, n_enc, n_dec, n_experts, n_heads, vocab, moe_every, max_seq_len
CFG = [64, 128, 2, 2, 4, 4, 16, 2, 8]


def main():
    lib = C.CDLL(REF_SO)
    lib.ref_last_error.restype = C.c_char_p
    out = {"cfg": np.array(CFG, np.uint32)}
    cfg = (C.c_uint32 * 9)(*CFG)
    for bits, name in ((4, "model_int4.moec"), (16, "model_f16.moec")):
        path = os.path.join(HERE, name)
        if lib.ref_make_moec(path.encode(), cfg, bits, C.c_uint64(77)) != 0:
            raise SystemExit(lib.ref_last_error().decode())
        n_blocks = CFG[2] // CFG[7] + CFG[3] // CFG[7]
        for b in range(n_blocks):
            rng = np.random.default_rng(1000 * bits + b)
            T = 13
            x = rng.standard_normal((T, CFG[0])).astype(np.float16).view(np.uint16)
            fin = (rng.random(T) < 0.25).astype(np.uint8)
            y = np.zeros_like(x)
            st = lib.ref_moec_block_forward(path.encode(), b, x.ctypes.data_as(C.c_void_p),
                                            C.c_size_t(T), fin.ctypes.data_as(C.c_void_p),
                                            y.ctypes.data_as(C.c_void_p))
            if st != 0:
                raise SystemExit(lib.ref_last_error().decode())
            out[f"b{bits}_{b}_x"], out[f"b{bits}_{b}_fin"], out[f"b{bits}_{b}_out"] = x, fin, y
    np.savez_compressed(os.path.join(HERE, "moec_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
