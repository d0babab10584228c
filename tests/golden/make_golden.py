"""Generate tests/golden/*.npz from the UNMODIFIED reference engine
(oracle/_ref/libmoeref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run here (where /root/reference exists):

    make oracle && python tests/golden/make_golden.py

Inputs are regenerated from seeds by ``oracle.oracle.random_layer`` (numpy
PCG64, stable across machines) and stored too, so the fixtures are
self-contained.  The GPU box has no /root/reference: tests read only these
files there.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference, random_layer  # noqa: E402


def u16(a):
    return np.ascontiguousarray(a).view(np.uint16)


def main():
    ref = Reference()
    out = {}
    # quantizer KAT tensor (quantize.cpp:74-122)
    rng = np.random.default_rng(2211)
    w = (rng.standard_normal((2, 32, 64)) * 0.3).astype(np.float16)
    w[1, :, 5] = 0
    out["quant_w"] = u16(w)
    for bits in (4, 8):
        p, s = ref.quantize(w, bits)
        out[f"quant{bits}_packed"], out[f"quant{bits}_scales"] = p, u16(s)
        out[f"quant{bits}_deq"] = u16(ref.dequantize(p, s, w.shape, bits, fast=True))
    # small layers, every precision (model.cpp:299-349), 25% finished rows
    for bits in (16, 8, 4):
        d, f, E, T = 64, 128, 8, 40
        lw = random_layer(d, f, E, seed=5000 + bits)
        x = np.random.default_rng(bits).standard_normal((T, d)).astype(np.float16)
        fin = (np.random.default_rng(bits + 1).random(T) < 0.25).astype(np.uint8)
        R = ref.layer(lw, bits)
        out[f"small{bits}_x"], out[f"small{bits}_fin"] = u16(x), fin
        out[f"small{bits}_out"] = u16(R.forward(x, fin))
        xn = ref.layer_norm(x, lw.ln_g, lw.ln_b)
        lg = ref.gate_logits(xn, lw.gw, lw.gb)
        ex, sc = ref.gate_top1(lg)
        perm, inv, offs, act = ref.build_plan(ex, fin, E)
        out[f"small{bits}_logits"] = lg
        out[f"small{bits}_expert"], out[f"small{bits}_scale"] = ex, sc
        out[f"small{bits}_perm"], out[f"small{bits}_inv"] = perm, inv
        out[f"small{bits}_offsets"] = offs
        out[f"small{bits}_active"] = np.array([act], np.uint32)
        if bits != 16:
            q1, s1, q2, s2 = R.export_quant()
            out[f"small{bits}_q1"], out[f"small{bits}_s1"] = q1, u16(s1)
            out[f"small{bits}_q2"], out[f"small{bits}_s2"] = q2, u16(s2)
    # BASELINE config 1 (E=8, d=512, f=2048, T=256, top-1), FP16 and int4 experts
    lw = random_layer(512, 2048, 8, seed=1)
    x = np.random.default_rng(2).standard_normal((256, 512)).astype(np.float16)
    out["c1_x"] = u16(x)
    for bits in (16, 4):
        R = ref.layer(lw, bits, threads=os.cpu_count() or 1)
        out[f"c1_{bits}_out"] = u16(R.forward(x, None, threads=os.cpu_count() or 1))
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
