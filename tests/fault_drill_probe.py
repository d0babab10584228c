"""Run under MOE_FAULT_INJECT (read once per process, proj/src/dequant.cpp:
12-30): prints JSON saying whether the GPU dequant, the EXACT layer and the
FAST layer still match the (un-faulted) oracle.  Driven by
tests/test_gpu_fault_drill.py in a subprocess."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import bits16, layer_err, to_dev, to_np  # noqa: E402
from oracle.oracle import Oracle, random_layer  # noqa: E402
from paper_2211_10017_b200 import ops  # noqa: E402


def main(bits):
    import ctypes as C
    from paper_2211_10017_b200 import abi
    # the CUDA library reads MOE_FAULT_INJECT once (first use, here); the
    # oracle reads it on every call -- unset it so the oracle is the healthy
    # expectation the faulted GPU run is checked against
    u8, u4 = C.c_uint16(), C.c_uint16()
    abi.lib().moe_cuda_debias(C.byref(u8), C.byref(u4))
    os.environ.pop("MOE_FAULT_INJECT", None)
    orc = Oracle()
    res = {"debias_u8": hex(u8.value), "debias_u4": hex(u4.value)}
    rng = np.random.default_rng(1)
    w = rng.uniform(-2, 2, (2, 64, 64)).astype(np.float16)
    p, s = orc.quantize(w, bits)
    got = to_np(ops.dequantize(to_dev(p), to_dev(s), (2, 64, 64), bits, True))
    want = orc.dequantize(p, s, (2, 64, 64), bits, True)
    res["dequant_equal"] = bool(np.array_equal(bits16(got), bits16(want)))
    lw = random_layer(128, 256, 8, seed=3)
    x = rng.standard_normal((300, 128)).astype(np.float16)
    L = ops.MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits)
    q = tuple(to_np(t) for t in L.quant)
    want = orc.moe_forward(lw, x, None, k=2, bits=bits, q=q)
    ex = to_np(L.forward(to_dev(x), None, k=2, mode=0))
    fa = to_np(L.forward(to_dev(x), None, k=2, mode=1))
    res["exact_equal"] = bool(np.array_equal(bits16(ex), bits16(want)))
    res["fast_err"] = layer_err(fa, want, x)
    print(json.dumps(res))


if __name__ == "__main__":
    main(int(sys.argv[1]))
