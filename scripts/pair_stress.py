"""Dev probe: repeated decode-layer forwards (pair GEMV kernel by default);
saves the first output per case, reports run-to-run mismatches.  Args:
out.npz [compare.npz]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
res = {}
ref = np.load(sys.argv[2]) if len(sys.argv) > 2 else None
bad = 0
for bits in (16, 8, 4):
    for T, k in ((37, 2), (64, 1), (200, 1), (1, 1), (8, 2)):
        seed = 900 + T + bits
        lw = random_layer(256, 1024, 32, seed=seed)
        rng = np.random.default_rng(seed + 1)
        x = rng.standard_normal((T, 256)).astype(np.float16)
        fin = (rng.random(T) < 0.1).astype(np.uint8)
        L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits)
        xd = torch.from_numpy(x).cuda(); fd = torch.from_numpy(fin).cuda()
        first = L.forward(xd, fd, k=k, mode=1).cpu().numpy().view(np.uint16)
        key = f"b{bits}_T{T}_k{k}"
        res[key] = first
        n = 0
        for _ in range(30):
            y = L.forward(xd, fd, k=k, mode=1).cpu().numpy().view(np.uint16)
            n += int((y != first).any())
        msg = f"{key}: {n}/30 repeats differ"
        if ref is not None:
            msg += f"; vs ref {'same' if (ref[key] == first).all() else 'DIFF'}"
        if n: bad += 1
        print(msg, flush=True)
np.savez(sys.argv[1], **res)
print("bad cases", bad)
