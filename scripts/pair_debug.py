"""Dev probe: the decode FFN pair (one launch) vs two launches on one case;
prints per-expert row counts and which expert groups differ."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
bits, T, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
out = sys.argv[4]
d, f, E = 256, 1024, 32
seed = 900 + T + bits + (int(sys.argv[5]) if len(sys.argv) > 5 else 0)
lw = random_layer(d, f, E, seed=seed)
rng = np.random.default_rng(seed + 1)
x = rng.standard_normal((T, d)).astype(np.float16)
fin = (rng.random(T) < 0.1).astype(np.uint8)
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits)
xd = torch.from_numpy(x).cuda(); fd = torch.from_numpy(fin).cuda()
y = L.forward(xd, fd, k=k, mode=1).cpu().numpy()
r = L.routing(T, k)
np.savez(out, y=y, offsets=r["offsets"], perm=r["perm"], inv=r["inv"])
print("offsets", r["offsets"].tolist())
