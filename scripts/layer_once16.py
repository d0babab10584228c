"""Dev probe: a few device-resident layer forwards at one config (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
d, f, E, T, k = [int(v) for v in sys.argv[1:6]]
n = int(sys.argv[6]) if len(sys.argv) > 6 else 3
lw = random_layer(d, f, E, seed=1)
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=16)
x = torch.randn(T, d, device="cuda").half()
L.reserve(T, k)
for _ in range(n):
    L.forward(x, None, k=k, mode=1)
torch.cuda.synchronize()
