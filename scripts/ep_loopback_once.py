"""Dev probe: one EP forward (loopback, G=4) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ep import LoopbackEP, owner_range
from paper_2211_10017_b200.ops import MoELayer
lw = random_layer(128, 256, 8, seed=1)
G = 4
layers = []
for g in range(G):
    e0, el = owner_range(8, G, g)
    sl = slice(e0, e0 + el)
    layers.append(MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1[sl], lw.b1[sl], lw.w2[sl], lw.b2[sl],
                           bits=4, expert_range=(e0, el)))
ep = LoopbackEP(layers)
xs = [torch.randn(300, 128, device="cuda").half() for _ in range(G)]
for mode in (0, 1):
    ep.forward(xs, None, k=2, mode=mode)
torch.cuda.synchronize()
print("ok")
