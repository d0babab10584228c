"""Dev probe: MOE_GEMV_TRACE phase times of the decode GEMV (K5) inside a
layer forward.  Args: d f E T k"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
d, f, E, T, k = [int(v) for v in sys.argv[1:6]]
lw = random_layer(d, 64, E, seed=1)
g = torch.Generator(device="cuda"); g.manual_seed(1)
w1 = (torch.randn((E, d, f), generator=g, device="cuda") / d ** 0.5).half()
w2 = (torch.randn((E, f, d), generator=g, device="cuda") / f ** 0.5).half()
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, w1, np.zeros((E, f), np.float16), w2,
             np.zeros((E, d), np.float16), bits=4)
x = torch.randn((T, d), device="cuda").half()
for _ in range(3): L.forward(x, None, k=k, mode=1)
torch.cuda.synchronize()
os.environ["MOE_GEMV_TRACE"] = "1"
L.forward(x, None, k=k, mode=1)
torch.cuda.synchronize()
