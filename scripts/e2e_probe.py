"""Dev probe: pinned-host layer forward (moe_layer_forward_host) time per
step at one config; run under MOE_HOST_CHUNKS=c to force the chunk count.
Args: d f E T k"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
d, f, E, T, k = [int(v) for v in sys.argv[1:6]]
lw = random_layer(d, 64, E, seed=1)
g = torch.Generator(device="cuda"); g.manual_seed(1)
w1 = (torch.randn((E, d, f), generator=g, device="cuda") / d ** 0.5).half()
w2 = (torch.randn((E, f, d), generator=g, device="cuda") / f ** 0.5).half()
b1 = np.zeros((E, f), np.float16); b2 = np.zeros((E, d), np.float16)
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, w1, b1, w2, b2, bits=4)
xt = torch.randn((T, d)).half().pin_memory(); ot = torch.empty_like(xt).pin_memory()
xh = xt.view(torch.int16).numpy().view(np.float16); oh = ot.view(torch.int16).numpy().view(np.float16)
for _ in range(5): L.forward_host(xh, None, k=k, mode=1, out_host=oh)
torch.cuda.synchronize()
n = 50
t0 = time.perf_counter()
for _ in range(n): L.forward_host(xh, None, k=k, mode=1, out_host=oh)
dt = (time.perf_counter() - t0) / n
xd = torch.randn((T, d), device="cuda").half()
for _ in range(5): L.forward(xd, None, k=k, mode=1, graph=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(n): L.forward(xd, None, k=k, mode=1, graph=True)
torch.cuda.synchronize()
dd = (time.perf_counter() - t1) / n
print(f"chunks={os.environ.get('MOE_HOST_CHUNKS','auto')} d={d} f={f} E={E} T={T} k={k}: host path {dt*1e6:.1f} us/step "
      f"({T/dt/1e6:.2f} M tok/s), device graph {dd*1e6:.1f} us/step")
