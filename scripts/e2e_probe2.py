"""Dev probe: per-call wall time distribution of the pinned-host layer
forward (moe_layer_forward_host) at C2; run under MOE_HOST_CHUNKS /
MOE_HOST_GRAPH."""
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
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, w1, np.zeros((E, f), np.float16), w2, np.zeros((E, d), np.float16), bits=4)
from paper_2211_10017_b200.ops import HostBuffer
xb, ob = HostBuffer((T, d), np.float16, write_combined=True), HostBuffer((T, d), np.float16)
xh, oh = xb.array, ob.array
xh[...] = np.random.default_rng(0).standard_normal((T, d)).astype(np.float16)
xt = torch.from_numpy(xh.view(np.int16)).view(torch.float16)
ot = torch.from_numpy(oh.view(np.int16)).view(torch.float16)
for _ in range(10): L.forward_host(xh, None, k=k, mode=1, out_host=oh)
ts = []
for _ in range(200):
    t0 = time.perf_counter(); L.forward_host(xh, None, k=k, mode=1, out_host=oh); ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e6
# raw copy bandwidth for reference
xd = torch.empty((T, d), device="cuda").half()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50): xd.copy_(xt, non_blocking=True)
torch.cuda.synchronize(); h2d = (time.perf_counter() - t0) / 50
t0 = time.perf_counter()
for _ in range(50): ot.copy_(xd, non_blocking=True)
torch.cuda.synchronize(); d2h = (time.perf_counter() - t0) / 50
print(f"chunks={os.environ.get('MOE_HOST_CHUNKS','auto')} graph={os.environ.get('MOE_HOST_GRAPH','1')}: "
      f"min {ts.min():.0f} p50 {np.median(ts):.0f} p90 {np.percentile(ts,90):.0f} us; "
      f"H2D {T*d*2/h2d/1e9:.1f} GB/s D2H {T*d*2/d2h/1e9:.1f} GB/s")
