"""Quick device timing of the MoE layer at a BASELINE config (dev probe)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
d, f, E, T, k = [int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (512, 2048, 8, 4096, 2))]
lw = random_layer(d, f, E, seed=1)
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4)
x = torch.randn(T, d, device="cuda").half()
L.reserve(T, k)
for mode in [int(m) for m in os.environ.get('MODES', '1,0').split(',')]:
    for _ in range(3): L.forward(x, None, k=k, mode=mode)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20 if mode == 1 else 3
    s.record()
    for _ in range(n): L.forward(x, None, k=k, mode=mode)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    print(f"mode={mode} d={d} f={f} E={E} T={T} k={k}: {ms*1e3:.1f} us/layer  {T/ms*1e3/1e6:.2f} Mtok/s", flush=True)
