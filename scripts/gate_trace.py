"""Dev probe: LN + gate kernel traces (MOE_GATE_TRACE) and route timings per
gate config at one layer shape.  Args: d E T k [cfg ...] (cfg "EPG,RPT")."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
d, E, T, k = [int(v) for v in sys.argv[1:5]]
cfgs = sys.argv[5:] or ["auto"]
lw = random_layer(d, 64, E, seed=1)
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=16)
x = torch.randn(T, d, device="cuda").half()
L.reserve(T, k)
for cfg in cfgs:
    if cfg == "auto":
        os.environ.pop("MOE_GATE_CFG", None)
    else:
        os.environ["MOE_GATE_CFG"] = cfg
    for _ in range(3): L.route(x, None, k)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): L.route(x, None, k)
    e.record(); torch.cuda.synchronize()
    print(f"route d={d} E={E} T={T} k={k} cfg={cfg}: {s.elapsed_time(e)/20*1e3:.1f} us", flush=True)
    os.environ["MOE_GATE_TRACE"] = "1"
    L.route(x, None, k)
    torch.cuda.synchronize()
    del os.environ["MOE_GATE_TRACE"]
