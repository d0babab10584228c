"""Dev probe: a few device-resident layer forwards at one config with
weights generated on the GPU (C4/C5 sizes), for ncu captures.
Args: d f E T k [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import torch
from paper_2211_10017_b200.ops import MoELayer
d, f, E, T, k = [int(v) for v in sys.argv[1:6]]
n = int(sys.argv[6]) if len(sys.argv) > 6 else 3
g = torch.Generator(device="cuda"); g.manual_seed(1)
r = lambda shape, s: (torch.randn(shape, generator=g, device="cuda") * s).half()  # noqa: E731
L = MoELayer((1 + 0.1 * torch.randn(d, generator=g, device="cuda")).half(), r((d,), 0.05),
             r((d, E), 1 / math.sqrt(d)), r((E,), 0.02), r((E, d, f), 1 / math.sqrt(d)), r((E, f), 0.02),
             r((E, f, d), 1 / math.sqrt(f)), r((E, d), 0.02), bits=4)
L.quant = None
torch.cuda.empty_cache()
x = torch.randn(T, d, device="cuda", generator=g).half()
L.reserve(T, k)
for _ in range(n):
    L.forward(x, None, k=k, mode=1)
torch.cuda.synchronize()
