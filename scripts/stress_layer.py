"""Dev stress: repeated forwards of one layer config; reports the first CUDA
error.  Args: d f E T k bits iters."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import random_layer
from paper_2211_10017_b200.ops import MoELayer
d, f, E, T, k, bits, iters = [int(v) for v in sys.argv[1:8]]
lw = random_layer(d, f, E, seed=E + d + T)
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits)
rng = np.random.default_rng(T)
x = torch.from_numpy(rng.standard_normal((T, d)).astype(np.float16).view(np.int16)).cuda().view(torch.float16)
fin = torch.from_numpy((rng.random(T) < 0.1).astype(np.uint8)).cuda()
ref = None
for i in range(iters):
    try:
        out = L.forward(x, fin, k=k, mode=1)
        torch.cuda.synchronize()
    except Exception as e:
        print(f"iter {i}: {str(e)[:200]}", flush=True)
        sys.exit(1)
    if ref is None:
        ref = out.clone()
    elif not torch.equal(out.view(torch.int16), ref.view(torch.int16)):
        print(f"iter {i}: output differs from iteration 0", flush=True)
print(f"ok {iters} iterations", flush=True)
