"""Dev probe: expert-sorted FFN2 rows (layer workspace y) of the decode
pair kernel, first and second forward, for one case.  Args: bits T k out.npz"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle.oracle import random_layer
from paper_2211_10017_b200 import abi
from paper_2211_10017_b200.ops import MoELayer
bits, T, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
d, f, E = 256, 1024, 32
seed = 900 + T + bits
lw = random_layer(d, f, E, seed=seed)
rng = np.random.default_rng(seed + 1)
x = rng.standard_normal((T, d)).astype(np.float16)
fin = (rng.random(T) < 0.1).astype(np.uint8)
L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=bits)
xd = torch.from_numpy(x).cuda(); fd = torch.from_numpy(fin).cuda()
ys = []
outs = []
for it in range(3):
    outs.append(L.forward(xd, fd, k=k, mode=1).cpu().numpy().view(np.uint16))
    torch.cuda.synchronize()
    _, yp = L.buffers()
    a = np.empty((T * k, d), np.uint16)
    abi.call("moe_cuda_memcpy", C.c_void_p(a.ctypes.data), C.c_void_p(yp), a.nbytes, 1, None)
    ys.append(a)
r = L.routing(T, k)
np.savez(sys.argv[4], y0=ys[0], y1=ys[1], y2=ys[2], o0=outs[0], o1=outs[1], o2=outs[2], offsets=r["offsets"], inv=r["inv"], scale=r["scale"])
