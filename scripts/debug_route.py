import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import Oracle, random_layer
from paper_2211_10017_b200.ops import MoELayer
from paper_2211_10017_b200.ep import _dev_view
o = Oracle()
for (d, E, T, k) in [(512, 8, 256, 1), (64, 8, 40, 1), (512, 8, 4096, 2), (1024, 32, 64, 1)]:
    lw = random_layer(d, 64, E, seed=1)
    x = np.random.default_rng(2).standard_normal((T, d)).astype(np.float16)
    L = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=16)
    xt = torch.from_numpy(x.view(np.int16)).cuda().view(torch.float16)
    L.route(xt, None, k)
    torch.cuda.synchronize()
    r = L.routing(T, k)
    xp = _dev_view(L.buffers()[0], T * k, d).cpu().view(torch.int16).numpy().view(np.float16)
    xn = o.layer_norm(x, lw.ln_g, lw.ln_b)
    want_xp = xn[r["perm"] // k]
    lg = o.gate_logits(xn, lw.gw, lw.gb)
    ex, sc = o.gate_topk(lg, k)
    bad = np.nonzero((xp.view(np.uint16) != want_xp.view(np.uint16)).any(1))[0]
    print(d, E, T, k, "xn rows wrong:", len(bad), "experts ok:", np.array_equal(r["expert"], ex), "scales ok:", np.array_equal(r["scale"], sc))
    if len(bad):
        i = bad[0]; c = np.nonzero(xp[i].view(np.uint16) != want_xp[i].view(np.uint16))[0]
        print("  row", i, "cols", c[:8], xp[i][c[:4]], want_xp[i][c[:4]])
