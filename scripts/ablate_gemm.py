"""Dev probe: time the tcgen05 grouped GEMM at C2 FFN shapes under the
MOE_TC_DBG ablation bits (1 no epilogue, 2 no TMEM A stores, 4 no W loads)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2211_10017_b200 import ops
E, rows = 8, 8192
offs = np.concatenate([[0], np.cumsum(np.full(E, rows // E))]).astype(np.int32)
probs = torch.tensor(np.stack([np.arange(E), offs[:-1], offs[1:]], 1).astype(np.int32), device="cuda")
for (m, n) in ((512, 2048), (2048, 512)):
    w = torch.randn(E, m, n, device="cuda").half() * 0.05
    q, s = ops.quantize(w, 4)
    tiled = ops.tile_weights(q, E, m, n, 4)
    x = torch.randn(rows, m, device="cuda").half()
    bias = torch.zeros(E, n, device="cuda").half()
    for dbg in [0, 1, 2, 4, 3, 7]:
        os.environ["MOE_TC_DBG"] = str(dbg)
        for i in range(3):
            ops.grouped_gemm(x, probs, tiled, s, 4, E, n, bias, True, 1)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); st.record()
        for i in range(10):
            ops.grouped_gemm(x, probs, tiled, s, 4, E, n, bias, True, 1)
        en.record(); torch.cuda.synchronize()
        ms = st.elapsed_time(en) / 10
        print(f"m={m} n={n} dbg={dbg}: {ms*1e3:.1f} us  {2*rows*m*n/ms/1e9:.1f} TFLOP/s", flush=True)
