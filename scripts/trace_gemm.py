"""Dev probe: run the tcgen05 grouped GEMM at the C2 FFN shapes with
MOE_TC_TRACE set (CTA 0 role timestamps appended to the given file)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tc_trace.bin"
from paper_2211_10017_b200 import ops
E, rows = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (8, 8192)
shapes = ((int(sys.argv[4]), int(sys.argv[5])), (int(sys.argv[5]), int(sys.argv[4]))) if len(sys.argv) > 5 else ((512, 2048), (2048, 512))
rng = np.random.default_rng(0)
counts = np.full(E, rows // E)
offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
probs = torch.tensor(np.stack([np.arange(E), offs[:-1], offs[1:]], 1).astype(np.int32), device="cuda")
for (m, n) in shapes:
    w = torch.randn(E, m, n, device="cuda").half() * 0.05
    q, s = ops.quantize(w, 4)
    tiled = ops.tile_weights(q, E, m, n, 4)
    x = torch.randn(rows, m, device="cuda").half()
    bias = torch.zeros(E, n, device="cuda").half()
    for i in range(3):
        ops.grouped_gemm(x, probs, tiled, s, 4, E, n, bias, True, 1)
    torch.cuda.synchronize()
    os.environ["MOE_TC_TRACE"] = out
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    ops.grouped_gemm(x, probs, tiled, s, 4, E, n, bias, True, 1)
    en.record(); torch.cuda.synchronize()
    del os.environ["MOE_TC_TRACE"]
    st.record()
    for i in range(10):
        ops.grouped_gemm(x, probs, tiled, s, 4, E, n, bias, True, 1)
    en.record(); torch.cuda.synchronize()
    ms = st.elapsed_time(en) / 10
    print(f"m={m} n={n}: {ms*1e3:.1f} us  {2*rows*m*n/ms/1e9:.1f} TFLOP/s", flush=True)
