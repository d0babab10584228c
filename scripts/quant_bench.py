"""Dev probe: K1 quantizer throughput (moe_quantize) at C4 / C5 expert-tensor
shapes; prints GB/s over the algorithmic bytes (2mn read + mn/2 + 2n written
per expert) and the fraction of the measured HBM peak."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2211_10017_b200 import ops
peak = 6550.0
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass
for name, (E, m, n) in {"c4_w1": (64, 1024, 4096), "c4_w2": (64, 4096, 1024),
                        "c5_w1": (128, 2048, 8192), "c2_w1": (8, 512, 2048)}.items():
    for bits in (4, 8):
        w = (torch.randn((E, m, n), device="cuda") * 0.03).half()
        for _ in range(2):
            ops.quantize(w, bits)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            ops.quantize(w, bits)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        nbytes = E * (2 * m * n + (m * n // 2 if bits == 4 else m * n) + 2 * n)
        print(json.dumps({"tensor": name, "bits": bits, "shape": [E, m, n], "ms": ms,
                          "GBps": nbytes / ms / 1e6, "hbm_frac": nbytes / ms / 1e6 / peak}))
        del w
