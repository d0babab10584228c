"""Summarise MOE_TC_TRACE output (slots of k_gemm_tc.cu TC_TRACE)."""
import sys
import numpy as np
N, SL = 1024, 12
raw = np.fromfile(sys.argv[1], dtype=np.int64)
rec = 4 + SL * N
for r in range(len(raw) // rec):
    bits, bn, stg, nkb = raw[r * rec: r * rec + 4]
    t = raw[r * rec + 4:(r + 1) * rec].reshape(SL, N).astype(np.float64)
    nit = int((t[3] > 0).sum())
    t0 = t[0][0]
    print(f"== bits={bits} BN={bn} NS={stg // 100} NA={stg % 100} nkb={nkb} iters={nit}")
    iss = t[3][:nit] - t0
    rdy = t[2][:nit] - t0
    print(f"  per k-block: {np.diff(iss).mean():.1f} cycles (MMA work {4*bn/2:.0f}); issue section {np.mean(iss-rdy):.1f}")
    gaps = rdy[1:] - iss[:-1]
    print(f"  MMA thread wait before ready: mean={gaps.mean():.1f} p50={np.median(gaps):.0f} max={gaps.max():.0f}")
    dq0, dq1 = t[4][:nit] - t0, t[5][:nit] - t0
    m = (dq0 > -t0 / 2) & (dq1 > -t0 / 2)
    print(f"  dequant (group0 its) dur mean={(dq1 - dq0)[m].mean():.1f}")
    ne = int((t[7] > 0).sum())
    es, ed = t[6][:ne] - t0, t[7][:ne] - t0
    print(f"  epilogue tiles={ne} dur mean={(ed - es).mean():.1f}")
    nc = int((t[11] > 0).sum())
    if nc:
        w, f, e = (t[i][:nc] - t0 for i in (9, 10, 11))
        print(f"  epi chunks={nc}: compute+sts {np.mean(f-w):.0f}  store issue {np.mean(e-f):.0f}  chunk-to-chunk {np.mean(np.diff(w)):.0f}")
    print(f"  total={iss[-1]:.0f} cycles")
# full-vs-afull attribution of the MMA thread's waits
for r in range(len(raw) // rec):
    t = raw[r * rec + 4:(r + 1) * rec].reshape(SL, N).astype(np.float64)
    nit = int((t[3] > 0).sum())
    f, a, i = t[1][:nit], t[2][:nit], t[3][:nit]
    print(f"  [rec {r}] wait on full: {np.mean(f[1:] - i[:-1]):.0f}  then afull: {np.mean(a - f):.0f}")
