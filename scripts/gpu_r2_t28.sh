MOE_GEMV_PAIR=0 python scripts/pair_debug2.py 16 37 2 gpurun_out/d2_two.npz
cmp() {
python - <<PY
import numpy as np
a=np.load('gpurun_out/d2_pair.npz'); b=np.load('gpurun_out/d2_two.npz')
off=a['offsets']; live=int(off[-1])
res=[]
for name in ('y0','y1','y2'):
    ya=a[name][:live].view(np.float16).astype(np.float32); yb=b['y0'][:live].view(np.float16).astype(np.float32)
    bad=np.nonzero(np.abs(ya-yb).max(1)>1e-3)[0]
    res.append(sorted(set(int(np.searchsorted(off, r, side='right')-1) for r in bad)))
print('$1 bad experts per call', res)
PY
}
for dbg in 32 40 34; do for rep in 1 2; do MOE_GEMV_PAIR_DBG=$dbg python scripts/pair_debug2.py 16 37 2 gpurun_out/d2_pair.npz; cmp dbg$dbg; done; done
MOE_GEMV_CTAS=2 python scripts/pair_debug2.py 16 37 2 gpurun_out/d2_pair.npz; cmp ctas2
MOE_GEMV_CTAS=1 python scripts/pair_debug2.py 16 37 2 gpurun_out/d2_pair.npz; cmp ctas1
