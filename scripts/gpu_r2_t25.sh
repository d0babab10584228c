python scripts/pair_debug2.py 16 37 2 gpurun_out/d2_pair.npz
MOE_GEMV_PAIR=0 python scripts/pair_debug2.py 16 37 2 gpurun_out/d2_two.npz
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/d2_pair.npz'); b=np.load('gpurun_out/d2_two.npz')
off=a['offsets']; print('offsets', off.tolist())
live=int(off[-1])
for name in ('y0','y1','y2'):
    ya=a[name][:live].view(np.float16).astype(np.float32); yb=b['y0'][:live].view(np.float16).astype(np.float32)
    bad=np.nonzero(np.abs(ya-yb).max(1)>1e-3)[0]
    ex=[int(np.searchsorted(off, r, side='right')-1) for r in bad]
    print(name, 'bad rows', bad.tolist(), 'experts', ex)
    if len(bad):
        r=bad[0]; cols=np.nonzero(np.abs(ya[r]-yb[r])>1e-3)[0]; print('  row',r,'bad cols',cols.tolist()[:40], len(cols))
print('two-launch y0==y1', (b['y0']==b['y1']).all())
for n in ('o0','o1','o2'):
    oa=a[n].view(np.float16).astype(np.float32); ob=b['o0'].view(np.float16).astype(np.float32)
    bad=np.nonzero(np.abs(oa-ob).max(1)>1e-3)[0]
    print(n,'bad out rows',bad.tolist())
print('inv same',(a['inv']==b['inv']).all(),'scale same',(a['scale']==b['scale']).all())
PY
