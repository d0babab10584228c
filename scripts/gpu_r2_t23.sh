set -x
python scripts/pair_debug.py 16 37 2 gpurun_out/pd_pair.npz
MOE_GEMV_PAIR=0 python scripts/pair_debug.py 16 37 2 gpurun_out/pd_two.npz
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/pd_pair.npz'); b=np.load('gpurun_out/pd_two.npz')
ya=a['y'].astype(np.float32); yb=b['y'].astype(np.float32)
diff=np.abs(ya-yb).max(axis=1)
print('rows differing', np.nonzero(diff>1e-2)[0].tolist())
print('max diff per row', np.round(diff,3).tolist())
off=a['offsets']; inv=a['inv'].reshape(ya.shape[0],-1); perm=a['perm']
for t in np.nonzero(diff>1e-2)[0]:
    slots=inv[t]; ex=[int(np.searchsorted(off, s, side='right')-1) for s in slots]
    print('token',t,'slots',slots.tolist(),'experts',ex)
PY
for i in 1 2 3; do python scripts/pair_debug.py 16 37 2 gpurun_out/pd_pair$i.npz > /dev/null; done
python -c "
import numpy as np
ys=[np.load('gpurun_out/pd_pair%d.npz'%i)['y'] for i in (1,2,3)]
print('pair runs identical', all((ys[0].view(np.uint16)==y.view(np.uint16)).all() for y in ys))"
for b in 4 8 16; do for s in 0 1 2; do
python scripts/pair_debug.py $b 37 2 gpurun_out/pa.npz $s > /dev/null 2>&1
MOE_GEMV_PAIR=0 python scripts/pair_debug.py $b 37 2 gpurun_out/pb.npz $s > /dev/null 2>&1
python -c "
import numpy as np
a=np.load('gpurun_out/pa.npz')['y'].astype(np.float32); b=np.load('gpurun_out/pb.npz')['y'].astype(np.float32)
print('bits $b seed $s maxdiff', float(np.abs(a-b).max()), 'rows', np.nonzero(np.abs(a-b).max(1)>1e-2)[0].tolist())"
done; done
