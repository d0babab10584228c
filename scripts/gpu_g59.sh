for e in "X=1" "MOE_NO_FUSED_COMBINE=1"; do for w in c1i4 c3_64; do env $e timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']), {k: round(v*1e3,1) for k,v in j.get('stage_ms',{}).items()})"; done; done
git stash -q 2>/dev/null
