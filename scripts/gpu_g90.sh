timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python scripts/stress_layer.py 512 2048 8 4096 2 4 60 2>&1 | grep -E "iter|ok" | head -2
for e in "X=1" "MOE_FUSED_COMBINE=0"; do for w in c2 c5; do env $e timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), {k: round(v*1e3,1) for k,v in j.get('stage_ms',{}).items()})"; done; done
