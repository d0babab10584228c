timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
for w in c4 c2 c3_64; do timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), {k: round(v*1e3,1) for k,v in j.get('stage_ms',{}).items()})"; done
