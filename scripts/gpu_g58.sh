timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in c3_1 c3_8 c3_64 c4 c1i4 c2; do timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']), 'frac=%.3f'%j['roofline']['frac'], {k: round(v*1e3,1) for k,v in j.get('stage_ms',{}).items()})"; done
