timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 120 python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep plan
timeout 120 python scripts/gate_trace.py 1024 32 1 1 2>&1 | grep plan
for e in "X=1" "MOE_PLAN_NO_STAGE=1"; do for w in c2 c3_1; do env $e timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']))"; done; done
