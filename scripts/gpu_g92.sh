for bn in 128 160 192 224 128 192; do MOE_TC_BNM=$bn timeout 300 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('BNM=$bn', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done
for bn in 128 160 192 224; do MOE_TC_BNM=$bn timeout 300 python bench.py --workload c4 --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('BNM=$bn', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done
