timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu 2>&1 | tail -1
timeout 120 python scripts/gate_trace.py 1024 64 16384 1 2>&1 | grep ln_gate
timeout 120 python scripts/gate_trace.py 1024 32 1 1 2>&1 | grep ln_gate
for w in c4 c3_1 c2; do timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']))"; done
