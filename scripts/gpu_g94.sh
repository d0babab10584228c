timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py tests/test_gpu_dropin.py -q -m gpu 2>&1 | tail -1
timeout 120 python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep plan
for i in 1 2; do for w in c2 c3_1; do timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']))"; done; done
