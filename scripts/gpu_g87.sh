timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu -k "gemv or decode or layer" 2>&1 | tail -1
for w in c3_1 c3_8 c3_64 c1i4; do timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done
