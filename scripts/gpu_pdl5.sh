for e in "MOE_PDL=4" "MOE_PDL=5" "MOE_PDL=4" "MOE_PDL=5"; do for w in c3_1 c3_8 c3_64; do env $e timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:36], 'us=%.1f'%(1e3*j['ms_per_step']))"; done; done
MOE_PDL=5 timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -m gpu -k "gemv or decode or layer" 2>&1 | tail -1
