timeout 600 python -m pytest tests/test_gpu_layer.py -q -m gpu -k "repeat or fast or c2_c3" 2>&1 | tail -1
for e in "MOE_PDL=0" "MOE_PDL=3" "MOE_PDL=0" "MOE_PDL=3"; do for w in c2 c4; do env $e timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done; done
