for e in "MOE_PDL=3" "MOE_PDL=4" "MOE_PDL=3" "MOE_PDL=4"; do for w in c2 c3_1; do env $e timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']))"; done; done
MOE_PDL=4 timeout 600 python -m pytest tests/test_gpu_layer.py -q -m gpu 2>&1 | tail -1
