set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "gemm_fast or cta_pair" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for P in 1 0; do for w in c2 c4 c5; do MOE_TC_PAIR=$P timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('PAIR=$P', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'gemm_us=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']), 'frac=%.3f'%j['roofline']['frac'], j.get('stage_ms'))"; done; done
