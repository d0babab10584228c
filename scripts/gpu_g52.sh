for bn in 128 160 192; do MOE_TC_BN=$bn timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "cta_pair or gemm_fast" 2>&1 | tail -1; done
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -1
for bn in 0 128 160 192 224 256; do for w in c2 c4 c1i4; do MOE_TC_BN=$bn timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('BN=$bn', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'gemm=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']), 'frac=%.3f'%j['roofline']['frac'])"; done; done
