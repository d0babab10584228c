timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -2
timeout 300 bash scripts/gpu_tctrace2.sh
for P in 1 0; do for w in c2 c4 c1i4; do MOE_TC_PAIR=$P timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('PAIR=$P', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'gemm_us=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']), 'frac=%.3f'%j['roofline']['frac'])"; done; done
timeout 120 python scripts/gate_trace.py 512 8 4096 2 auto 8,1 4,1 2,1 8,2
timeout 120 python scripts/gate_trace.py 1024 64 16384 1 auto 8,1 4,1
timeout 120 python scripts/gate_trace.py 1024 32 64 1 auto 8,1 1,1 2,1
timeout 120 python scripts/gate_trace.py 1024 32 1 1 auto 8,1 1,1 2,1
