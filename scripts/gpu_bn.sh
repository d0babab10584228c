for bn in 0 192 256; do
  for w in c2 c4; do MOE_TC_BN=$bn python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('BN=$bn', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'gemm_us=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']), 'frac=%.3f'%j['roofline']['frac'])"; done
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
