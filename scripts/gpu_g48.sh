timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python scripts/gate_trace.py 512 8 4096 2
timeout 120 python scripts/gate_trace.py 1024 32 1 1
timeout 120 python scripts/gate_trace.py 1024 64 16384 1
for w in c2 c4 c3_1 c3_64 c1i4; do timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'gemm=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']), {k: round(v*1e3,1) for k,v in j.get('stage_ms',{}).items()})"; done
