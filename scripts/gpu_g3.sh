timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_dropin.py tests/test_gpu_ep.py -x -q -m gpu 2>&1 | tail -3
for O in 0 1; do for w in c2 c4 c3_1 c3_64; do if [ $O = 1 ]; then export MOE_GATE_OLD=1; else unset MOE_GATE_OLD; fi; timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('OLD=$O', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), {k: round(v*1e3,1) for k,v in j.get('stage_ms',{}).items()})"; done; done
unset MOE_GATE_OLD
timeout 120 python scripts/gate_trace.py 512 8 4096 2
timeout 120 python scripts/gate_trace.py 1024 64 16384 1
timeout 120 python scripts/gate_trace.py 1024 32 64 1
timeout 120 python scripts/gate_trace.py 1024 32 1 1
timeout 120 python scripts/gate_trace.py 2048 128 4096 2
