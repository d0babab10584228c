timeout 300 python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep -v plan_place | tail -2
timeout 300 python scripts/gate_trace.py 1024 32 64 1 2>&1 | grep -v plan_place | tail -2
MOE_GATE_EPG1=1 timeout 300 python scripts/gate_trace.py 1024 32 64 1 2>&1 | grep -v plan_place | tail -2
MOE_GATE_EPG1=1 timeout 300 python scripts/gate_trace.py 1024 32 1 1 2>&1 | grep -v plan_place | tail -2
for w in c2 c3_1 c3_64; do for e in 0 1; do
  if [ $e = 1 ]; then export MOE_GATE_EPG1=1; else unset MOE_GATE_EPG1; fi
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w epg1=$e', round(j['ms_per_step']*1000,2), s.get('layer_norm'), s.get('routing_plan'))"
done; done
unset MOE_GATE_EPG1
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x -k "routing_exact or gate or layer_norm" 2>&1 | tail -3
