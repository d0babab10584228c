for m in 8192 32768; do for w in c4 c5; do
  MOE_PLAN_FUSED_MAX=$m timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w fusedmax=$m', round(j['ms_per_step']*1000,2), s.get('routing_plan'))"
done; done
MOE_PLAN_FUSED_MAX=32768 timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x -k "routing" 2>&1 | tail -3
