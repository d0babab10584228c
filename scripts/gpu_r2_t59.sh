timeout 300 python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep "plan_place_fused" | tail -1
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py tests/test_gpu_parity_configs.py -q -x -k "routing or plan or c2 or layer_exact or decode" 2>&1 | tail -2
for w in c2 c3_64 c1i4; do timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w', round(j['ms_per_step']*1000,2), s.get('routing_plan'))"; done
