timeout 300 python scripts/gate_trace.py 1024 64 16384 1 2>&1 | grep -v plan_place | tail -3
for r in 8 4; do MOE_GATE_TILE_RPT=$r timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c4 rpt=$r', round(j['ms_per_step']*1000,1), j.get('stage_ms'))"; done
timeout 900 python -m pytest tests/test_gpu_layer.py -q -x -k "routing_exact" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity_configs.py -q -x -k "c4" 2>&1 | tail -3
