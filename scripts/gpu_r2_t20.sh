set -x
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py -q -x -k "decode" 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity_configs.py -q -x -k "c3" 2>&1 | tail -4
for w in c3_1 c3_8 c3_64; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w pair', j['ms_per_step']*1000, j.get('stage_ms'), j['roofline']['frac'])"
  MOE_GEMV_PAIR=0 timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w two', j['ms_per_step']*1000, j.get('stage_ms'), j['roofline']['frac'])"
done
timeout 600 python bench.py --workload decode_prune --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1
MOE_GEMV_PAIR=0 timeout 600 python bench.py --workload decode_prune --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1
ncu --set full --clock-control none --import-source on -k regex:gate_tile -c 1 -o gpurun_out/r2_gate_tile_c4 python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_pair -c 1 -s 8 -o gpurun_out/r2_gemv_pair_c3_64 python bench.py --workload c3_64 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
