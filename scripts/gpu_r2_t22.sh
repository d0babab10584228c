set -x
MOE_GEMV_PAIR=0 timeout 900 python -m pytest tests/test_gpu_layer.py -q -k "decode_pair_repeat" 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_layer.py -q -k "decode_pair_repeat" 2>&1 | tail -12
for w in c3_1 c3_8 c3_64; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w pair', j['ms_per_step']*1000, j.get('stage_ms'), j['roofline']['frac'])"
done
for w in c4 c5; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w tile', j['ms_per_step']*1000, j.get('stage_ms'))"
done
ncu --set full --clock-control none --import-source on -k regex:gemv_pair -c 1 -s 8 -o gpurun_out/r2_gemv_pair4_c3_64 python bench.py --workload c3_64 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_tile -c 1 -o gpurun_out/r2_gate_tile2_c4 python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
