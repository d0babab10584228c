set -x
timeout 900 python -m pytest tests/test_gpu_layer.py -q -x -k "routing_exact or fused" 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity_configs.py -q -x 2>&1 | tail -4
for w in c4 c5 c4_stack; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 2>/dev/null | tail -1
  MOE_GATE_NO_TILE=1 timeout 600 python bench.py --workload $w --steps 20 --warmup 3 2>/dev/null | tail -1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_t19_c4_launches.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_t19_c5_launches.csv python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
