set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x -k "gate or routing or layer_fast or decode_shapes or pair" 2>&1 | tail -2
for w in c2 c4; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-260; MOE_TC_NS12=1 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-260; done
for cfg in "512 8 4096 2" "1024 32 1 1"; do python scripts/gate_trace.py $cfg 2>&1 | grep ln_gate; done
bash scripts/ncu_traffic.sh
