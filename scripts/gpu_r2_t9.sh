set -x
./scripts/ffma2_bench 2>&1 | tail -12
./scripts/chain_bench 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x -k "gate or routing or layer_fast or decode_shapes" 2>&1 | tail -2
for cfg in "512 8 4096 2" "1024 32 1 1" "1024 64 16384 1"; do python scripts/gate_trace.py $cfg 2>&1 | grep ln_gate; MOE_GATE_LN_WIDE=1 python scripts/gate_trace.py $cfg 2>&1 | grep ln_gate; done
for w in c2 c3_1 c3_64 c4; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-280; done
bash scripts/sanitize.sh 2>&1 | tail -25
