set -x
for c in 1 2 4; do for gr in 1 0; do MOE_HOST_CHUNKS=$c MOE_HOST_GRAPH=$gr python scripts/e2e_probe2.py 512 2048 8 4096 2; done; done
for cfg in "512 8 4096 2" "1024 32 1 1" "1024 32 64 1"; do python scripts/gate_trace.py $cfg 2>&1 | tail -2; done
MOE_GATE_NO_EPG1=1 python scripts/gate_trace.py 512 8 4096 2 2>&1 | tail -2
python scripts/trace_gemm.py gpurun_out/tc_trace_c5b.bin 128 8192 2048 8192 2>&1 | tail -2
python scripts/trace_analyze.py gpurun_out/tc_trace_c5b.bin 2>&1 | grep -E "per k-block|wait|total"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x -k "pair or gate or routing or decode_shapes" 2>&1 | tail -3
python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
python bench.py --workload c3_1 --steps 50 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
