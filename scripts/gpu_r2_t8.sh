set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_decode.py -q -x -k "gemv or decode" 2>&1 | tail -2
python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep ln_gate
python scripts/gate_trace.py 1024 32 1 1 2>&1 | grep ln_gate
python scripts/gemv_trace.py 1024 4096 32 64 1 2>&1 | grep gemv
for w in c3_1 c3_64; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300; done
python bench.py --workload decode_prune --steps 5 --warmup 3 2>&1 | tail -1 | grep -o '"pruning.*'
python scripts/trace_gemm.py gpurun_out/tc_trace_c2.bin 8 8192 512 2048 2>&1 | tail -3
python scripts/trace_analyze.py gpurun_out/tc_trace_c2.bin 2>&1 | tail -24
