set -x
for c in 2 4; do MOE_HOST_CHUNKS=$c MOE_HOST_GRAPH=0 python scripts/e2e_probe.py 512 2048 8 4096 2; MOE_HOST_CHUNKS=$c python scripts/e2e_probe.py 512 2048 8 4096 2; done
MOE_HOST_CHUNKS=4 MOE_HOST_GRAPH=0 python scripts/e2e_probe.py 1024 4096 64 16384 1
set -x
for cfg in "1024 4096 32 1 1" "1024 4096 32 8 1" "1024 4096 32 64 1" "1024 4096 64 256 1"; do
  python scripts/gemv_trace.py $cfg 2>&1 | grep gemv
done
python scripts/trace_gemm.py gpurun_out/tc_trace_c5.bin 128 8192 2048 8192 2>&1 | tail -4
python scripts/trace_analyze.py gpurun_out/tc_trace_c5.bin 2>&1 | tail -20
MOE_TC_SMALL_PAIR=0 python scripts/trace_gemm.py gpurun_out/tc_trace_c5s.bin 128 8192 2048 8192 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "pair or quantize" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity_configs.py -q -x -k "c5" 2>&1 | tail -3
python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
MOE_TC_SMALL_PAIR=0 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
