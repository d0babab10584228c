rm -f gpurun_out/tc_trace_c2.bin gpurun_out/tc_trace_c4.bin
python scripts/trace_gemm.py gpurun_out/tc_trace_c2.bin 8 8192 512 2048
python scripts/trace_gemm.py gpurun_out/tc_trace_c4.bin 64 16384 1024 4096
python scripts/trace_analyze.py gpurun_out/tc_trace_c2.bin
python scripts/trace_analyze.py gpurun_out/tc_trace_c4.bin
