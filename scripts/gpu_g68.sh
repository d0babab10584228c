rm -f gpurun_out/tc_trace_*.bin
python scripts/trace_gemm.py gpurun_out/tc_trace_c2_auto.bin 8 8192 512 2048 2>&1 | grep "us "
MOE_TC_BN=257 python scripts/trace_gemm.py gpurun_out/tc_trace_c2_257.bin 8 8192 512 2048 2>&1 | grep "us "
python scripts/trace_analyze.py gpurun_out/tc_trace_c2_auto.bin
python scripts/trace_analyze.py gpurun_out/tc_trace_c2_257.bin
