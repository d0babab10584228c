rm -f gpurun_out/tc_trace_c5.bin
MOE_TC_TRACE=gpurun_out/tc_trace_c5.bin timeout 600 python scripts/trace_gemm.py gpurun_out/tc_trace_c5.bin 128 8192 2048 8192 2>&1 | tail -3
python scripts/trace_analyze.py gpurun_out/tc_trace_c5.bin 2>&1 | head -60
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc" -s 2 -c 1 -o gpurun_out/prof_c5_ffn1 python scripts/layer_once_gpu.py 2048 8192 128 4096 2 3 > /dev/null 2>&1
ls gpurun_out | grep c5
