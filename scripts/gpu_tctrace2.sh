rm -f gpurun_out/tc_trace_*.bin
for P in 1 0; do
MOE_TC_PAIR=$P python scripts/trace_gemm.py gpurun_out/tc_trace_c2_p$P.bin 8 8192 512 2048
MOE_TC_PAIR=$P python scripts/trace_gemm.py gpurun_out/tc_trace_c4_p$P.bin 64 16384 1024 4096
MOE_TC_PAIR=$P MOE_TC_BN=224 python scripts/trace_gemm.py gpurun_out/tc_trace_c4_p${P}_224.bin 64 16384 1024 4096
done
for f in gpurun_out/tc_trace_*.bin; do echo $f; python scripts/trace_analyze.py $f; done
