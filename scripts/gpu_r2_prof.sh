# round-2 profiling: tcgen05 issue microbench, gate phase traces, ncu full captures
set -x
./scripts/mma_issue_bench
for cfg in "512 8 4096 2" "1024 32 1 1" "1024 32 64 1" "1024 64 16384 1"; do
  python scripts/gate_trace.py $cfg 2>&1 | tail -3
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemv|ln_gate" -s 6 -c 3 -o gpurun_out/r2_prof_c3_64 python scripts/layer_once.py 1024 4096 32 64 1 6 > gpurun_out/ncu_c3_64.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemv|ln_gate" -s 6 -c 3 -o gpurun_out/r2_prof_c3_1 python scripts/layer_once.py 1024 4096 32 1 1 6 > gpurun_out/ncu_c3_1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc|ln_gate|plan|combine" -s 8 -c 5 -o gpurun_out/r2_prof_c2 python scripts/layer_once.py 512 2048 8 4096 2 6 > gpurun_out/ncu_c2.log 2>&1
ls -la gpurun_out
