timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attention_tc|gemm_tc_kernel<16" -c 2 -o gpurun_out/prof_c4_encoder python bench.py --workload c4_encoder --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/prof_c4_encoder.ncu-rep
