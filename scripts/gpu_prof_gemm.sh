ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 4 -c 2 -o gpurun_out/prof_gemm5_c2 python scripts/layer_once.py 512 2048 8 4096 2 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 2 -o gpurun_out/prof_gemm5_c4 python scripts/layer_once.py 1024 4096 64 16384 1 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"combine|permute|plan_" -s 8 -c 4 -o gpurun_out/prof_small_c2 python scripts/layer_once.py 512 2048 8 4096 2 3 > /dev/null 2>&1
ls gpurun_out/*gemm5* gpurun_out/*small*
