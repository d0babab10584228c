timeout 300 ncu --set full --import-source on --clock-control none -k regex:plan_place_fused -s 3 -c 1 -o gpurun_out/prof_place_c2 python scripts/gate_trace.py 512 8 4096 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:combine -s 3 -c 1 -o gpurun_out/prof_combine_c2 python scripts/layer_once.py 512 2048 8 4096 2 6 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 6 -c 2 -o gpurun_out/prof_gemm_c2 python scripts/layer_once.py 512 2048 8 4096 2 6 > /dev/null 2>&1
ls gpurun_out
