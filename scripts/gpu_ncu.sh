# full ncu captures of the hot kernels (one launch each)
set -x
python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:gate_fused -s 2 -c 1 -o gpurun_out/prof_gate_c2 python scripts/layer_once.py 512 2048 8 4096 2 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_fused -s 2 -c 1 -o gpurun_out/prof_gate_c4 python scripts/layer_once.py 1024 4096 64 16384 1 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 2 -o gpurun_out/prof_gemv_c3 python scripts/layer_once.py 1024 4096 32 64 1 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 2 -o gpurun_out/prof_gemm_c4 python scripts/layer_once.py 1024 4096 64 16384 1 3 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
