python -m pytest tests/test_gpu_kernels.py -x -q -k "gemv" 2>&1 | tail -3
ncu --set full --sampling-interval 0 --clock-control none --import-source on -k regex:gate_topk -s 2 -c 1 -o gpurun_out/prof_gate4_c3 python scripts/layer_once.py 1024 4096 32 64 1 3 > gpurun_out/ncu_a.log 2>&1
ncu --set full --sampling-interval 0 --clock-control none --import-source on -k regex:gemv -s 2 -c 1 -o gpurun_out/prof_gemv4_c3 python scripts/layer_once.py 1024 4096 32 64 1 3 > gpurun_out/ncu_b.log 2>&1
tail -3 gpurun_out/ncu_a.log
