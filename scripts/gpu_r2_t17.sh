timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ln_gate" -s 2 -c 1 -o gpurun_out/r2_prof_gate_c4 python scripts/layer_once_gpu.py 1024 4096 64 16384 1 3 > gpurun_out/ncu_gate_c4.log 2>&1
echo rc=$?
