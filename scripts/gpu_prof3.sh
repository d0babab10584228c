for cfg in auto 1,1 2,1 4,1 8,1 8,2; do
  for shape in "1024 4096 32 64 1" "512 2048 8 4096 2" "1024 4096 64 16384 1"; do
    if [ $cfg = auto ]; then python scripts/route_probe.py $shape; else MOE_GATE_CFG=$cfg python scripts/route_probe.py $shape; fi
  done
done 2>&1 | grep route
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:gate_topk -s 2 -c 1 -o gpurun_out/prof_gate4_c3 python scripts/layer_once.py 1024 4096 32 64 1 3 > gpurun_out/ncu_a.log 2>&1
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:gemv -s 2 -c 1 -o gpurun_out/prof_gemv4_c3 python scripts/layer_once.py 1024 4096 32 64 1 3 > gpurun_out/ncu_b.log 2>&1
tail -2 gpurun_out/ncu_a.log
