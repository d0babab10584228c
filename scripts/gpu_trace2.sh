python -m pytest tests/test_gpu_layer.py tests/test_golden.py tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -2
for cfg in auto 1,1 4,1 8,1 8,2; do
  for shape in "1024 4096 32 64 1" "512 2048 8 4096 2" "1024 4096 64 16384 1" "1024 4096 32 1 1"; do
    if [ $cfg = auto ]; then MOE_GATE_TRACE=1 python scripts/route_probe.py $shape 2>&1 | grep -E "gate_trace|route" | tail -2;
    else MOE_GATE_TRACE=1 MOE_GATE_CFG=$cfg python scripts/route_probe.py $shape 2>&1 | grep -E "gate_trace" | tail -1; fi
  done
done
