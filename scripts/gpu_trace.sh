for cfg in 1,1 4,1 8,1 8,2; do
  for shape in "1024 4096 32 64 1" "512 2048 8 4096 2" "1024 4096 64 16384 1"; do
    MOE_GATE_TRACE=1 MOE_GATE_CFG=$cfg python scripts/route_probe.py $shape 2>&1 | grep gate_trace | tail -1
  done
done
