set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for cfg in "512 2048 8 4096 2" "512 2048 8 4096 1" "1024 4096 32 1 1" "1024 4096 32 8 1" "1024 4096 32 64 1" "1024 4096 64 16384 1"; do
  MODES=1 timeout 300 python scripts/probe_layer.py $cfg 2>&1 | tail -2
done
