echo "b16 f64 E64"; timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 100 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f64 E64 pair0"; MOE_TC_PAIR=0 timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 100 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f256 E64"; timeout 300 python scripts/stress_layer.py 1024 256 64 16384 1 16 60 2>&1 | grep -E "iter|ok" | head -3
