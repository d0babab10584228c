echo "C2 int4"; timeout 300 python scripts/stress_layer.py 512 2048 8 4096 2 4 100 2>&1 | grep -E "iter|ok" | head -3
echo "C4 int4"; timeout 300 python scripts/stress_layer.py 1024 4096 64 16384 1 4 60 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f64 pair0"; MOE_TC_PAIR=0 timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 100 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f64 BN256"; MOE_TC_BN=256 timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 100 2>&1 | grep -E "iter|ok" | head -3
echo "b4 f64"; timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 4 100 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f64 exact-ish E8"; timeout 300 python scripts/stress_layer.py 1024 64 8 16384 1 16 100 2>&1 | grep -E "iter|ok" | head -3
