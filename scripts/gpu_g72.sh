for cfg in "X=1" "MOE_TC_PAIR=0" "MOE_TC_BN=256" "MOE_TC_BN=224"; do echo "== $cfg"; env $cfg timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 200 2>&1 | tail -2; done
echo "== bits4"; timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 4 200 2>&1 | tail -2
echo "== f4096 bits4"; timeout 300 python scripts/stress_layer.py 1024 4096 64 16384 1 4 100 2>&1 | tail -2
