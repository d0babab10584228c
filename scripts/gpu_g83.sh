timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
for a in "1024 64 64 16384 1 16 100" "1024 4096 64 16384 1 4 50" "1024 256 64 16384 1 8 60" "512 2048 8 4096 2 4 60"; do echo "== $a"; timeout 300 python scripts/stress_layer.py $a 2>&1 | grep -E "iter|ok" | head -2; done
for e in "MOE_FUSED_COMBINE=1" "MOE_FUSED_COMBINE=0"; do for w in c4 c2; do env $e timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done; done
