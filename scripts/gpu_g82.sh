echo "b16 f64 E64 both k2"; timeout 300 python scripts/stress_stage.py 1024 64 64 16384 2 16 100 both 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f64 E64"; timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 150 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f64 E64 pair0"; MOE_TC_PAIR=0 timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 100 2>&1 | grep -E "iter|ok" | head -3
echo "b16 f256 E64"; timeout 300 python scripts/stress_layer.py 1024 256 64 16384 1 16 60 2>&1 | grep -E "iter|ok" | head -3
echo "fused b16"; MOE_FUSED_COMBINE=1 timeout 300 python scripts/stress_layer.py 1024 64 64 16384 1 16 100 2>&1 | grep -E "iter|ok" | head -3
echo "C4 int4"; timeout 300 python scripts/stress_layer.py 1024 4096 64 16384 1 4 40 2>&1 | grep -E "iter|ok" | head -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
for w in c2 c4; do timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done
