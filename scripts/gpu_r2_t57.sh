for bn in 0 160 192 224 256 257; do
  MOE_TC_BN=$bn timeout 600 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c2 BN=$bn', round(j['ms_per_step']*1000,2), round(j['roofline']['kernel_ms_per_step']*1000,2), round(j['roofline']['frac'],3))"
done
for bnm in 160 224 256 257; do
  MOE_TC_BNM=$bnm timeout 600 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c2 BNM=$bnm', round(j['ms_per_step']*1000,2), round(j['roofline']['kernel_ms_per_step']*1000,2), round(j['roofline']['frac'],3))"
done
