for sp in 0 2 4 8; do for c in 3 4; do
  MOE_GEMV_SPLITS=$sp MOE_GEMV_CTAS=$c timeout 600 python bench.py --workload c3_64 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('c3_64 splits=$sp ctas=$c', round(j['ms_per_step']*1000,2), s.get('ffn1'), s.get('ffn2'))"
done; done
for sp in 0 2 4; do MOE_GEMV_SPLITS=$sp timeout 600 python bench.py --workload c3_8 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('c3_8 splits=$sp', round(j['ms_per_step']*1000,2), s.get('ffn1'), s.get('ffn2'))"; done
