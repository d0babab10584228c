for sp in 0 1 2; do for w in c3_1 c3_8; do
  MOE_GEMV_SPLITS=$sp timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w splits=$sp', round(j['ms_per_step']*1000,2), s.get('ffn1'), s.get('ffn2'))"
done; done
