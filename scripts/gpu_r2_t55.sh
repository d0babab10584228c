for mr in 0 4 8 16; do for w in c3_8 c3_64 decode_prune; do
  if [ $w = decode_prune ]; then st=5; wu=3; else st=50; wu=5; fi
  MOE_GATE_MIN_ROWS=$mr timeout 600 python bench.py --workload $w --steps $st --warmup $wu --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w minrows=$mr', round(j['ms_per_step']*1000,2), s.get('layer_norm'), s.get('routing_plan'))"
done; done
