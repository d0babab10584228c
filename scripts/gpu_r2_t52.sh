for t in 0 128; do for r in 0 2 4; do
  MOE_GATE_TILE=$t MOE_GATE_TILE_RPT=$r timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('c5 tile=$t rpt=$r', round(j['ms_per_step']*1000,1), s.get('layer_norm'), s.get('gate_logits'))"
done; done
