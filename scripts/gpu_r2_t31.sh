set -x
for r in 4 8 2; do MOE_GATE_TILE_RPT=$r timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c4 rpt=$r', round(j['ms_per_step']*1000,1), j.get('stage_ms'))"; done
ncu --set full --clock-control none --import-source on -k regex:ln_gate -c 1 -o gpurun_out/r2_ln_only_c4 python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
