for rm in 1 0; do
  for a in "512 8 4096 2" "1024 32 64 1" "2048 128 4096 2" "1024 32 8 1"; do MOE_GATE_ROWMAJOR=$rm timeout 300 python scripts/gate_trace.py $a 2>&1 | grep "^ln_gate" | tail -1 | sed "s/^/rowmajor=$rm /" | cut -c1-230; done
done
for rm in 1 0; do for w in c2 c3_8 c3_64 c5; do
  MOE_GATE_ROWMAJOR=$rm timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w rowmajor=$rm', round(j['ms_per_step']*1000,2), s.get('layer_norm'))"
done; done
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x -k "routing or gate or layer_norm or decode" 2>&1 | tail -2
