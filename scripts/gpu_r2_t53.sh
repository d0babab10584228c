for w0 in 1 0; do
  for a in "512 8 4096 2" "1024 32 64 1" "1024 64 16384 1" "2048 128 4096 2"; do MOE_GATE_LN_WARP0=$w0 timeout 300 python scripts/gate_trace.py $a 2>&1 | grep "^ln_gate\|^ln_rows" | tail -1 | sed "s/^/warp0=$w0 /" | cut -c1-200; done
  for w in c2 c3_64 c4 c5; do MOE_GATE_LN_WARP0=$w0 timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w warp0=$w0', round(j['ms_per_step']*1000,2), s.get('layer_norm'))"; done
done
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py tests/test_gpu_encoder.py -q -x -k "routing or gate or layer_norm or decode or encoder" 2>&1 | tail -2
