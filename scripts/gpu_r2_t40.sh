for c in 3 2; do for w in c3_1 c3_8 c3_64; do
  MOE_GEMV_CTAS=$c timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms',{}); print('$w ctas=$c', round(j['ms_per_step']*1000,2), s.get('ffn1'), s.get('ffn2'), round(j['roofline']['frac'],3))"
done; done
for c in 3 2; do MOE_GEMV_CTAS=$c timeout 600 python bench.py --workload decode_prune --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('decode_prune ctas=$c', j['ms_per_step'])"; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x -k "gemv or decode" 2>&1 | tail -2
