set -x
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x -k "fused_gate_routing or gate or decode_shapes" 2>&1 | tail -2
python scripts/gate_trace.py 1024 64 16384 1 2>&1 | grep ln_gate
python scripts/gate_trace.py 2048 128 4096 2 2>&1 | grep ln_gate
for w in c4 c5; do python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys,os; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:12], round(j['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in j['stage_ms'].items()})"; done
