set -x
for c in 1 2; do MOE_HOST_CHUNKS=$c python scripts/e2e_probe2.py 512 2048 8 4096 2; done
python scripts/e2e_probe2.py 512 2048 8 4096 2
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x -k "gate or routing or layer" 2>&1 | tail -2
python scripts/gate_trace.py 1024 64 16384 1 2>&1 | grep ln_gate
python scripts/gate_trace.py 2048 128 4096 2 2>&1 | grep ln_gate
for w in c2 c4 c5; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:12], round(j['ms_per_step']*1e3,1), 'us', round(j['value']/1e6,2), 'Mtok/s e2e', round(j['e2e']['value']/1e6,2), 'stage', {k: round(v*1e3,1) for k,v in j['stage_ms'].items()})"; done
