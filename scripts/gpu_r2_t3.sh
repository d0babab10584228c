set -x
for c in 1 2 4; do MOE_HOST_CHUNKS=$c python scripts/e2e_probe.py 512 2048 8 4096 2; done
for c in 1 4; do MOE_HOST_CHUNKS=$c python scripts/e2e_probe.py 1024 4096 64 16384 1; done
python scripts/e2e_probe.py 512 2048 8 4096 2
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_layer.py tests/test_gpu_kernels.py tests/test_gpu_ep.py -q -x -k "decode or pinned or quantize or host or ep" 2>&1 | tail -4
timeout 600 python bench.py --force-ep --workload c5 --steps 20 --warmup 3 2>/dev/null | tail -1
timeout 600 python bench.py --force-ep --workload c2 --steps 20 --warmup 3 2>/dev/null | tail -1
