set -x
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x -k "decode or pinned or quantize or host" 2>&1 | tail -6
timeout 600 python bench.py --force-ep --workload c5 --steps 20 --warmup 3 2>/dev/null | tail -1
timeout 600 python bench.py --workload decode_prune --steps 5 --warmup 3 2>&1 | tail -1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
timeout 300 python bench.py --workload c4 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
python scripts/quant_bench.py 2>&1 | tail -8
bash scripts/gpu_r2_prof.sh
