set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_moec.py tests/test_gpu_dropin.py -q -x -k "gemv or decode or layer or moec or quantize_model" 2>&1 | tail -3
for cfg in "1024 4096 32 1 1" "1024 4096 32 8 1" "1024 4096 32 64 1" "1024 4096 64 256 1"; do python scripts/gemv_trace.py $cfg 2>&1 | grep gemv; done
for w in c3_1 c3_8 c3_64 c1i4; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-330; done
python bench.py --workload decode_prune --steps 5 --warmup 3 2>&1 | tail -1 | cut -c 1-200
python bench.py --workload decode_prune --steps 5 --warmup 3 2>&1 | tail -1 | grep -o '"pruning.*'
