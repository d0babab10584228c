timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_moec.py -q -x 2>&1 | tail -3
timeout 1500 python bench.py --workload c4_encoder --steps 5 --warmup 2 2>&1 | tail -1
