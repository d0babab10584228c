timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_moec.py -q -x 2>&1 | tail -15
