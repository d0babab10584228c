MOE_NO_PDL=1 timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu 2>&1 | grep -E "^E |Error|FAILED|assert|passed|failed" | head -20
