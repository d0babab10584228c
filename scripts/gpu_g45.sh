nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/chain_bench scripts/chain_bench.cu && /tmp/chain_bench
timeout 120 python scripts/gate_trace.py 512 8 4096 2
timeout 120 python scripts/gate_trace.py 1024 32 1 1
timeout 120 python scripts/gate_trace.py 1024 32 64 1
timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k fused_gate 2>&1 | tail -2
