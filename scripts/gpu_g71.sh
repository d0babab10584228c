timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -m gpu -rf 2>&1 | grep -E "FAILED|passed|failed" | head
n=0; for i in 1 2 3 4 5; do r=$(timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "fused_gate_routing_exact and 16384" 2>&1 | tail -1); case "$r" in *failed*) n=$((n+1));; esac; done; echo "16384 failures=$n/5"
timeout 120 python scripts/gate_trace.py 512 8 4096 2
timeout 120 python scripts/gate_trace.py 1024 32 1 1
