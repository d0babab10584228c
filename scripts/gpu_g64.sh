for i in 1 2 3; do MOE_NO_PDL=1 timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "fused_gate_routing_exact and 16384" 2>&1 | tail -1; done
for i in 1 2; do timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "fused_gate_routing_exact and 16384" 2>&1 | tail -1; done
MOE_NO_PDL=1 CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu 2>&1 | grep -E "FAILED|passed|failed|Error" | head -5
