MOE_NO_PDL=1 MOE_NO_FUSED_COMBINE=1 timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "fused_gate_routing_exact and 16384" 2>&1 | tail -1
MOE_NO_PDL=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "fused_gate_routing_exact and 16384" 2>&1 | grep -v "^=========         Host Frame" | head -40
