set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_golden.py -q -x -k "gate or routing or layer or combine or plan or golden" 2>&1 | tail -2
python scripts/gate_trace.py 512 8 4096 2 "2,1" "4,1" "8,1" "2,2" "4,2" 2>&1 | grep "route\|ln_gate\|plan_place"
python scripts/gate_trace.py 1024 32 1 1 "2,1" "4,1" "8,1" 2>&1 | grep "route\|ln_gate"
python scripts/gate_trace.py 1024 32 64 1 "2,1" "4,1" "8,1" 2>&1 | grep "route\|ln_gate"
python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-260
