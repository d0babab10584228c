timeout 300 python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep "plan_place_fused" | tail -2
timeout 300 python scripts/gate_trace.py 1024 32 64 1 2>&1 | grep "plan_place_fused" | tail -1
