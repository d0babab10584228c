timeout 300 python scripts/gate_trace.py 1024 64 16384 1 2>&1 | grep -v plan_place | tail -8
