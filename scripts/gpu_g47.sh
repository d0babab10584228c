timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python scripts/gate_trace.py 512 8 4096 2 2>&1 | head -60
