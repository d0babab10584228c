for a in "1024 32 1 1" "1024 32 64 1" "512 8 4096 2"; do timeout 300 python scripts/gate_trace.py $a 2>&1 | grep "^ln_gate" | tail -1 | cut -c1-260; done
