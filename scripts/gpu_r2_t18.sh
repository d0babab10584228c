set -x
python scripts/gate_trace.py 1024 64 16384 1 "8,2" "8,1,512" "8,2,512" "4,1,512" 2>&1 | grep "route\|ln_gate"
python scripts/gate_trace.py 2048 128 4096 2 "8,2" "8,1,512" "8,2,512" 2>&1 | grep "route\|ln_gate"
python scripts/gate_trace.py 512 8 4096 2 "2,1" "2,1,512" 2>&1 | grep "route\|ln_gate"
python bench.py --workload c4_stack --steps 5 --warmup 3 2>&1 | tail -1
