n=0; for i in 1 2 3 4; do r=$(timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "fused_gate_routing_exact and 16384" 2>&1 | tail -1); case "$r" in *failed*) n=$((n+1));; esac; done; echo "PDL default failures=$n/4"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for e in "X=1" "MOE_NO_PDL=1"; do for w in c2 c3_1 c3_64 c4; do env $e timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$e', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'kern=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done; done
