for cfg in "X=1" "MOE_NO_FUSED_COMBINE=1" "MOE_TC_PAIR=0" "MOE_TC_BN=256"; do
  n=0; for i in 1 2 3 4 5; do r=$(env $cfg MOE_NO_PDL=1 timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "fused_gate_routing_exact and 16384" 2>&1 | tail -1); case "$r" in *failed*) n=$((n+1));; esac; done; echo "$cfg failures=$n/5"
done
