nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/chain_bench scripts/chain_bench.cu && /tmp/chain_bench
for cfg in "MOE_TC_PAIR=0" "MOE_TC_PAIR=1" "MOE_TC_BN=224"; do for w in c2 c4; do env $cfg timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('$cfg', j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), 'gemm=%.1f'%(1e3*j['roofline']['kernel_ms_per_step']))"; done; done
for w in c2 c3_1 c4; do timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/warm_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; done
