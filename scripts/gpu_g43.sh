nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/chain_bench scripts/bench/chain_bench.cu && /tmp/chain_bench
timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -1
for w in c2 c3_1; do timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:30], 'us=%.1f'%(1e3*j['ms_per_step']), {k: round(v*1e3,1) for k,v in j.get('stage_ms',{}).items()})"; done
for w in c2 c3_1 c4; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; done
