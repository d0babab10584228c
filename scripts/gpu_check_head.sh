timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for a in "1024 64 64 16384 1 16 80" "512 2048 8 4096 2 4 80" "1024 4096 32 64 1 4 80"; do timeout 300 python scripts/stress_layer.py $a 2>&1 | grep -E "iter|ok" | head -2; done
python bench.py 2>&1 | tail -1 > gpurun_out/bench_c2_head.json; python3 -c "
import json; j=json.load(open('gpurun_out/bench_c2_head.json')); print('C2', 'us=%.1f'%(1e3*j['ms_per_step']), 'tok/s=%.4g'%j['value'], 'e2e=%.4g'%j['e2e']['value'], 'frac=%.3f'%j['roofline']['frac'], j['clocks'])"
for w in c3_1 c3_64 c4; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
