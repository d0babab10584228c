timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/bench_c2_final.json; cat gpurun_out/bench_c2_final.json | python3 -c "
import sys,json; j=json.loads(sys.stdin.read()); print('C2', 'us=%.1f'%(1e3*j['ms_per_step']), 'tok/s=%.4g'%j['value'], 'e2e=%.4g'%j['e2e']['value'], 'frac=%.3f'%j['roofline']['frac'], 'cpu=', j['cpu_baseline']['value'], 'launches=', j['gpu_launches'], j['clocks'])"
python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1
