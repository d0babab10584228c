set -x
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 | cut -c1-300
python bench.py --workload c4_encoder --steps 5 --warmup 2 2>&1 | tail -1 > gpurun_out/final_c4_encoder.json
