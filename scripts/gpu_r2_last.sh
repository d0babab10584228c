set -x
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/last_c2.json; cut -c1-400 gpurun_out/last_c2.json
python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 | cut -c1-300
