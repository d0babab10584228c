# round-2 baseline: GPU tests + bench lines for C2/C3/C4/C5
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python bench.py 2>&1 | tail -1
for w in c3_1 c3_64 c4 c5; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
