set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for cfg in "1024 32 1 1" "1024 32 64 1"; do python scripts/gate_trace.py $cfg 2>&1 | tail -2 | head -1; done
for c in 2 3; do MOE_GEMV_CTAS=$c python scripts/gemv_trace.py 1024 4096 32 64 1 2>&1 | grep gemv; done
for w in c3_1 c3_64; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300; done
for w in c3_1 c3_64; do MOE_PDL=3 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300; done
python bench.py --steps 100 --warmup 5 2>&1 | tail -1
python bench.py --workload decode_prune --steps 5 --warmup 3 2>&1 | tail -1
