set -x
python scripts/h2d_probe.py 2>&1 | tail -5
python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep plan_place
MOE_PLAN_COPY_LANES=1 python scripts/gate_trace.py 512 8 4096 2 2>&1 | grep plan_place
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -k "load_report or pinned" 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200; MOE_PLAN_COPY_LANES=1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200; done
