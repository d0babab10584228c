# GPU tests, then the C2 bench and the decode/prefill workloads, then a launch list
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1
for w in c3_1 c3_8 c3_64 c4; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_64.csv python bench.py --workload c3_64 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
