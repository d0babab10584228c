set -x
timeout 600 python -m pytest tests/test_gpu_dropin.py -x -q 2>&1 | tail -5
python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1
for w in c3_1 c3_8 c3_64 c4; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_64.csv python bench.py --workload c3_64 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
