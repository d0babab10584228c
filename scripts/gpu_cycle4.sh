set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1
for w in c1i4 c3_1 c3_8 c3_64 c4; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
for w in c2 c4 c3_64; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:"gemv" -s 4 -c 2 -o gpurun_out/prof_gemv2_c3 python scripts/layer_once.py 1024 4096 32 64 1 3 > /dev/null 2>&1
