set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1
for w in c3_64 c4; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
for w in c2 c4; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:gate_topk -s 2 -c 1 -o gpurun_out/prof_gtk_c2 python scripts/layer_once.py 512 2048 8 4096 2 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_topk -s 2 -c 1 -o gpurun_out/prof_gtk_c4 python scripts/layer_once.py 1024 4096 64 16384 1 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 2 -o gpurun_out/prof_gemm_c4 python scripts/layer_once.py 1024 4096 64 16384 1 3 > /dev/null 2>&1
