timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemv -s 4 -c 2 -o gpurun_out/prof_gemv_c3_1 python scripts/layer_once.py 1024 4096 32 1 1 6 > /dev/null 2>&1
timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/warm_c3_1.csv python bench.py --workload c3_1 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | tail -3
