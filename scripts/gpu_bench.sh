# bench + launch list + one full ncu capture of the top kernel (C2)
set -x
python bench.py --steps 200 --warmup 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json
for w in c3_1 c3_64 c4; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 6 -c 2 -o gpurun_out/prof_gemm_c2 python scripts/layer_once.py 512 2048 8 4096 2 5 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
