# round-end evidence: tests, bench lines (both arms), launch lists, ncu captures
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
python bench.py 2>&1 | tail -1 > gpurun_out/bench_c2.json; cat gpurun_out/bench_c2.json
python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1
for w in c1i4 c3_1 c3_8 c3_64 c4 c5; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
for w in c2 c3_64 c4; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc|ln_gate|plan_place|combine" -s 8 -c 5 -o gpurun_out/prof_final_c2 python scripts/layer_once.py 512 2048 8 4096 2 6 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemv|ln_gate" -s 6 -c 3 -o gpurun_out/prof_final_c3 python scripts/layer_once.py 1024 4096 32 64 1 6 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc" -s 4 -c 2 -o gpurun_out/prof_final_c4 python scripts/layer_once.py 1024 4096 64 16384 1 4 > /dev/null 2>&1
ls -la gpurun_out
