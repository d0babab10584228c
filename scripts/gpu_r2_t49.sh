timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4enc.csv python bench.py --workload c4_encoder --steps 1 --warmup 0 > /dev/null 2>&1
python scripts/make_profiles.py r2_c4_encoder gpurun_out/launches_c4enc.csv 2>&1 | tail -1
cat profiles/r2_c4_encoder.md | head -30
