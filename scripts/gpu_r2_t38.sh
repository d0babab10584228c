timeout 600 python -m pytest tests/test_moe_bench.py -q 2>&1 | tail -5
paper_2211_10017_b200/moe_bench --config tests/golden/model_int4.moec --precision int4 --batch 8 64 --beam 1 4 --prune both --src-len 8 --max-len 32 --out gpurun_out/moe_bench_report.jsonl
