# round-2 evidence: tests, smoke, bench lines (all workloads, both arms),
# launch lists and ncu captures (summarised into profiles/ by
# scripts/make_profiles.py)
set -x
export PARITY_LOG=gpurun_out/parity_final.jsonl
rm -f $PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/final_c2.json; cat gpurun_out/final_c2.json
python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 > gpurun_out/final_ref.json; cat gpurun_out/final_ref.json
for w in c1i4 c3_1 c3_8 c3_64 c4 c5; do python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/final_$w.json; cat gpurun_out/final_$w.json | cut -c1-200; done
python bench.py --workload decode_prune --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/final_decode.json
python bench.py --workload c4_stack --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/final_c4_stack.json
python bench.py --workload c4_encoder --steps 5 --warmup 2 2>&1 | tail -1 > gpurun_out/final_c4_encoder.json
python bench.py --force-ep --workload c5 --steps 20 --warmup 3 2>/dev/null | tail -1 > gpurun_out/final_ep_c5.json
python scripts/quant_bench.py > gpurun_out/final_quant.jsonl 2>&1
for w in c2 c3_64 c4; do
  case $w in c2) a="512 2048 8 4096 2";; c3_64) a="1024 4096 32 64 1";; c4) a="1024 4096 64 16384 1";; esac
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python scripts/layer_once_gpu.py $a 4 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc|ln_gate|plan|combine" -s 5 -c 5 -o gpurun_out/prof_final_c2 python scripts/layer_once_gpu.py 512 2048 8 4096 2 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemv|ln_gate" -s 3 -c 3 -o gpurun_out/prof_final_c3 python scripts/layer_once_gpu.py 1024 4096 32 64 1 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc|gate_tile|ln_gate" -s 4 -c 4 -o gpurun_out/prof_final_c4 python scripts/layer_once_gpu.py 1024 4096 64 16384 1 3 > /dev/null 2>&1
ls -la gpurun_out | tail -30
