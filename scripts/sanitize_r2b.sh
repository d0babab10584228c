# compute-sanitizer over the round-2 late kernels: the wide gate (LN-only
# pass + gate_tile_kernel), the device encoder (attention, embeddings,
# residual adds, fp16 projections) -- memcheck / racecheck / synccheck
set -x
S="compute-sanitizer --print-limit 50 --error-exitcode 9"
run() { # tool tag cmd...
  local tool=$1 tag=$2; shift 2
  timeout 1200 $S --tool $tool "$@" > gpurun_out/san_${tool}_${tag}.log 2>&1; echo "$tool $tag rc=$?"
}
for tool in memcheck racecheck synccheck; do
  run $tool gatetile python scripts/layer_once.py 256 512 64 5000 1 2
  run $tool encoder python -m pytest tests/test_gpu_encoder.py -q -k "matches_reference and int4 and 0"
done
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|hazard\|passed\|failed" gpurun_out/san_*gatetile*.log gpurun_out/san_*encoder*.log | sort | uniq -c
