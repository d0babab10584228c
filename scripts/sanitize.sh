# compute-sanitizer memcheck / racecheck / synccheck over one small layer
# forward per kernel family (tcgen05 GEMM pair + fused gate + plan + fused
# combine; decode GEMV; fp16-weight GEMM; EP loopback): logs to gpurun_out/
set -x
S="compute-sanitizer --print-limit 50 --error-exitcode 9"
run() { # tool tag args...
  local tool=$1 tag=$2; shift 2
  timeout 900 $S --tool $tool python "$@" > gpurun_out/san_${tool}_${tag}.log 2>&1; echo "$tool $tag rc=$?"
}
for tool in memcheck racecheck synccheck; do
  run $tool tc4   scripts/layer_once.py 256 512 8 1200 2 2
  run $tool tck1  scripts/layer_once.py 256 512 8 1200 1 2
  run $tool gemv  scripts/layer_once.py 256 512 8 64 1 2
done
run memcheck tc16 scripts/layer_once16.py 256 512 8 1200 1 2
run racecheck tc16 scripts/layer_once16.py 256 512 8 1200 1 2
run memcheck ep   scripts/ep_loopback_once.py
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|hazard" gpurun_out/san_*.log | sort | uniq -c
