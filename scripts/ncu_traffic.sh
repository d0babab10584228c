# DRAM bytes per launch of the dominant kernels (FFN1 + FFN2) per bench
# workload: ncu (one GPU) -> gpurun_out/traffic_<workload>.csv
set -x
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
cap() { local w=$1; shift; timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_tc|gemv" -s 4 -c 4 --csv --log-file gpurun_out/traffic_$w.csv python scripts/layer_once_gpu.py "$@" > /dev/null 2>&1; echo "$w rc=$?"; }
cap c2 512 2048 8 4096 2 4
cap c3_1 1024 4096 32 1 1 4
cap c3_8 1024 4096 32 8 1 4
cap c3_64 1024 4096 32 64 1 4
cap c4 1024 4096 64 16384 1 4
cap c5 2048 8192 128 4096 2 4
cap c1i4 512 2048 8 256 1 4
