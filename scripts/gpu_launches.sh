for cfg in "1024 4096 32 1 1" "1024 4096 32 64 1" "512 2048 8 4096 2" "1024 4096 64 16384 1"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$tag.csv python scripts/layer_once.py $cfg 3 > /dev/null 2>&1
done
ls gpurun_out
