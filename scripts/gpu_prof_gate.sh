ncu --set full --clock-control none --import-source on -k regex:"gate_topk|ln_rows" -s 4 -c 2 -o gpurun_out/prof_gate3_c2 python scripts/layer_once.py 512 2048 8 4096 2 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gate_topk" -s 2 -c 1 -o gpurun_out/prof_gate3_c3 python scripts/layer_once.py 1024 4096 32 64 1 3 > /dev/null 2>&1
