timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -2
timeout 120 python scripts/gate_trace.py 512 8 4096 2
timeout 120 python scripts/gate_trace.py 1024 64 16384 1
timeout 120 python scripts/gate_trace.py 1024 32 64 1
timeout 120 python scripts/gate_trace.py 1024 32 1 1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:ln_gate -s 3 -c 1 -o gpurun_out/prof_lngate_c2 python scripts/gate_trace.py 512 8 4096 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:ln_gate -s 3 -c 1 -o gpurun_out/prof_lngate_c3 python scripts/gate_trace.py 1024 32 64 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:ln_gate -s 3 -c 1 -o gpurun_out/prof_lngate_c4 python scripts/gate_trace.py 1024 64 16384 1 > /dev/null 2>&1
ls -la gpurun_out/
