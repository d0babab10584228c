for rep in 1 2 3; do for v in 1 0; do
  MOE_HOST_D2D=$v timeout 300 python scripts/e2e_probe.py 512 2048 8 4096 2 2>&1 | tail -1 | sed "s/^/d2d=$v /"
done; done
for v in 1 0; do MOE_HOST_D2D=$v timeout 300 python scripts/e2e_probe.py 1024 4096 64 16384 1 2>&1 | tail -1 | sed "s/^/d2d=$v /"; done
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_dropin.py -q -x -k "host or pinned or chunk" 2>&1 | tail -2
