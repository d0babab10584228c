for g in 1 0; do for c in 1 2 3 4; do MOE_HOST_GRAPH=$g MOE_HOST_CHUNKS=$c timeout 300 python scripts/e2e_probe.py 512 2048 8 4096 2 2>&1 | tail -1 | sed "s/^/graph=$g /"; done; done
for g in 1 0; do for c in 2 4; do MOE_HOST_GRAPH=$g MOE_HOST_CHUNKS=$c timeout 300 python scripts/e2e_probe.py 1024 4096 64 16384 1 2>&1 | tail -1 | sed "s/^/graph=$g /"; done; done
python scripts/h2d_probe.py 2>&1 | tail -12
