set -x
for c in 2 4; do MOE_HOST_CHUNKS=$c MOE_HOST_GRAPH=0 python scripts/e2e_probe.py 512 2048 8 4096 2; MOE_HOST_CHUNKS=$c python scripts/e2e_probe.py 512 2048 8 4096 2; done
MOE_HOST_CHUNKS=4 MOE_HOST_GRAPH=0 python scripts/e2e_probe.py 1024 4096 64 16384 1
