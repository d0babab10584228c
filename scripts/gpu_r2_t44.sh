for rep in 1 2; do
for c in 2 3; do MOE_HOST_CHUNKS=$c timeout 300 python scripts/e2e_probe.py 512 2048 8 4096 2 2>&1 | tail -1; done
MOE_HOST_EVEN=1 MOE_HOST_CHUNKS=3 timeout 300 python scripts/e2e_probe.py 512 2048 8 4096 2 2>&1 | tail -1 | sed 's/^/even /'
done
for c in 2 3; do MOE_HOST_CHUNKS=$c timeout 300 python scripts/e2e_probe.py 1024 4096 64 16384 1 2>&1 | tail -1; done
for c in 1 2 3; do MOE_HOST_CHUNKS=$c timeout 300 python scripts/e2e_probe.py 2048 8192 128 4096 2 2>&1 | tail -1; done
