timeout 600 python scripts/ablate_gemm.py 2>&1 | tail -14
