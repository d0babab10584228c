nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/chain_bench scripts/chain_bench.cu && /tmp/chain_bench
