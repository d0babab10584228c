set -x
export PARITY_LOG=gpurun_out/parity_r2.jsonl
rm -f $PARITY_LOG
timeout 1800 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_ep.py tests/test_gpu_fault_drill.py -q -x 2>&1 | tail -15
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --force-ep --workload c5 --steps 20 --warmup 3 2>&1 | grep -v NCCL | tail -2
timeout 300 python bench.py --steps 50 --warmup 5 2>&1 | tail -1
