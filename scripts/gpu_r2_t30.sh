set -x
MOE_GEMV_PAIR=0 timeout 600 python scripts/pair_stress.py gpurun_out/ps_two.npz 2>&1 | tail -2
MOE_GEMV_PAIR=1 timeout 600 python scripts/pair_stress.py gpurun_out/ps_pair.npz gpurun_out/ps_two.npz 2>&1 | tail -17
MOE_GEMV_PAIR=1 timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_parity_configs.py -q -k "decode or c3" 2>&1 | tail -3
for w in c3_1 c3_8 c3_64; do for pr in 0 1; do
  MOE_GEMV_PAIR=$pr timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w pair=$pr', round(j['ms_per_step']*1000,2), j.get('stage_ms',{}).get('ffn1'), j['roofline']['frac'])"
done; done
for pr in 0 1; do MOE_GEMV_PAIR=$pr timeout 600 python bench.py --workload decode_prune --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('decode_prune pair=$pr', j['ms_per_step'], j['pruning'])"; done
