# A/B of the bulk (reduce-)copy epilogue of the FC weight-gradient tiles (DQN_BULK_ACCUM) on BJ.configs[1] / [3]
for rep in 1 2 3; do for v in 0 1; do
  echo "c2 bulk=$v: $(DQN_BULK_ACCUM=$v timeout 300 python bench.py --steps 2000 --warmup 20 --e2e-steps 10 --profile-steps 0 --no-cpu-baseline --no-acting 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step']*1e3,2))")"
  echo "c4 bulk=$v: $(DQN_BULK_ACCUM=$v timeout 300 python bench.py --config c4 --steps 1000 --warmup 20 --e2e-steps 10 --profile-steps 0 --no-cpu-baseline --no-acting 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step']*1e3,2))")"
done; done
timeout 900 python -m pytest tests/test_gpu_bulk_accum.py tests/test_gpu_parity_gated.py tests/test_gpu_parity_bf16.py tests/test_gpu_async.py tests/test_gpu_full_size.py -m gpu -q -x 2>&1 | tail -2
