# A/B of the Store folded into the conv forward (DQN_STORE_IN_FWD) on BJ.configs[1]'s e2e loop (dqn_store_and_train)
timeout 900 python -m pytest tests/test_gpu_store_and_train.py tests/test_gpu_replay_dedup.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2 3; do for v in 0 1; do
  echo "c2 early=$v: $(DQN_STORE_IN_FWD=$v timeout 300 python bench.py --steps 200 --warmup 20 --e2e-steps 2000 --profile-steps 0 --no-cpu-baseline --no-acting 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['e2e']['value']), round(d['e2e']['sync_per_step']['value']))")"
done; done
