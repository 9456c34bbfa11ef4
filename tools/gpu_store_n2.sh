# N = 2 (fused server round): store-and-train bit identity, the multi-GPU suite, and an e2e A/B of the Store inside
# the conv forward (DQN_STORE_IN_FWD) on BJ.configs[2]
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -x 2>&1 | tail -2
tr() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 --steps 500 --warmup 20 --e2e-steps 1000 --profile-steps 0 --no-cpu-baseline --no-acting 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['e2e']['value']))"; }
for rep in 1 2 3; do for v in 0 1; do echo "N=2 store_in_fwd=$v: $(DQN_STORE_IN_FWD=$v tr)"; done; done
