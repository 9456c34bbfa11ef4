# A/B of the fused round's weight-image delivery (DQN_ROUND_IMG_COPY=1: one 16-byte copy by the last conv block;
# 0: 2-byte scattered peer stores per element) on BJ.configs[2] at N = 2 (and 4): bench lines, traces, multi-GPU tests
NG=$(nvidia-smi -L | wc -l)
tr() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2981$n bench.py --gpus $n --steps 3000 --warmup 50 --e2e-steps 20 --profile-steps 0 --no-cpu-baseline --no-acting "$@" 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step']*1e3,2))"; }
for rep in 1 2; do
  for go in 0 1; do echo "N=2 go=$go: $(DQN_ROUND_IMG_COPY=$go tr 2)"; done
  if [ $NG -ge 4 ]; then for go in 0 1; do echo "N=4 go=$go: $(DQN_ROUND_IMG_COPY=$go tr 4)"; done; fi
done
for go in 0 1; do DQN_ROUND_IMG_COPY=$go bash tools/trace_comm.sh > gpurun_out/trace_go$go.txt 2>&1; echo "trace go=$go"; grep -E "fused round \(6|relative to" gpurun_out/trace.log | head -4; done
DQN_ROUND_IMG_COPY=1 timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x 2>&1 | tail -2
