# N=2 bench with DQN_TRACE_COMM=1: per-phase timing of the fused server round (kernels_comm.cu)
# and of the next step's first kernel, printed by each rank to gpurun_out/trace.log
DQN_TRACE_COMM=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-2} \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus ${N:-2} --replay 100000 --steps 1000 \
  --e2e-steps 5 --profile-steps 0 > gpurun_out/trace.log 2>&1
grep -E "fused round \(6|next fwd" gpurun_out/trace.log | head -4
grep "^{" gpurun_out/trace.log | cut -c90-200
