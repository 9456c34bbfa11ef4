# N = 2 and N = 4 bench lines (configs[2], fused server round) + the N = 2 per-phase trace
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2961$n bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "bench N=$n rc $?"; cut -c1-160 gpurun_out/bench_n$n.json
done
N=2 bash tools/trace_comm.sh > gpurun_out/trace_n2_summary.txt 2>&1; cat gpurun_out/trace_n2_summary.txt
