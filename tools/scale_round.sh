# Multi-GPU evidence (gpurun --gpus 4): the whole GPU test suite, N = 2 and N = 4 bench lines (configs[2],
# fused server round), the N = 2 per-phase trace of the round, and the model-size sweep at N = 1 and 4.
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2961$n bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "bench N=$n rc $?"; grep "^{" gpurun_out/bench_n$n.json | cut -c1-200
done
N=2 bash tools/trace_comm.sh > gpurun_out/trace_n2_summary.txt 2>&1; cat gpurun_out/trace_n2_summary.txt
N=1 bash tools/model_sweep.sh > /dev/null 2>&1; N=4 bash tools/model_sweep.sh > /dev/null 2>&1
wc -l gpurun_out/sweep_n*.jsonl
