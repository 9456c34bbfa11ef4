# End-of-round evidence on a 4-GPU box: the GPU test suite, the one-GPU profile pass (tools/profile_round.sh),
# the N = 2 and N = 4 bench lines, the N = 2 per-phase trace, and BJ.configs[3] / [4] lines at N = 1.
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1; grep " rc " gpurun_out/profile_round.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2961$n bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "bench N=$n rc $?"
done
N=2 bash tools/trace_comm.sh > gpurun_out/trace_n2_summary.txt 2>&1
for c in c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-acting > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for f in n1 n2 n4 c4 c5; do grep "^{" gpurun_out/bench_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$f', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), d['clocks']['reasons'], d['roofline']['bound'], round(d['roofline']['frac'], 4))"; done
