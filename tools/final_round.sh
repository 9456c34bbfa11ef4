# End-of-round evidence on a 4-GPU box: the one-GPU profile pass (tools/profile_round.sh), then the N = 2 and
# N = 4 bench lines and the N = 2 per-phase trace of the fused round.
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1; tail -3 gpurun_out/profile_round.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2961$n bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "bench N=$n rc $?"
done
N=2 bash tools/trace_comm.sh > gpurun_out/trace_n2_summary.txt 2>&1
for n in 1 2 4; do grep "^{" gpurun_out/bench_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($n, round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), round(d['e2e']['sync_per_step']['value']), d['clocks']['reasons'])"; done
