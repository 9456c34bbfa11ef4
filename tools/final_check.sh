timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "N=1 rc $?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2961$n bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo "N=$n rc $?"
done
for n in 1 2 4; do grep "^{" gpurun_out/bench_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($n, round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), round(d['e2e']['sync_per_step']['value']), d['clocks']['reasons'], d.get('roofline'))"; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
