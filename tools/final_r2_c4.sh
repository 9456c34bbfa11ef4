# Refresh of the BJ.configs[3] lines after the bwd_reduce change, on a 4-GPU box (N = 1 and 4)
nvidia-smi -L
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n "$@"; }
timeout 600 python bench.py --config c4 --no-acting > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "c4 rc $?"
tr 4 --config c4 --no-acting > gpurun_out/r2_bench_c4_n4.json 2> gpurun_out/r2_bench_c4_n4.err; echo "c4 n4 rc $?"
for f in c4 c4_n4; do grep "^{" gpurun_out/r2_bench_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d.get('roofline') or {}
print('$f', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), d['clocks']['reasons'], r.get('bound'), round(r.get('frac') or 0, 4), d.get('regions_us'))"; done
