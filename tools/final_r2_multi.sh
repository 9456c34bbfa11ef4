# Refresh after the fused Store at N > 1, on a 4-GPU box: the multi-GPU tests (world 2 and 4) and the BJ.configs[2]
# lines at N = 2 / 4
nvidia-smi -L
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -rA > gpurun_out/r2_pytest_multi.log 2>&1; echo "multi rc $?"; grep -E "passed|failed" gpurun_out/r2_pytest_multi.log | tail -1
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n "$@"; }
tr 2 > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err; echo "n2 rc $?"
tr 4 > gpurun_out/r2_bench_n4.json 2> gpurun_out/r2_bench_n4.err; echo "n4 rc $?"
for f in n2 n4; do grep "^{" gpurun_out/r2_bench_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d.get('roofline') or {}
print('$f', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), d['clocks']['reasons'], r.get('bound'), round(r.get('frac') or 0, 4))"; done
