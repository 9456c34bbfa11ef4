# Last refresh of round 2 on a 4-GPU box: the GPU suite with test ids + smoke, and the BJ.configs[3] lines
# (N = 1 and 4) after the bulk reduce-add epilogue
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/r2_pytest_gpu.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/r2_smoke.log
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n "$@"; }
timeout 600 python bench.py --config c4 --no-acting > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "c4 rc $?"
tr 4 --config c4 --no-acting > gpurun_out/r2_bench_c4_n4.json 2> gpurun_out/r2_bench_c4_n4.err; echo "c4 n4 rc $?"
for f in c4 c4_n4; do grep "^{" gpurun_out/r2_bench_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d.get('roofline') or {}
print('$f', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), d['clocks']['reasons'], r.get('bound'), round(r.get('frac') or 0, 4), d.get('regions_us'))"; done
