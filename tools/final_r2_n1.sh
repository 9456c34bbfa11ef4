# Refresh after the Store moved into the conv forward: the GPU suite with test ids + smoke (2 GPUs: world-4/8
# cases skip) and the N = 1 BJ.configs[1] lines (default and the driver's 20 steps)
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/r2_pytest_gpu_2gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/r2_pytest_gpu_2gpu.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo "n1 rc $?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_n1_20.json 2> gpurun_out/r2_bench_n1_20.err; echo "n1 20 rc $?"
for f in n1 n1_20; do grep "^{" gpurun_out/r2_bench_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d.get('roofline') or {}
print('$f', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), round(d['e2e']['sync_per_step']['value']), d['clocks'], r.get('bound'), round(r.get('frac') or 0, 4), d.get('gpu_launches'))"; done
