# final check of the committed tree: GPU suite (ids), smoke, mutation check, the N = 1 bench lines that changed
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/r2_pytest_gpu_final.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/r2_pytest_gpu_final.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1; echo "smoke rc $?"
CUDA_VISIBLE_DEVICES=0 timeout 3000 python tools/mutation_check.py > gpurun_out/r2_mutations.txt 2>&1; echo "mutations rc $?"; tail -1 gpurun_out/r2_mutations.txt
export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py > gpurun_out/r2_bench_n1_final.json 2> /dev/null; echo "n1 rc $?"
timeout 900 python bench.py --config c5 --no-acting > gpurun_out/r2_bench_c5_final.json 2> /dev/null; echo "c5 rc $?"
for f in n1_final c5_final; do grep "^{" gpurun_out/r2_bench_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d.get('roofline') or {}
print('$f', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), d['clocks']['reasons'], r.get('bound'), round(r.get('frac') or 0, 4), r.get('traffic'))"; done
