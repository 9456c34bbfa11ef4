# End-of-round-2 evidence on a 4-GPU box (gpurun --gpus 4): the GPU suite with test ids, smoke, the bench lines
# (N = 1 / 2 / 4 on BJ.configs[1] / [2], configs[0], [3], [4] at N = 1 and N = 2 / 4 for [4]), the reference arm,
# the model-size sweep, and (one GPU) the ncu launch lists + one `ncu --set full` step of the Mnih and generic paths.
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/r2_pytest_gpu.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r2_smoke.log
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n "$@"; }
timeout 900 python bench.py > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo "n1 rc $?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_n1_20.json 2> gpurun_out/r2_bench_n1_20.err; echo "n1 20 rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc $?"
tr 2 > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err; echo "n2 rc $?"
tr 4 > gpurun_out/r2_bench_n4.json 2> gpurun_out/r2_bench_n4.err; echo "n4 rc $?"
timeout 600 python bench.py --config c1 --no-acting > gpurun_out/r2_bench_c1.json 2> gpurun_out/r2_bench_c1.err; echo "c1 rc $?"
timeout 600 python bench.py --config c4 --no-acting > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "c4 rc $?"
tr 4 --config c4 --no-acting > gpurun_out/r2_bench_c4_n4.json 2> gpurun_out/r2_bench_c4_n4.err; echo "c4 n4 rc $?"
timeout 900 python bench.py --config c5 --no-acting > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo "c5 rc $?"
tr 2 --config c5 --no-acting > gpurun_out/r2_bench_c5_n2.json 2> gpurun_out/r2_bench_c5_n2.err; echo "c5 n2 rc $?"
tr 4 --config c5 --no-acting > gpurun_out/r2_bench_c5_n4.json 2> gpurun_out/r2_bench_c5_n4.err; echo "c5 n4 rc $?"
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-acting --prio-alpha 1 > gpurun_out/r2_bench_c2_prio.json 2>/dev/null; echo "prio rc $?"
N=1 bash tools/model_sweep.sh > /dev/null 2>&1; cp gpurun_out/sweep_n1.jsonl gpurun_out/r2_sweep_n1.jsonl
N=4 bash tools/model_sweep.sh > /dev/null 2>&1; cp gpurun_out/sweep_n4.jsonl gpurun_out/r2_sweep_n4.jsonl
for f in n1 n1_20 n2 n4 c1 c4 c4_n4 c5 c5_n2 c5_n4 c2_prio; do grep "^{" gpurun_out/r2_bench_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d.get('roofline') or {}
print('$f', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), d['clocks']['reasons'], r.get('bound'), round(r.get('frac') or 0, 4))"; done
# one GPU from here: ncu passes (each after the plain command exited 0 above)
export CUDA_VISIBLE_DEVICES=0
B2="python bench.py --replay 20000 --steps 10 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
B5="python bench.py --config c5 --replay 50000 --steps 4 --warmup 3 --e2e-steps 1 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 300 $B2 > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c2_launches.csv $B2 > /dev/null 2>&1; echo "c2 list rc $?"
timeout 300 $B5 > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c5_launches.csv $B5 > /dev/null 2>&1; echo "c5 list rc $?"
K2='regex:fwd_conv|tc_gemm|tc_pair|head_sample|bwd_conv|bwd_reduce|reduce_update|rmsprop'
timeout 1200 ncu --set full --import-source on --clock-control none -k "$K2" --launch-skip 60 --launch-count 6 -o gpurun_out/r2_c2_full $B2 > gpurun_out/r2_c2_full.log 2>&1; echo "c2 full rc $?"
K5='regex:gather|tconv|twgrad|tgemm|head|wreduce|rmsprop|chw_to_hwc|gpack'
timeout 1500 ncu --set full --import-source on --clock-control none -k "$K5" --launch-skip 66 --launch-count 22 -o gpurun_out/r2_c5_full $B5 > gpurun_out/r2_c5_full.log 2>&1; echo "c5 full rc $?"
DQN_TRACE_STEP=1 timeout 300 $B2 2> gpurun_out/r2_trace.err > /dev/null; grep timeline gpurun_out/r2_trace.err | tail -1 > gpurun_out/r2_trace_step.txt
