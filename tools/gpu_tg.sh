timeout 900 python -m pytest tests/test_gpu_parity_gated.py tests/test_gpu_parity_gconv.py tests/test_gpu_parity_bf16.py -q -x 2>&1 | tail -15
timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting --e2e-steps 5 > gpurun_out/bench_c5_tg.json 2> gpurun_out/bench_c5_tg.err; echo "c5 tg rc $?"
DQN_TGEMM=0 timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting --e2e-steps 5 > gpurun_out/bench_c5_old.json 2> gpurun_out/bench_c5_old.err; echo "c5 old rc $?"
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-acting --e2e-steps 5 > gpurun_out/bench_n1_short.json 2>&1; echo "n1 rc $?"
for f in bench_c5_tg bench_c5_old bench_n1_short; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/$f.json') if l.startswith('{')][0]); print('$f', round(d['value']), round(d['ms_per_step']*1e3,1), d['regions_us'])"; done
