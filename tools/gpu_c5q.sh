# generic path quick check: parity of the scaled-net cases (gated + gconv + dedup), then the c5 bench line
timeout 900 python -m pytest tests/test_gpu_parity_gated.py tests/test_gpu_parity_gconv.py tests/test_gpu_replay_dedup.py -q -x -m gpu 2>&1 | tail -4
timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting --e2e-steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc $?"
python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c5.json') if l.startswith('{')][0]); print('c5', round(d['value']), round(d['ms_per_step']*1e3,1), d.get('regions_us'))"
