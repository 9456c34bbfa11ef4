timeout 900 python -m pytest tests/test_gpu_parity_gated.py tests/test_gpu_parity_gconv.py -q -x -k "scaled" 2>&1 | tail -4
timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting --e2e-steps 5 > gpurun_out/bench_c5_tc.json 2> gpurun_out/bench_c5_tc.err; echo "c5 rc $?"
python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c5_tc.json') if l.startswith('{')][0]); print('c5', round(d['value']), round(d['ms_per_step']*1e3,1), d['regions_us'])"
B5="python bench.py --config c5 --replay 50000 --steps 10 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv $B5 > /dev/null 2>&1; echo "ncu list rc $?"
python tools/launches_by_grid.py gpurun_out/c5_launches.csv 2>/dev/null | grep dqn | head -20
