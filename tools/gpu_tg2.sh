timeout 900 python -m pytest tests/test_gpu_parity_gated.py -q -x -k "scaled" 2>&1 | tail -3
timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting --e2e-steps 5 > gpurun_out/bench_c5_tg.json 2> gpurun_out/bench_c5_tg.err; echo "c5 tg rc $?"
python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c5_tg.json') if l.startswith('{')][0]); print('c5', round(d['value']), round(d['ms_per_step']*1e3,1), d['regions_us'])"
B5="python bench.py --config c5 --replay 50000 --steps 10 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tgemm --launch-skip 9 --launch-count 3 -o gpurun_out/tg_full $B5 > gpurun_out/tg_full.log 2>&1; echo "ncu rc $?"
