# Mnih path at large b (BJ.configs[3]): parity (gated b256, async, full size, bf16), then the c4 bench line
timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_parity_gated.py tests/test_gpu_async.py tests/test_gpu_full_size.py tests/test_gpu_parity_bf16.py 2>&1 | tail -3
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-acting > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc $?"
python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c4.json') if l.startswith('{')][0]); print('c4', round(d['value']), round(d['ms_per_step']*1e3,1), d.get('regions_us'))"
