# Mnih path after the head-finish change: parity (gated, bf16, full size) + BJ.configs[1] / [3] bench lines
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity_gated.py tests/test_gpu_parity_bf16.py tests/test_gpu_full_size.py tests/test_gpu_parity_fp32.py 2>&1 | tail -1
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-acting 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c2', round(d['value']), round(d['ms_per_step']*1e3,2), d.get('regions_us'))"
timeout 300 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-acting 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c4', round(d['value']), round(d['ms_per_step']*1e3,2), d.get('regions_us'))"
