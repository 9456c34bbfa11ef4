for l in 1 2 3; do timeout 60 tools/probe_tconv $l 512 20; done
timeout 600 python -m pytest tests/test_gpu_parity_gated.py tests/test_gpu_parity_gconv.py -x -q -k scaled --timeout 120 2>&1 | tail -3
