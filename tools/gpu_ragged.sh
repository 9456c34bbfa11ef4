set -x
timeout 900 python -m pytest tests/test_gpu_parity_gated.py tests/test_gpu_parity_fp32.py tests/test_gpu_prio.py tests/test_gpu_branches.py -m gpu -q -rA -x 2>&1 | tail -60 > gpurun_out/ragged_pytest.log
