timeout 300 python -m pytest tests/test_gpu_parity_gated.py -q -x -k "scaled-b32" 2>&1 | grep -E "Error|error|assert" | head -8
