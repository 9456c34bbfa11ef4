# b=32 (BASELINE.json configs[1]) per-image kernel check: parity of the Mnih path, the bench line, the step timeline
timeout 900 python -m pytest -x -q tests/test_gpu_parity_gated.py tests/test_gpu_parity_bf16.py -m gpu -k "mnih or bf16 or fused" > gpurun_out/b32_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/b32_pytest.log
timeout 300 python bench.py --steps 200 --warmup 20 > gpurun_out/b32_bench.json 2> gpurun_out/b32_bench.err; echo "bench rc $?"; cut -c1-200 gpurun_out/b32_bench.json
DQN_TRACE_STEP=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2> gpurun_out/b32_trace.err > /dev/null; grep timeline gpurun_out/b32_trace.err | tail -1
