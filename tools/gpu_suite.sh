# the GPU suite with test ids + smoke (gpurun --gpus 4: the world-4 cases run, world-8 skip)
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/r2_pytest_gpu.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/r2_smoke.log
