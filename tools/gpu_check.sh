# GPU check of the committed tree: the GPU suite (ids logged), the driver's bench command and the long one, smoke
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1_20.json 2> gpurun_out/bench_n1_20.err; echo "N=1 20 rc $?"
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "N=1 rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
