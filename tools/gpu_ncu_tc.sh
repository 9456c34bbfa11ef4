# ncu --set full of one step's TMA conv kernels (forward, data and weight gradient) at BJ.configs[4]
B5="python bench.py --config c5 --replay 50000 --steps 4 --warmup 3 --e2e-steps 1 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 300 $B5 > /dev/null 2>&1; echo "plain rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:tconv|twgrad' --launch-skip 24 --launch-count 8 -o gpurun_out/tc_r2b $B5 > gpurun_out/tc_r2b.log 2>&1; echo "ncu rc $?"
timeout 600 python -m pytest -q -x tests/test_gpu_replay_dedup.py -m gpu 2>&1 | tail -2
