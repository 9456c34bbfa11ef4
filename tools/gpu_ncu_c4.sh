# one ncu --set full capture of the Mnih conv backward at b = 256 (BJ.configs[3])
B4="python bench.py --config c4 --replay 50000 --steps 4 --warmup 3 --e2e-steps 1 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 300 $B4 > /dev/null 2>&1; echo "plain rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bwd_conv --launch-skip 3 --launch-count 1 -o gpurun_out/c4_bwd $B4 > gpurun_out/c4_bwd.log 2>&1; echo "ncu rc $?"
