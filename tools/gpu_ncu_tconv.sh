B5="python bench.py --config c5 --replay 50000 --steps 10 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 300 $B5 > /dev/null 2>&1; echo "plain rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tconv --launch-skip 24 --launch-count 8 -o gpurun_out/tconv_full $B5 > gpurun_out/tconv_full.log 2>&1; echo "ncu rc $?"
