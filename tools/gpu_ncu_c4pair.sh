# ncu --set full of the Mnih FC backward (tc_pair: dW, dX tiles + head finish) at BJ.configs[3] (b = 256)
B4="python bench.py --config c4 --replay 20000 --steps 10 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 300 $B4 > /dev/null 2>&1; echo "plain rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_pair --launch-skip 5 --launch-count 1 -o gpurun_out/c4_pair $B4 > gpurun_out/c4_pair.log 2>&1; echo "ncu rc $?"
