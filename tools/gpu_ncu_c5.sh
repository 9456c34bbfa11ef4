# one ncu --set full capture of every repo kernel of one BJ.configs[4] step (after the plain command exits 0)
B5="python bench.py --config c5 --replay 50000 --steps 4 --warmup 3 --e2e-steps 1 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 300 $B5 > /dev/null 2> gpurun_out/c5_small.err; rc=$?; echo "c5 small rc $rc"
if [ $rc -eq 0 ]; then
  timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:gather|tconv|twgrad|tgemm|head|wreduce|rmsprop' \
    --launch-skip 60 --launch-count 20 -o gpurun_out/c5_r2_full $B5 > gpurun_out/c5_r2_full.log 2>&1; echo "ncu full rc $?"
fi
