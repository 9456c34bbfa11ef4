# generic-path evidence: BJ.configs[3] and [4] bench lines, the c5 launch list and one ncu --set full capture
# of the heaviest generic-path kernels (each ncu pass only after the plain command exited 0)
B5="python bench.py --config c5 --replay 50000 --steps 20 --warmup 3 --e2e-steps 3 --profile-steps 5 --no-cpu-baseline --no-acting"
timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc $?"
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-acting > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc $?"
timeout 300 $B5 > /dev/null 2> gpurun_out/c5_small.err; rc=$?; echo "c5 small rc $rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv $B5 > /dev/null 2>&1; echo "ncu list rc $?"
  timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:gconv_wgrad|gconv_fwd|gconv_dgrad|tc_pair|gemm_pipe' \
    --launch-skip 30 --launch-count 10 -o gpurun_out/c5_full $B5 > gpurun_out/c5_full.log 2>&1; echo "ncu full rc $?"
fi
