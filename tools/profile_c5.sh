# configs[4] (scaled net, generic bf16 path): plain bench, then the ncu launch list of the same command
B="python bench.py --config c5 --replay 50000 --steps 20 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline"
timeout 300 $B > gpurun_out/c5_small.json 2> gpurun_out/c5_small.err; rc=$?; echo "c5 small rc $rc"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:gconv|gpack|gemm_pipe|tc_gemm|tc_pair|head_|rmsprop|fc_reduce' \
    --csv --log-file gpurun_out/c5_launches.csv $B > gpurun_out/c5_ncu.log 2>&1; echo "ncu rc $?"
fi
