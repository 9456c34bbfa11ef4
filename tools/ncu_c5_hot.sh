# one `ncu --set full` capture of the generic path's heaviest kernels (after a plain run exited 0)
B="python bench.py --config c5 --replay 50000 --steps 20 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline"
timeout 300 $B > /dev/null 2>&1; rc=$?; echo "plain rc $rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:gconv_wgrad|gconv_fwd|tc_pair' \
    --launch-skip 24 --launch-count 6 -o gpurun_out/c5_hot $B > gpurun_out/c5_hot.log 2>&1; echo "ncu rc $?"
fi
