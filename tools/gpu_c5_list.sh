B5="python bench.py --config c5 --replay 50000 --steps 10 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
timeout 300 $B5 > /dev/null 2> gpurun_out/c5_small.err; rc=$?; echo "c5 small rc $rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv $B5 > /dev/null 2>&1; echo "ncu list rc $?"
  python tools/launches_by_grid.py gpurun_out/c5_launches.csv | head -30
fi
