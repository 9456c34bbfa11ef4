# ncu launch list (per-launch durations, cold, serialised) of a short bench run: bash tools/gpu_list.sh c4 [extra bench args]
C=$1; shift
B="python bench.py --config $C --steps 10 --warmup 3 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline $*"
timeout 300 $B > /dev/null 2> gpurun_out/${C}_small.err; rc=$?; echo "$C small rc $rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none ${NCU_CACHE:+--cache-control $NCU_CACHE} --csv --log-file gpurun_out/${C}_launches.csv $B > /dev/null 2>&1; echo "ncu list rc $?"
  python tools/launches_by_grid.py gpurun_out/${C}_launches.csv | head -30
fi
