# One-GPU evidence for profiles/: the default bench line, a small bench, the ncu launch list of the
# small bench (per-launch gpu__time_duration, serialised, cold-cache) and one `ncu --set full`
# capture of every kernel of one step (+ its raw metrics as CSV). Each ncu pass runs only after its
# command exited 0 plainly. The N > 1 lines come from tools/scale_round.sh (needs gpurun --gpus 4).
set -x
B="python bench.py --replay 20000 --steps 200 --warmup 5 --e2e-steps 5 --profile-steps 20 --no-cpu-baseline --no-acting"
K='regex:fwd_conv|tc_gemm|tc_pair|head_sample|bwd_conv|bwd_reduce|reduce_update|rmsprop|server_round|fused_round'
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,lts__t_sector_hit_rate.pct,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc $?"
timeout 300 $B > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err; rc=$?; echo "small rc $rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc $?"
  timeout 1200 ncu --set full --import-source on --clock-control none -k "$K" --launch-skip 60 --launch-count 6 \
    -o gpurun_out/full $B > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
  ncu -i gpurun_out/full.ncu-rep --page raw --csv --metrics $M > gpurun_out/full_raw.csv 2>/dev/null
  DQN_TRACE_STEP=1 timeout 300 $B 2> gpurun_out/trace_step.err > /dev/null; grep timeline gpurun_out/trace_step.err | tail -1 > gpurun_out/trace_step.txt
fi
