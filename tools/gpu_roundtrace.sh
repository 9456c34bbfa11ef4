# fused-round phase trace on BJ.configs[2] (N = 2, 4 when present): block spread at barrier A, conv release
NG=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -le $NG ] || continue
  N=$n bash tools/trace_comm.sh > /dev/null 2>&1
  echo "N=$n"; grep -E "fused round \(6|relative to|next fwd" gpurun_out/trace.log | head -6
done
