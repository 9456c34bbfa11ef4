# Model-size sweep (BJ.c5; the paper's Fig. 3 axis): transitions/s and the per-step
# gradient time T, update/round time tau per model size, at N = ${N:-1} GPUs. One JSON line per point in
# gpurun_out/sweep_n$N.jsonl; tools/model_sweep_table.py turns them into a table.
N=${N:-1}
out=gpurun_out/sweep_n$N.jsonl; : > $out
run() {
  if [ $N -eq 1 ]; then timeout 600 python bench.py "$@" 2>/dev/null | grep "^{" >> $out
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
         --master-port 29633 bench.py --gpus $N "$@" 2>/dev/null | grep "^{" >> $out; fi
}
C="--steps 300 --warmup 10 --replay 100000 --e2e-steps 10 --profile-steps 40 --no-cpu-baseline --no-acting"
for fc in 128 256 512; do run --config c2 --fc $fc $C; done  # Mnih stack, b = 32 (tc_pair stages (128 + b) fc 2 B <= 200 KB)
for fc in 512 1024 2048; do run --config c5 --fc $fc $C; done  # scaled net, b = 512: the TMA GEMMs take any fc
cat $out | cut -c1-200
