# BJ.configs[3] (Mnih, b = 256): step timeline (CTA 0 stamps) + ncu launch list with warm caches
DQN_TRACE_STEP=1 timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline --no-acting > gpurun_out/c4t.json 2> gpurun_out/c4t.err
echo "trace rc $?"; grep "step timeline" gpurun_out/c4t.err | tail -1
NCU_CACHE=none bash tools/gpu_list.sh c4
