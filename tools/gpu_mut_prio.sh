# mutation check of the GPU parity suite + the prioritized variant's bench lines
timeout 3000 python tools/mutation_check.py > gpurun_out/mutations.txt 2>&1; echo "mutations rc $?"; tail -3 gpurun_out/mutations.txt
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-acting --prio-alpha 1 > gpurun_out/bench_c2_prio.json 2> gpurun_out/bench_c2_prio.err; echo "c2 prio rc $?"; cut -c1-200 gpurun_out/bench_c2_prio.json
timeout 300 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting --prio-alpha 1 > gpurun_out/bench_c5_prio.json 2> gpurun_out/bench_c5_prio.err; echo "c5 prio rc $?"; cut -c1-200 gpurun_out/bench_c5_prio.json
