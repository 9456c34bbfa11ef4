# A/B of the generic path's FC forward split count (DQN_FC_SPLITS_MIN) on BJ.configs[4]: parity, then
# interleaved bench lines (D = 3136: 7 splits of 448, 14 of 224, 28 of 112, 49 of 64)
B="python bench.py --config c5 --replay 50000 --steps 300 --warmup 5 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
for sp in 14 49; do
  DQN_FC_SPLITS_MIN=$sp timeout 600 python -m pytest tests/test_gpu_parity_gconv.py -q -x 2>&1 | tail -1 | sed "s/^/sp=$sp parity: /"
done
for rep in 1 2; do for sp in 1 14 28 49; do
  DQN_FC_SPLITS_MIN=$sp timeout 300 $B > gpurun_out/sp_${sp}_$rep.json 2> gpurun_out/sp_${sp}_$rep.err
  grep "^{" gpurun_out/sp_${sp}_$rep.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('sp=$sp rep=$rep', round(d['value']), round(d['ms_per_step']*1e3,1), d['clocks']['reasons'])"
done; done
