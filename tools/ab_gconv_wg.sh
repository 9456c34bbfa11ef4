# A/B of the generic weight-gradient grid (DQN_GCONV_WG_CTAS) on BJ.configs[4]: parity, then interleaved bench lines
B="python bench.py --config c5 --replay 50000 --steps 300 --warmup 5 --e2e-steps 2 --profile-steps 0 --no-cpu-baseline --no-acting"
for w in 592 888; do
  DQN_GCONV_WG_CTAS=$w timeout 600 python -m pytest tests/test_gpu_parity_gconv.py -q -x 2>&1 | tail -1 | sed "s/^/wg=$w parity: /"
done
for rep in 1 2; do for w in 296 444 592 888 1184; do
  DQN_GCONV_WG_CTAS=$w timeout 300 $B > gpurun_out/wg_${w}_$rep.json 2> gpurun_out/wg_${w}_$rep.err
  grep "^{" gpurun_out/wg_${w}_$rep.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('wg=$w rep=$rep', round(d['value']), round(d['ms_per_step']*1e3,1), d['clocks']['reasons'])"
done; done
