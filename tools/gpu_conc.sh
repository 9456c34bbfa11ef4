# two-branch conv backward: generic-path parity, then the A/B at BJ.configs[4]
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity_gated.py tests/test_gpu_parity_gconv.py tests/test_gpu_full_size.py tests/test_gpu_replay_dedup.py tests/test_gpu_prio.py 2>&1 | tail -2
for cb in 1 0; do
  DQN_CONC_BWD=$cb timeout 300 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting > gpurun_out/c5_cb$cb.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/c5_cb$cb.json') if l.startswith('{')][0]); r=d.get('regions_us',{}); print('conc $cb', round(d['value']), round(d['ms_per_step']*1e3,1), r.get('conv_bwd'))"
done
