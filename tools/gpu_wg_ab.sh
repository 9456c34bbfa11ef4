# after the tconv WGRAD dead-code removal: generic-path parity, the two re-anchored mutations, the wgrad range A/B
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity_gated.py tests/test_gpu_parity_gconv.py tests/test_gpu_prio.py 2>&1 | tail -2
for m in twgrad_tap_shift_dropped prio_max_priority_not_kept; do timeout 600 python tools/mutation_check.py --only $m 2>&1 | head -1; done
for d in 1 2 4 8; do
  DQN_WG_RANGE_DIV=$d timeout 300 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting > gpurun_out/c5_wg$d.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/c5_wg$d.json') if l.startswith('{')][0]); print('div $d', round(d['value']), round(d['ms_per_step']*1e3,1), d.get('regions_us',{}).get('conv_bwd'))"
done
