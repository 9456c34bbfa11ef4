# tgemm CTAs per SM A/B at BJ.configs[4]
for c in 0 2 1; do
  if [ $c -eq 0 ]; then unset DQN_TG_CTAS; else export DQN_TG_CTAS=$c; fi
  timeout 300 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-acting > gpurun_out/tg$c.json 2> gpurun_out/tg$c.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/tg$c.json') if l.startswith('{')][0]); r=d['regions_us']; print('tg_ctas $c', round(d['value']), round(d['ms_per_step']*1e3,1), r['fc1_fwd'], r['fc1_bwd_head_finish'])"
done
