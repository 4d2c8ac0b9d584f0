#!/bin/bash
# bench line of every BASELINE config (device timing only; e2e and CPU baseline skipped)
out=gpurun_out; mkdir -p $out
for cfg in 1 2 3 4 5; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu > $out/allcfg_$cfg.json 2>&1
  python -c "
import json
d=json.loads(open('$out/allcfg_$cfg.json').read().strip().split('\n')[-1])
print('cfg $cfg', d['config']['workload'], 'step %.3f ms'%d['ms_per_step'], 'fwd %.3f ms (%.3g int/s, frac %.3f)'%(d['forward']['ms'], d['forward']['intersections_per_s'], d['forward']['roofline_frac']), 'adj %.3f ms (frac %.3f)'%(d['adjoint']['ms'], d['adjoint']['roofline_frac']), 'rays/s %.3g'%d['value'])" || tail -3 $out/allcfg_$cfg.json
done
