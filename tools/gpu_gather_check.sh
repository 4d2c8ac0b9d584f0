timeout 900 python -m pytest tests -m gpu -x -q -k "adjoint or dot or gather" 2>&1 | tail -3
for cfg in 5 3 4; do timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu --adj-algo gather > gpurun_out/g_$cfg.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/g_$cfg.json').read().strip().split('\n')[-1]); print($cfg, 'fwd', d['forward']['ms'], 'adj(gather)', d['adjoint']['ms'])" || tail -5 gpurun_out/g_$cfg.json; done
