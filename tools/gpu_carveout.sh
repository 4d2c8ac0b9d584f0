#!/bin/bash
# shared-memory carveout sweep of the column kernels (XRT_CARVEOUT percent; unset = driver default)
set -u
for cv in default ${CVS:-0 25 50 100}; do
  for cfg in 4 5; do
    if [ $cv = default ]; then unset XRT_CARVEOUT; else export XRT_CARVEOUT=$cv; fi
    timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-attenuated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('carveout $cv cfg $cfg', round(d['forward']['ms'],2), round(d['adjoint']['ms'],2))"
  done
done
