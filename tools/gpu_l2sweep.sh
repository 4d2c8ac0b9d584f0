#!/bin/bash
# L2 budget sweep of the xy tiling (forward / adjoint), cfg 4: bash tools/gpu_l2sweep.sh
for f in 40 96; do XRT_FWD_L2_MB=$f timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-attenuated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fwd budget $f', round(d['forward']['ms'],2), round(d['adjoint']['ms'],2))"; done
for a in 40 96; do XRT_ADJ_L2_MB=$a timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-attenuated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('adj budget $a', round(d['forward']['ms'],2), round(d['adjoint']['ms'],2))"; done
