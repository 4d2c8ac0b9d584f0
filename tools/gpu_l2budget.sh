#!/bin/bash
# adjoint L2 budget sweep (per-operator xy tiling): bash tools/gpu_l2budget.sh "64 160 256"
set -u
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_l2b.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_l2b.log
for mb in ${1:-64 160}; do
  for cfg in 4 5 3; do
    XRT_ADJ_L2_MB=$mb timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-attenuated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('adj budget $mb MB cfg $cfg', round(d['forward']['ms'],2), round(d['adjoint']['ms'],2))"
  done
done
