#!/bin/bash
# staged (bulk-copy) forward A/B: parity with XRT_FWD_BULK=1, then cfg 4/5/3 forward timing both ways
set -u
XRT_FWD_BULK=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forward or column or sharding or host or zslab or random" > gpurun_out/pytest_bulk.log 2>&1; echo "pytest bulk exit $?"; tail -3 gpurun_out/pytest_bulk.log
for b in 0 1; do
  for cfg in 4 5 3; do
    XRT_FWD_BULK=$b timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-attenuated 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t); print('bulk $b cfg $cfg', round(d['forward']['ms'],2), round(d['adjoint']['ms'],2))
except Exception: print('bulk $b cfg $cfg FAILED', t[-300:])"
  done
done
