#!/bin/bash
# NP (ray pairs per lane) experiment: parity of the column kernels and cfg 4/5/3 timing per NP.
set -u
out=gpurun_out; mkdir -p $out
[ -n "${SKIPTEST:-}" ] || XRT_COL_NP=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "column" > $out/pytest_np4.log 2>&1; echo "pytest np4 exit $?"; tail -1 $out/pytest_np4.log
for np in ${NPS:-2 4}; do
  for cfg in 4 5 3; do
    XRT_COL_NP=$np timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-attenuated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('np $np cfg $cfg', round(d['forward']['ms'],2), round(d['adjoint']['ms'],2))"
  done
done
