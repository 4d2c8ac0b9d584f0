#!/bin/bash
# cfg 1 / 2 (2D) timing for lib variants: bash tools/gpu_cfg2.sh lib...
for lib in paper_2006_00686_b200/libxrt.so "$@"; do
  for cfg in 2 1; do
    XRT_LIB=$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-attenuated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib cfg $cfg', round(d['forward']['ms'],4), round(d['adjoint']['ms'],4))"
  done
done
