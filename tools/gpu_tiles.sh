#!/bin/bash
# time cfg4 forward/adjoint for tile-size overrides and lib variants
set -u
out=gpurun_out; mkdir -p $out
for lib in ${LIBS:-paper_2006_00686_b200/libxrt.so}; do
  for tile in ${TILES:-default 256 4096}; do
    if [ $tile = default ]; then unset XRT_COLUMN_TILE; else export XRT_COLUMN_TILE=$tile; fi
    f=$out/tiles_$(basename $lib .so)_$tile.json
    XRT_LIB=$lib timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu > $f 2>&1
    python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().split('\n')[-1]); print('$lib','tile $tile','fwd %.2f adj %.2f'%(d['forward']['ms'],d['adjoint']['ms']))
except Exception: print('$lib tile $tile FAILED', open('$f').read()[-400:])"
  done
done
unset XRT_COLUMN_TILE
