#!/bin/bash
# ncu --set full of the cfg 2 (2D fan) forward and adjoint kernels (AUTO), one launch each
set -u
out=gpurun_out; mkdir -p $out
CMD="python tools/time_2d.py"
timeout 600 $CMD > $out/plain_cfg2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_slice2d_v2" -s 2 -c 2 \
    -o $out/prof_cfg2 $CMD > $out/ncu_cfg2.log 2>&1
echo "ncu exit $?"; tail -2 $out/ncu_cfg2.log
