#!/bin/bash
# A/B of RAY-family kernels (plain + attenuated) for lib variants: bash tools/gpu_ab_ray.sh lib...
set -u
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_abray.log 2>&1; echo "pytest exit $?" >> $out/pytest_abray.log
tail -2 $out/pytest_abray.log
for lib in "$@"; do
  for c in 1 2 5 4; do
    echo -n "$lib "; XRT_LIB=$lib timeout 300 python tools/time_atten.py $c 3
  done
done
