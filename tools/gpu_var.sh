#!/bin/bash
# GPU tests (PYTEST=1), then forward timing of library variants: bash tools/gpu_var.sh "cfgs" lib1 lib2 ...
set -u
out=gpurun_out; mkdir -p $out
cfgs=$1; shift
if [ "${PYTEST:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_var.log 2>&1; echo "pytest exit $?" >> $out/pytest_var.log
  tail -3 $out/pytest_var.log
fi
for lib in paper_2006_00686_b200/libxrt.so "$@"; do
  for cfg in $cfgs; do
    XRT_LIB=$lib timeout 300 python tools/time_fwd.py $cfg 5 ${ADJ:-} >> $out/var.log 2>&1 || echo "$lib $cfg failed" >> $out/var.log
  done
done
cat $out/var.log
