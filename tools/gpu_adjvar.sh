#!/bin/bash
# adjoint A/B: default lib + variants, and the NP=2 adjoint (XRT_COL_NP_ADJ=2) for the last lib
set -u
out=gpurun_out; mkdir -p $out; : > $out/adjvar.log
for lib in paper_2006_00686_b200/libxrt.so "$@"; do
  for cfg in 4 5; do
    XRT_LIB=$lib timeout 300 python tools/time_fwd.py $cfg 3 adj >> $out/adjvar.log 2>&1
  done
done
for cfg in 4 5; do
  XRT_COL_NP_ADJ=2 XRT_LIB=${!#} timeout 300 python tools/time_fwd.py $cfg 3 adj | sed 's/"lib"/"np_adj2_lib"/' >> $out/adjvar.log 2>&1
done
cat $out/adjvar.log
