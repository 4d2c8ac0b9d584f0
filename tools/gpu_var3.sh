#!/bin/bash
set -u
out=gpurun_out; mkdir -p $out
for np in 3 4; do for t in 512 640 384; do
  XRT_COL_NP=$np XRT_LIB=paper_2006_00686_b200/libxrt_np34t$t.so timeout 300 python tools/time_fwd.py 4 5 | sed "s/^/np$np t$t /" >> $out/var.log 2>&1
done; done
cat $out/var.log
