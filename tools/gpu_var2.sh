#!/bin/bash
set -u
out=gpurun_out; mkdir -p $out
for lib in paper_2006_00686_b200/libxrt.so paper_2006_00686_b200/libxrt_w8.so paper_2006_00686_b200/libxrt_w16.so paper_2006_00686_b200/libxrt_fdm8.so; do
  XRT_LIB=$lib timeout 300 python tools/time_fwd.py 4 5 >> $out/var.log 2>&1
done
XRT_COL_NP=1 timeout 300 python tools/time_fwd.py 4 5 >> $out/var.log 2>&1
XRT_COL_NP=1 XRT_LIB=paper_2006_00686_b200/libxrt_w8.so timeout 300 python tools/time_fwd.py 4 5 >> $out/var.log 2>&1
cat $out/var.log
