#!/bin/bash
# ncu --set full of one k_fwd_fd launch with library variant $1 (tag $2), cfg ${3:-4}
set -u
out=gpurun_out; mkdir -p $out
lib=$1; tag=$2; cfg=${3:-4}
export XRT_LIB=$lib
CMD="python tools/time_fwd.py $cfg 1"
timeout 600 $CMD > $out/plain_ncu_$tag.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fwd_fd -s 2 -c 1 \
    -o $out/prof_$tag $CMD > $out/ncu_$tag.log 2>&1
echo "ncu exit $?"
