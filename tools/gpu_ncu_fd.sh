#!/bin/bash
# ncu --set full of one forward launch (k_fwd_fd) on cfg ${1:-4}
set -u
out=gpurun_out; mkdir -p $out
cfg=${1:-4}; tag=${2:-fd}
CMD="python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu --no-attenuated"
timeout 600 $CMD > $out/plain_ncu_$tag.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fwd_fd -s 1 -c 1 \
    -o $out/prof_$tag $CMD > $out/ncu_$tag.log 2>&1
echo "ncu exit $?"
tail -3 $out/ncu_$tag.log
