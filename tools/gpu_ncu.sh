#!/bin/bash
# One ncu --set full capture: bash tools/gpu_ncu.sh tag cfg skip count [lib]
set -u
tag=$1; cfg=$2; skip=$3; cnt=$4; lib=${5:-paper_2006_00686_b200/libxrt.so}
out=gpurun_out; mkdir -p $out
CMD="python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu"
XRT_LIB=$lib timeout 600 $CMD > $out/plain_$tag.log 2>&1 && \
XRT_LIB=$lib timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_column -s $skip -c $cnt \
    -o $out/prof_$tag $CMD > $out/ncu_$tag.log 2>&1
echo "exit $?" >> $out/ncu_$tag.log
tail -2 $out/ncu_$tag.log
