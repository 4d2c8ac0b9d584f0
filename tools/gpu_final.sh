#!/bin/bash
# Final evidence of a round: all-config lines, ncu launch list of one timed step, ncu --set full of the
# forward (with its per-block account taken here).  bash tools/gpu_final.sh <tag>
set -u
tag=${1:-final}
out=gpurun_out; mkdir -p $out
for c in 1 2 3 5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $out/allcfg_${tag}_$c.json 2>> $out/final_$tag.err
done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-attenuated"
timeout 600 $CMD > $out/plain_$tag.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(column|fwd_fd|to_fd|transpose)" -s 12 -c 4 --csv \
    --log-file $out/launches_$tag.csv $CMD > $out/ncu_launches_$tag.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fwd_fd -s 1 -c 1 \
    -o $out/prof_fwd_$tag $CMD > $out/ncu_fwd_$tag.log 2>&1
echo "done" >> $out/plain_$tag.log
