#!/bin/bash
# Round evidence in one gpurun call: GPU tests, the default bench line, the ncu launch list of one
# timed step (our kernels only) and ncu --set full captures of the forward and adjoint kernels.
#   bash tools/gpu_round.sh <tag>      (outputs in gpurun_out/, summarised into profiles/ here)
set -u
tag=${1:-r1}
out=gpurun_out; mkdir -p $out
nvidia-smi > $out/nvsmi_$tag.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $?" >> $out/bench_$tag.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
# launch list: the 4 launches of the timed step (warm-up steps skipped)
timeout 600 $CMD > $out/plain_$tag.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(column|transpose|combine)" -s 12 -c 4 --csv \
    --log-file $out/launches_$tag.csv $CMD > $out/ncu_launches_$tag.log 2>&1
echo "launches exit $?" >> $out/plain_$tag.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_column -s 2 -c 1 \
    -o $out/prof_fwd_$tag $CMD > $out/ncu_fwd_$tag.log 2>&1
echo "full fwd exit $?" >> $out/plain_$tag.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_column -s 3 -c 1 \
    -o $out/prof_adj_$tag $CMD > $out/ncu_adj_$tag.log 2>&1
echo "full adj exit $?" >> $out/plain_$tag.log
cat $out/plain_$tag.log | tail -3
# attenuated transform (N4): one ncu --set full capture of each RAY-family attenuated kernel, cfg 5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(forward|adjoint)_att" -s 2 -c 2 \
    -o $out/prof_att_$tag python tools/time_atten.py 5 1 > $out/ncu_att_$tag.log 2>&1
echo "full att exit $?" >> $out/plain_$tag.log
tail -1 $out/plain_$tag.log
