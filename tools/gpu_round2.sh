#!/bin/bash
# Round-2 evidence in one gpurun call: GPU tests, the default bench line and the all-config lines,
# the ncu launch list of one timed step (our kernels), ncu --set full of the forward (k_fwd_fd) and
# the adjoint (k_column<1,1>), and the pipe / reduction microbenchmarks.
#   bash tools/gpu_round2.sh <tag>
set -u
tag=${1:-r2}
out=gpurun_out; mkdir -p $out
nvidia-smi > $out/nvsmi_$tag.txt 2>&1
nproc > $out/nproc_$tag.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu_$tag.log
tail -3 $out/pytest_gpu_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $?" >> $out/bench_$tag.err
for c in 1 2 3 5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $out/allcfg_${tag}_$c.json 2>> $out/bench_$tag.err
done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-attenuated"
timeout 600 $CMD > $out/plain_$tag.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(column|fwd_fd|to_fd|transpose|slice|forward_ray|fd2d)" -s 12 -c 4 --csv \
    --log-file $out/launches_$tag.csv $CMD > $out/ncu_launches_$tag.log 2>&1
echo "launches exit $?" >> $out/plain_$tag.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fwd_fd -s 1 -c 1 \
    -o $out/prof_fwd_$tag $CMD > $out/ncu_fwd_$tag.log 2>&1
echo "full fwd exit $?" >> $out/plain_$tag.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_column -s 1 -c 1 \
    -o $out/prof_adj_$tag $CMD > $out/ncu_adj_$tag.log 2>&1
echo "full adj exit $?" >> $out/plain_$tag.log
timeout 300 ./tools/issue_peak > $out/issue_peak_$tag.json 2>&1
timeout 120 ./tools/red_peak > $out/red_peak_$tag.json 2>&1
tail -4 $out/plain_$tag.log
