#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the ncu launch list and one full capture
# of the top kernel. Usage (from the repo root, on the GPU box):  bash tools/gpu_profile.sh [tag]
set -u
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
nvidia-smi > $out/nvsmi_$tag.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $?" >> $out/bench_$tag.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $out/plain_$tag.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_$tag.csv $CMD > $out/ncu_launches_$tag.log 2>&1
echo "launches exit $?" >> $out/plain_$tag.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_column -s 2 -c 2 \
    -o $out/prof_$tag $CMD > $out/ncu_full_$tag.log 2>&1
echo "full exit $?" >> $out/plain_$tag.log
