#!/bin/bash
# Quick health check of the tree on a B200: GPU suite, default bench line, cfg 2 line.
#   bash tools/gpu_sanity.sh <tag>
set -u
tag=${1:-s}
out=gpurun_out; mkdir -p $out
timeout 2000 python -m pytest tests -m gpu -q -x --durations=10 > $out/pytest_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_$tag.log
tail -14 $out/pytest_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $?" >> $out/bench_$tag.err
timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu --no-attenuated > $out/cfg2_$tag.json 2>> $out/bench_$tag.err
tail -2 $out/bench_$tag.err
