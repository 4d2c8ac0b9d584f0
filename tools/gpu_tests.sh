#!/bin/bash
# The GPU test suite with per-test durations: bash tools/gpu_tests.sh [tag] [pytest args...]
set -u
out=gpurun_out; mkdir -p $out
tag=${1:-t}; shift || true
nproc > $out/nproc_$tag.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=25 "$@" > $out/pytest_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_$tag.log
tail -45 $out/pytest_$tag.log
