#!/bin/bash
set -u
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "host or staged" > $out/pytest_e2e.log 2>&1; echo "pytest exit $?" >> $out/pytest_e2e.log
tail -2 $out/pytest_e2e.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-attenuated > $out/bench_e2e.json 2> $out/bench_e2e.err
python -c "
import json; d=json.load(open('$out/bench_e2e.json')); print('value', d['value'], 'step', d['ms_per_step'], 'e2e', d['e2e'])"
