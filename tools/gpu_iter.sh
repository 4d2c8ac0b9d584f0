#!/bin/bash
# Quick GPU iteration: column-path parity tests + forward/adjoint timing of lib variants.
# usage: bash tools/gpu_iter.sh tag [lib variants...]
set -u
tag=$1; shift
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_$tag.log
tail -3 $out/pytest_$tag.log
for lib in paper_2006_00686_b200/libxrt.so "$@"; do
  for cfg in 4 5 3; do
    XRT_LIB=$lib timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu > $out/bench_${tag}_$(basename $lib .so)_c$cfg.json 2>&1
    python - "$out/bench_${tag}_$(basename $lib .so)_c$cfg.json" "$lib" $cfg <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().split('\n')[-1])
    print(sys.argv[2], 'cfg', sys.argv[3], 'fwd %.2f ms adj %.2f ms' % (d['forward']['ms'], d['adjoint']['ms']), 'clk', d['clocks']['sm_mhz'])
except Exception as e:
    print(sys.argv[2], 'cfg', sys.argv[3], 'FAILED', open(sys.argv[1]).read()[-500:])
PY
  done
done
