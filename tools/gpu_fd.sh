#!/bin/bash
# GPU tests, then the forward on the (f, delta f) volume against the legacy k_column forward (cfg 4, 3, 5).
set -u
out=gpurun_out; mkdir -p $out
tag=${1:-fd}
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_$tag.log
tail -3 $out/pytest_$tag.log
for cfg in 4 3 5; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-attenuated > $out/b_${tag}_c$cfg.json 2> $out/b_${tag}_c$cfg.err
  XRT_FWD_LEGACY=1 timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-attenuated > $out/b_${tag}_legacy_c$cfg.json 2>> $out/b_${tag}_c$cfg.err
  python - <<PY
import json
for t in ["$tag", "${tag}_legacy"]:
    try:
        d = json.load(open("$out/b_%s_c$cfg.json" % t))
        print(t, "cfg $cfg", "fwd", d["forward"]["ms"], "adj", d["adjoint"]["ms"], "step", d["ms_per_step"])
    except Exception as e:
        print(t, "cfg $cfg", "failed", e)
PY
done
