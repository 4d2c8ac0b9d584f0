#!/bin/bash
# Default bench line (cfg 4) and the all-config lines: bash tools/gpu_bench.sh tag [cfgs]
set -u
out=gpurun_out; mkdir -p $out
tag=${1:-b}; cfgs=${2:-"1 2 3 5"}
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $?" >> $out/bench_$tag.err
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $out/allcfg_${tag}_$c.json 2>> $out/bench_$tag.err
done
python - $tag "$cfgs" <<'PY'
import json, sys
tag = sys.argv[1]
for f in [f"gpurun_out/bench_{tag}.json"] + [f"gpurun_out/allcfg_{tag}_{c}.json" for c in sys.argv[2].split()]:
    try:
        d = json.loads(open(f).read().strip().split("\n")[-1])
        print(d["config"]["workload"], "step %.3f ms" % d["ms_per_step"], "fwd %.3f" % d["forward"]["ms"], "adj %.3f" % d["adjoint"]["ms"],
              "value %.3e" % d["value"], "frac %.3f" % d["roofline"]["frac"], "e2e %.3e" % d.get("e2e", {}).get("value", 0),
              "cpu", d.get("cpu_baseline", {}).get("value"), d.get("cpu_baseline", {}).get("cores"), "clk", d["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "FAILED", e)
PY
tail -5 $out/bench_$tag.err
