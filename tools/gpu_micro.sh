#!/bin/bash
# Microbenchmarks: pipe / issue rates (tools/issue_peak) and the reduction path (tools/red_peak).
set -u
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > $out/clocks_micro.csv &
CP=$!
timeout 300 ./tools/issue_peak > $out/issue_peak.json 2> $out/issue_peak.err; echo "exit $?" >> $out/issue_peak.err
timeout 120 ./tools/red_peak > $out/red_peak2.json 2>&1
kill $CP
cat $out/issue_peak.json
