#!/bin/bash
# B200 die map of device buffers (tools/die_map): block homes seen from two SMs
set -u
out=gpurun_out; mkdir -p $out
timeout 120 ./tools/die_map 64 4096 0 147 > $out/die_4k_0_147.txt 2>&1
timeout 120 ./tools/die_map 2 256 0 147 > $out/die_256_0_147.txt 2>&1
timeout 120 ./tools/die_map 64 4096 0 1 > $out/die_4k_0_1.txt 2>&1
timeout 120 ./tools/die_map 64 4096 0 74 > $out/die_4k_0_74.txt 2>&1
for f in $out/die_*.txt; do echo "$f"; head -1 $f; awk 'NR>1{a+=$2; b+=$3; n++} END{print "meanA", a/n, "meanB", b/n}' $f; done
