#!/bin/bash
# Timing of environment variants of the default library: bash tools/gpu_env.sh "cfgs" "ENV=1 ..." "ENV2=..." ...
# (the first run is always the default environment; CUDA events, tools/time_fwd.py)
set -u
out=gpurun_out; mkdir -p $out
cfgs=$1; shift
for envs in "" "$@"; do
  for cfg in $cfgs; do
    echo "env: ${envs:-default}" >> $out/env.log
    env $envs timeout 300 python tools/time_fwd.py $cfg 5 ${ADJ:-} >> $out/env.log 2>&1 || echo "$envs $cfg failed" >> $out/env.log
  done
done
cat $out/env.log
