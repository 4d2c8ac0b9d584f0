#!/bin/bash
# Functional check of bench.py's N > 1 step on a 1-GPU box: 2 ranks share the GPU, collectives go
# through gloo on the host (no kernel waits on another rank).  Not a measurement.
set -u
out=gpurun_out; mkdir -p $out
for cfg in ${CFGS:-3 5 4}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $((29500 + cfg)) bench.py --gpus 2 --config $cfg --steps 2 --warmup 3 --no-cpu \
      --no-attenuated --dist-backend gloo > $out/dist_smoke_$cfg.json 2> $out/dist_smoke_$cfg.err
  echo "cfg $cfg exit $?" >> $out/dist_smoke.log
done
cat $out/dist_smoke.log
