#!/bin/bash
# N > 1 correctness through libxrt on a 1-GPU box (tools/dist_check.py, gloo, 2 ranks share the GPU)
set -u
out=gpurun_out; mkdir -p $out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NPROC:-2} --master-addr 127.0.0.1 \
    --master-port 29611 tools/dist_check.py > $out/dist_check.json 2> $out/dist_check.err
echo "exit $?" >> $out/dist_check.json
cat $out/dist_check.json
