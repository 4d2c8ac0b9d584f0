timeout 600 python -m pytest tests -m gpu -q -k "adjoint or dot or gather" > gpurun_out/gfail.log 2>&1; grep -E "^FAILED|Error:" gpurun_out/gfail.log | head; tail -1 gpurun_out/gfail.log
CMD="python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu --adj-algo gather"
timeout 600 $CMD > gpurun_out/gplain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather -s 3 -c 1 -o gpurun_out/prof_gather5 $CMD > gpurun_out/ncu_gather.log 2>&1; tail -1 gpurun_out/ncu_gather.log
