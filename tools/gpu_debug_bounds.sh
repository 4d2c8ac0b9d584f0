#!/bin/bash
# The GPU suite against a bounds-checking build (-DXRT_DEBUG_BOUNDS=1: every walk load and adjoint
# reduction address checked against the buffer its launch walks; a miss prints and traps).
# Build it first here:  python -c "from paper_2006_00686_b200 import build; build.build(out='paper_2006_00686_b200/libxrt_dbg.so', defines=['XRT_DEBUG_BOUNDS=1'])"
set -u
out=gpurun_out; mkdir -p $out
XRT_LIB=paper_2006_00686_b200/libxrt_dbg.so timeout 1800 python -m pytest tests -m gpu -q -x > $out/pytest_dbg.log 2>&1
echo "exit $?" >> $out/pytest_dbg.log
tail -3 $out/pytest_dbg.log
