#!/bin/bash
# Build here, then one GPU pass: gpu tests + per-pattern graph timings + per-CTA trace.
# usage: scripts/gpu_iter.sh [extra remote command]
set -e
cd /root/repo
python -c "from paper_2502_08910_b200 import build; build.build()" 2>&1 | grep -iE "error" && exit 1
HP_TRACE=1 python -c "from paper_2502_08910_b200 import build; build.build()" 2>&1 | grep -iE "error" && exit 1
/usr/local/graft/bin/gpurun --timeout 900 -- "timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/t.log; python scripts/quick_perf.py 1048576 > gpurun_out/qp.log 2>&1; HP_TRACE=1 python scripts/trace_decode.py 1048576 wr > gpurun_out/trace.log 2>&1; $1" 2>&1 | tail -1
cat gpurun_out/t.log gpurun_out/qp.log
