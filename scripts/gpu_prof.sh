#!/bin/bash
# ncu full capture of the fused decode kernels at C3 (1M ctx), one launch each of
# stage-1/2/3 descents, the three top-k selections and the BSA (first warm-up step).
mkdir -p gpurun_out
tag=${1:-prof}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'decode_(stage|topk|bsa)' -s 7 -c 7 \
   -o gpurun_out/$tag -f python scripts/quick_perf.py 1048576 --ncu > gpurun_out/${tag}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}.log
