#!/bin/bash
# ncu captures for profiles/: the decode kernels at C3 (1M) and the tcgen05 prefill kernel.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'decode_(stage_wide|stage_allrows|stage_look|stage_kernel|topk|bsa)' -s 7 -c 7 \
   -o gpurun_out/prof_decode_final -f python scripts/quick_perf.py 1048576 --ncu > gpurun_out/prof_decode_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bsa_prefill_tc' -c 1 \
   -o gpurun_out/prof_prefill_final -f python scripts/prefill_bench.py 131072 32768 > gpurun_out/prof_prefill_final.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
     python bench.py --steps 2 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
echo done
