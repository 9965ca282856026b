#!/bin/bash
# Final round-2 profiles (run under gpurun): launch list of the bench command and one
# ncu --set full capture each of the stage-1 one-wave kernel and the fused layer kernel.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ext --no-offload > gpurun_out/r2f_launch_bench.log 2>&1
echo "launch list rc=$?" >> gpurun_out/r2f_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'decode_(stage_wide|layer)' -s 4 -c 2 \
   -o gpurun_out/r2f_prof -f python scripts/quick_perf.py 1048576 --ncu > gpurun_out/r2f_prof.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2f_prof.log
python scripts/ncu_summary.py gpurun_out/r2f_prof.ncu-rep > gpurun_out/r2f_ncu_summary.txt 2>&1
python scripts/launch_summary.py gpurun_out/r2f_launches.csv "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ext --no-offload" > gpurun_out/r2f_launches_summary.txt 2>&1
ls -la gpurun_out | tail -8
