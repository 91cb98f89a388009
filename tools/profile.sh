#!/bin/bash
# Profiling recipe (B200_PROFILING.md): launch list + one full capture per
# hot kernel.  Run under gpurun; outputs land in gpurun_out/.
set -x
OUT=gpurun_out
mkdir -p $OUT
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $B > $OUT/launches.log 2>&1
for k in mask_fg plan_kernel gather_kernel; do
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $OUT/prof_$k -f $B > $OUT/prof_$k.log 2>&1
done
ls -la $OUT
