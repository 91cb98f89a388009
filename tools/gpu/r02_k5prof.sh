#!/bin/bash
# K5 (gather_kernel) in the config-4 pipeline: one ncu --set full capture,
# per-line and per-SASS summaries written on the box.
OUT=gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 2 -c 1 -o $OUT/k5 -f $B > $OUT/k5_ncu.log 2>&1; echo ncu rc=$?
python tools/ncu_lines.py $OUT/k5.ncu-rep 45 > $OUT/k5_lines.txt 2>&1
python tools/ncu_hot.py $OUT/k5.ncu-rep 40 > $OUT/k5_hot.txt 2>&1
ncu -i $OUT/k5.ncu-rep --page details --csv > $OUT/k5_details.csv 2>&1
ls -la $OUT/k5.ncu-rep
