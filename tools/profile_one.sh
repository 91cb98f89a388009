#!/bin/bash
# Full ncu capture of one kernel (regex $1) of the bench, output gpurun_out/prof_$2
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s 1 -c 1 -o gpurun_out/prof_$2 -f $B > gpurun_out/prof_$2.log 2>&1
