#!/bin/bash
# Per-launch times of K1 (mask_fg) and K1b (dilate_cells) of a short bench run.
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:mask_fg|dilate' -c 6 --csv --log-file gpurun_out/k1_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/k1_launches.log 2>&1
grep -E 'duration' gpurun_out/k1_launches.csv | awk -F'","' '{print $5, $(NF)}'
