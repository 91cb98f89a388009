# Round-2 profiling recipe (B200_PROFILING.md), run under gpurun: launch
# lists (device time + DRAM bytes of every launch) of the default bench
# (config 4) and of config 2, then one --set full capture per hot kernel.
OUT=gpurun_out
B4="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary"
B2="python bench.py --config cfg2 --steps 2 --warmup 1 --no-e2e --no-cpu"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
timeout -s KILL 900 ncu $M -c 400 --csv --log-file $OUT/r02_cfg4_launches.csv $B4 > $OUT/r02_cfg4_launches.log 2>&1
timeout -s KILL 600 ncu $M -c 400 --csv --log-file $OUT/r02_cfg2_launches.csv $B2 > $OUT/r02_cfg2_launches.log 2>&1
for k in mask_fg dilate_cells plan_kernel gather_kernel; do
  timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o $OUT/r02_cfg4_prof_$k -f $B4 > $OUT/r02_cfg4_prof_$k.log 2>&1
done
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:mask_fg -s 1 -c 1 \
  -o $OUT/r02_cfg2_prof_mask_fg -f $B2 > $OUT/r02_cfg2_prof_mask_fg.log 2>&1
ls -la $OUT | grep r02_
