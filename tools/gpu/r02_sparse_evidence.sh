# Sparse raw bitmap as the build default: GPU suite (incl. the stale-bitmap
# split-path cases), same-box A/B vs the dense variant, the config-4 launch
# list + K1/K1b captures, then the config-4 and config-3 bench lines.
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/se_gputest.log 2>&1; echo gputest_rc=$?; tail -3 $OUT/se_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/se_smoke.log 2>&1; echo smoke_rc=$?; tail -1 $OUT/se_smoke.log
bash tools/gpu/cfg4_lib_ms.sh default dense 2>&1
unset TANGRAM_GPU_LIB
B4="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
timeout -s KILL 900 ncu $M -c 400 --csv --log-file $OUT/r02s_cfg4_launches.csv $B4 > $OUT/r02s_cfg4_launches.log 2>&1; echo ncu_list_rc=$?
for k in mask_fg dilate_cells; do
  timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o $OUT/r02s_cfg4_prof_$k -f $B4 > $OUT/r02s_cfg4_prof_$k.log 2>&1; echo ncu_$k=$?
done
timeout 900 python bench.py > $OUT/se_bench_cfg4.json 2> $OUT/se_bench_cfg4.err; echo cfg4_rc=$?
timeout 900 python bench.py --config cfg3 > $OUT/se_bench_cfg3.json 2> $OUT/se_bench_cfg3.err; echo cfg3_rc=$?
