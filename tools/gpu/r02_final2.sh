# Round-2 evidence with the sparse raw bitmap as the default (split and fused
# launches): GPU suite, smoke, memcheck, launch lists + K1/K1b captures
# (exported to CSV on the box: the reports are too large to copy back), then
# every bench line.
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/f2_gputest.log 2>&1; echo gputest_rc=$?; tail -3 $OUT/f2_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/f2_smoke.log 2>&1; echo smoke_rc=$?; tail -1 $OUT/f2_smoke.log
timeout 900 compute-sanitizer --tool memcheck --leak-check none python tools/sanitize_smoke.py > $OUT/f2_memcheck.log 2>&1; echo memcheck_rc=$?; tail -3 $OUT/f2_memcheck.log
B4="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary"
B2="python bench.py --config cfg2 --steps 2 --warmup 1 --no-e2e --no-cpu"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
timeout -s KILL 900 ncu $M -c 400 --csv --log-file $OUT/r02s_cfg4_launches.csv $B4 > $OUT/r02s_cfg4_launches.log 2>&1; echo ncu4_rc=$?
timeout -s KILL 600 ncu $M -c 400 --csv --log-file $OUT/r02s_cfg2_launches.csv $B2 > $OUT/r02s_cfg2_launches.log 2>&1; echo ncu2_rc=$?
cap() {  # tag kernel bench...
  local tag=$1 k=$2; shift 2
  timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o /tmp/${tag}_prof_$k -f "$@" > $OUT/${tag}_prof_$k.log 2>&1; echo "cap $tag $k rc=$?"
  for pg in details raw; do ncu -i /tmp/${tag}_prof_$k.ncu-rep --page $pg --csv > $OUT/${tag}_prof_$k.$pg.csv; done
  rm -f /tmp/${tag}_prof_$k.ncu-rep
}
cap r02s_cfg4 mask_fg $B4
cap r02s_cfg4 dilate_cells $B4
cap r02s_cfg2 mask_fg $B2
# the traffic records the bench lines read (profiles/ on the box), then back
python tools/summarize_profiles.py r02s_cfg4 1984 profiles/r02_k1_cfg4_traffic.json "Config 4 (BASELINE configs[3]): 64 cameras x 30 4K frames on one GPU, one pass = K1 over 1,920 frames (64 chains + backgrounds = 1,984 frame reads; sparse raw bitmap), K1b, planner + device descriptors, one K5 launch for every invoke event's canvases." > /dev/null; echo sum4_rc=$?
python tools/summarize_profiles.py r02s_cfg2 301 profiles/k1_traffic.json "Config 2 (BASELINE configs[1]): one 4K camera, 300 frames per step (301 frame reads); fused mask launch (K1 + K1b tasks, sparse raw bitmap), planner, K5." > /dev/null; echo sum2_rc=$?
mkdir -p $OUT/prof && cp profiles/r02s_* profiles/r02_k1_cfg4_traffic.json profiles/k1_traffic.json $OUT/prof/
for c in cfg4 cfg2 cfg3 cfg5; do
  timeout 900 python bench.py --config $c > $OUT/f2_bench_$c.json 2> $OUT/f2_bench_$c.err; echo "$c rc=$?"
done
du -sh $OUT
