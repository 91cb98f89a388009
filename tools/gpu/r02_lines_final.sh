# every bench line with all legs + the reference arm (no tests / profiling)
OUT=gpurun_out
for c in cfg4 cfg2 cfg3 cfg5; do
  timeout 900 python bench.py --config $c > $OUT/fl_bench_$c.json 2> $OUT/fl_bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > $OUT/fl_ref_cfg4.json 2> $OUT/fl_ref_cfg4.err; echo "ref rc=$?"
