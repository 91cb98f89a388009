# Every bench line with all legs, and the reference arm (round-2 evidence).
OUT=gpurun_out
for c in cfg4 cfg2 cfg3 cfg5; do
  python bench.py --config $c > $OUT/r02_bench_$c.json 2> $OUT/r02_bench_$c.err; echo "$c rc=$?"
done
python bench.py --impl reference > $OUT/r02_ref_cfg4.json 2> $OUT/r02_ref_cfg4.err; echo "ref rc=$?"
