# Round-2 evidence at HEAD: the GPU test suite, every bench line with all legs,
# the reference arm, then the profiling recipe (launch lists + set-full captures).
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/ev_smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/ev_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/ev_pytest.log
for c in cfg4 cfg2 cfg3 cfg5; do
  timeout 900 python bench.py --config $c > $OUT/ev_bench_$c.json 2> $OUT/ev_bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > $OUT/ev_ref_cfg4.json 2> $OUT/ev_ref_cfg4.err; echo "ref rc=$?"
bash tools/gpu/r02_profile.sh > $OUT/ev_profile.log 2>&1; echo "profile rc=$?"
