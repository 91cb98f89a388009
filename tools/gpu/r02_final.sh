# Round-2 evidence run: compute-sanitizer (memcheck, synccheck) on the smoke
# paths, then every bench line with all legs and the reference arm.
OUT=gpurun_out
timeout 900 compute-sanitizer --tool memcheck --leak-check none python tools/sanitize_smoke.py > $OUT/r02_memcheck.log 2>&1; echo memcheck_rc=$?; tail -3 $OUT/r02_memcheck.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_smoke.py > $OUT/r02_synccheck.log 2>&1; echo synccheck_rc=$?; tail -2 $OUT/r02_synccheck.log
python bench.py > $OUT/r02_bench_cfg4.json 2> $OUT/r02_bench_cfg4.err; echo cfg4_rc=$?
python bench.py --config cfg2 > $OUT/r02_bench_cfg2.json 2> $OUT/r02_bench_cfg2.err; echo cfg2_rc=$?
python bench.py --config cfg3 > $OUT/r02_bench_cfg3.json 2> $OUT/r02_bench_cfg3.err; echo cfg3_rc=$?
python bench.py --config cfg5 > $OUT/r02_bench_cfg5.json 2> $OUT/r02_bench_cfg5.err; echo cfg5_rc=$?
python bench.py --impl reference > $OUT/r02_ref_cfg4.json 2> $OUT/r02_ref_cfg4.err; echo ref_rc=$?
