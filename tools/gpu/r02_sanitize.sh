# compute-sanitizer on the smoke paths (tools/sanitize_smoke.py)
OUT=gpurun_out
timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > $OUT/r02_memcheck.log 2>&1; echo memcheck_rc=$?; tail -3 $OUT/r02_memcheck.log
timeout 1200 compute-sanitizer --tool synccheck --num-cuda-barriers 65536 python tools/sanitize_smoke.py > $OUT/r02_synccheck.log 2>&1; echo synccheck_rc=$?; tail -3 $OUT/r02_synccheck.log
timeout 1800 compute-sanitizer --tool racecheck --num-cuda-barriers 65536 python tools/sanitize_smoke.py > $OUT/r02_racecheck.log 2>&1; echo racecheck_rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $OUT/r02_racecheck.log; grep -E "^=========     at .*\.(cu|cuh):" $OUT/r02_racecheck.log | sed 's/0x[0-9a-f]*//g' | sort | uniq -c | sort -rn | head -12
