OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/c1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > $OUT/c1_pytest.log 2>&1; echo pytest_rc=$?
tail -40 $OUT/c1_pytest.log
timeout 300 python tools/multicam_timeline.py cfg4 8 > $OUT/c1_timeline.log 2>&1; echo tl_rc=$?
cat $OUT/c1_timeline.log
for g in 148 128 112; do TG_K1_GRID=$g timeout 300 python tools/multicam_timeline.py cfg4 6 > $OUT/c1_timeline_g$g.log 2>&1; tail -1 $OUT/c1_timeline_g$g.log; done
