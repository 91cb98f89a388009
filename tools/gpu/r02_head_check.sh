# Re-entry check at HEAD: the GPU suite, smoke, and the default bench line.
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/hc_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/hc_gputest.log 2>&1; echo gputest_rc=$?; tail -3 $OUT/hc_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/hc_smoke.log 2>&1; echo smoke_rc=$?; tail -1 $OUT/hc_smoke.log
timeout 600 python bench.py > $OUT/hc_bench_cfg4.json 2> $OUT/hc_bench_cfg4.err; echo cfg4_rc=$?; head -c 400 $OUT/hc_bench_cfg4.json
