OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $OUT/su_gputest.log 2>&1; echo gputest_rc=$?; tail -3 $OUT/su_gputest.log
timeout 900 python bench.py > $OUT/su_bench_cfg4.json 2> $OUT/su_bench_cfg4.err; echo cfg4_rc=$?
python -c "import json;d=json.load(open('$OUT/su_bench_cfg4.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['path']['unique_frac'],d['clocks'])"
