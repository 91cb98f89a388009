OUT=gpurun_out
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r.get('launch_ms_isolated'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
timeout 600 python -m pytest tests/test_gpu_multicam.py -q -x > $OUT/el_pytest.log 2>&1; echo pytest_rc=$?; tail -1 $OUT/el_pytest.log
for rep in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/el_e$rep.json 2>&1; python -c "$S" $OUT/el_e$rep.json
  TG_BENCH_FIXED_GATHER=1 timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/el_f$rep.json 2>&1; python -c "$S" $OUT/el_f$rep.json
done
timeout 300 python bench.py --config cfg3 --no-e2e --no-cpu > $OUT/el_cfg3.json 2>&1; python -c "$S" $OUT/el_cfg3.json
TG_BENCH_FIXED_GATHER=1 timeout 300 python bench.py --config cfg3 --no-e2e --no-cpu > $OUT/el_cfg3f.json 2>&1; python -c "$S" $OUT/el_cfg3f.json
timeout 300 python tools/multicam_timeline.py cfg4 8 > $OUT/el_timeline.log 2>&1; tail -4 $OUT/el_timeline.log
