OUT=gpurun_out
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
timeout 600 python -m pytest tests/test_gpu_multicam.py -q -x > $OUT/tu_pytest.log 2>&1; echo pytest_rc=$?; tail -1 $OUT/tu_pytest.log
for rep in 1 2 3; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/tu_on$rep.json 2>&1; python -c "$S" $OUT/tu_on$rep.json
  TG_PROBE_TOPUP=0 timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/tu_off$rep.json 2>&1; python -c "$S" $OUT/tu_off$rep.json
done
timeout 300 python bench.py --config cfg3 --no-e2e --no-cpu > $OUT/tu_c3on.json 2>&1; python -c "$S" $OUT/tu_c3on.json
TG_PROBE_TOPUP=0 timeout 300 python bench.py --config cfg3 --no-e2e --no-cpu > $OUT/tu_c3off.json 2>&1; python -c "$S" $OUT/tu_c3off.json
