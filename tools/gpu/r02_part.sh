OUT=gpurun_out
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], r.get('launch_ms_isolated'), d['clocks']['sm_mhz'], d['clocks']['reasons'], d.get('mask_path',{}).get('partition'))"
timeout 600 python -m pytest tests/test_gpu_multicam.py -q -x > $OUT/$1_pytest.log 2>&1; echo pytest_rc=$?; tail -15 $OUT/$1_pytest.log | grep -E "passed|failed|Error|error" | head
for s in 16 0 24 12; do timeout 300 python bench.py --no-e2e --no-cpu --no-secondary --side-sms $s > $OUT/$1_cfg4_s$s.json 2>&1; python -c "$S" $OUT/$1_cfg4_s$s.json; done
