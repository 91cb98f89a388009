OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not cfg3 and not cfg4" > $OUT/$1_pytest.log 2>&1; echo pytest_rc=$?; tail -1 $OUT/$1_pytest.log
for i in 1 2; do timeout 120 python tools/mask_split.py 300 fused,k1,k1b 2>&1 | tail -3; done
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r.get('launch_ms_isolated'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/$1_cfg4.json 2>&1; python -c "$S" $OUT/$1_cfg4.json
timeout 300 python bench.py --config cfg2 --no-e2e --no-cpu > $OUT/$1_cfg2.json 2>&1; python -c "$S" $OUT/$1_cfg2.json
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:mask_fg -s 2 -c 1 -o $OUT/$1_k1 -f python tools/mask_split.py 300 k1 > $OUT/$1_k1ncu.log 2>&1; echo ncu rc=$?
