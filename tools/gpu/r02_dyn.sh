OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_multicam.py tests/test_gpu_parity.py -q -x -k "multicam or two_launch or pipelined or partitioned or edge_cases" > $OUT/dy_pytest.log 2>&1; echo pytest_rc=$?; tail -1 $OUT/dy_pytest.log
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], r.get('launch_ms_isolated'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
for rep in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/dy_on$rep.json 2>&1; python -c "$S" $OUT/dy_on$rep.json
  TG_K1_DYNAMIC=0 timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/dy_off$rep.json 2>&1; python -c "$S" $OUT/dy_off$rep.json
  for r in 16 64; do TG_K1_RUNS=$r timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/dy_r$r$rep.json 2>&1; python -c "$S" $OUT/dy_r$r$rep.json; done
done
