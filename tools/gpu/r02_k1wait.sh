OUT=gpurun_out
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
for rep in 1 2 3; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/kw_on$rep.json 2>&1; python -c "$S" $OUT/kw_on$rep.json
  TG_PROBE_K1WAIT=0 timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/kw_off$rep.json 2>&1; python -c "$S" $OUT/kw_off$rep.json
done
