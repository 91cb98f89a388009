OUT=gpurun_out
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['mask_path'])"
for rep in 1 2; do
timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/f4_split$rep.json 2>&1; python -c "$S" $OUT/f4_split$rep.json
TG_PROBE_FUSED=1 timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/f4_fused$rep.json 2>&1; python -c "$S" $OUT/f4_fused$rep.json
TG_PROBE_FUSED=1 TG_BENCH_GATHER_GRID=0 timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/f4_fusedg$rep.json 2>&1; python -c "$S" $OUT/f4_fusedg$rep.json
done
