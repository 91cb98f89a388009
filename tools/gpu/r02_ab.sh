# A/B on one box: $V1 vs the in-tree library (mask stage, cfg4 and cfg2 lines)
V=paper_2404_09267_b200/lib/variants/$1.so
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r.get('launch_ms_isolated'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
OUT=gpurun_out
for rep in 1 2; do
  echo "== $1"; TANGRAM_GPU_LIB=$V timeout 120 python tools/mask_split.py 300 fused,k1 2>&1 | tail -2
  echo "== new"; timeout 120 python tools/mask_split.py 300 fused,k1 2>&1 | tail -2
  TANGRAM_GPU_LIB=$V timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/ab_$1_$rep.json 2>&1; python -c "$S" $OUT/ab_$1_$rep.json
  timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/ab_new_$rep.json 2>&1; python -c "$S" $OUT/ab_new_$rep.json
done
