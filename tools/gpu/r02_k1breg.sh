OUT=gpurun_out
V=paper_2404_09267_b200/lib/variants
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
for rep in 1 2; do
  echo "== base $(timeout 120 python tools/mask_split.py 300 k1b,fused 2>&1 | tail -2 | tr '\n' ' ')"
  for r in 72 80; do echo "== k1b$r $(TANGRAM_GPU_LIB=$V/k1b$r.so timeout 120 python tools/mask_split.py 300 k1b,fused 2>&1 | tail -2 | tr '\n' ' ')"; done
  timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/kr_base$rep.json 2>&1; python -c "$S" $OUT/kr_base$rep.json
  for r in 72 80; do TANGRAM_GPU_LIB=$V/k1b$r.so timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/kr_$r$rep.json 2>&1; python -c "$S" $OUT/kr_$r$rep.json; done
done
