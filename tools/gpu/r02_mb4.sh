OUT=gpurun_out
V=paper_2404_09267_b200/lib/variants/mb4.so
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], d['path'].get('stage_ms'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
for rep in 1 2; do
timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/mb_base$rep.json 2>&1; python -c "$S" $OUT/mb_base$rep.json
TANGRAM_GPU_LIB=$V TG_BENCH_GATHER_GRID=0 timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/mb_4g0_$rep.json 2>&1; python -c "$S" $OUT/mb_4g0_$rep.json
TANGRAM_GPU_LIB=$V timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/mb_4g2_$rep.json 2>&1; python -c "$S" $OUT/mb_4g2_$rep.json
done
timeout 300 python bench.py --config cfg2 --no-e2e --no-cpu > $OUT/mb_c2base.json 2>&1; python -c "$S" $OUT/mb_c2base.json
TANGRAM_GPU_LIB=$V timeout 300 python bench.py --config cfg2 --no-e2e --no-cpu > $OUT/mb_c2mb4.json 2>&1; python -c "$S" $OUT/mb_c2mb4.json
