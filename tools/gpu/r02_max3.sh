OUT=gpurun_out
V=paper_2404_09267_b200/lib/variants/max3.so
TANGRAM_GPU_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "edge_cases or cfg2 or broken or empty or cfg1 or two_launch" > $OUT/m3_pytest.log 2>&1; echo pytest_rc=$?; tail -1 $OUT/m3_pytest.log
for i in 1 2; do
echo "== base"; timeout 120 python tools/mask_split.py 300 fused,k1,k1b 2>&1 | tail -3
echo "== max3"; TANGRAM_GPU_LIB=$V timeout 120 python tools/mask_split.py 300 fused,k1,k1b 2>&1 | tail -3
done
timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/m3_cfg4_base.json 2>&1
TANGRAM_GPU_LIB=$V timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/m3_cfg4_max3.json 2>&1
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r.get('launch_ms_isolated'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
python -c "$S" $OUT/m3_cfg4_base.json; python -c "$S" $OUT/m3_cfg4_max3.json
