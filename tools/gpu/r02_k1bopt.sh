OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not cfg3 and not cfg4" > $OUT/kp_pytest.log 2>&1; echo pytest_rc=$?; tail -1 $OUT/kp_pytest.log
for i in 1 2; do
 echo "== old"; TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/old.so timeout 120 python tools/mask_split.py 300 fused,k1b 2>&1 | tail -2
 echo "== new"; timeout 120 python tools/mask_split.py 300 fused,k1b 2>&1 | tail -2
done
S="import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); r=d['roofline']; print(sys.argv[1], d['value'], d['ms_per_step'], r['launch_ms'], r.get('launch_ms_isolated'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
for i in 1 2; do
TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/old.so timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/kp_old$i.json 2>&1; python -c "$S" $OUT/kp_old$i.json
timeout 300 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/kp_new$i.json 2>&1; python -c "$S" $OUT/kp_new$i.json
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:dilate -s 2 -c 1 -o $OUT/kp_k1b -f python tools/mask_split.py 300 k1b > $OUT/kp_ncu.log 2>&1; echo ncu rc=$?
