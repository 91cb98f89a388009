OUT=gpurun_out
for v in default dense; do
  if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "stale" --tb=line > $OUT/sd_$v.log 2>&1; echo "$v rc=$?"; grep -E "passed|failed|Error|assert" $OUT/sd_$v.log | head -30
done
unset TANGRAM_GPU_LIB
bash tools/gpu/r02_spfused.sh
