# Fused mask launch (config 2) on the sparse bitmap (TG_K1_SPARSE_FUSED=1
# variant): same-box A/B of the config-2 step, then the GPU suite on it.
OUT=gpurun_out
for round in 1 2; do
  for v in default spfused; do
    if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
    echo "[$v cfg2] $(python bench.py --config cfg2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['launch_ms'])")"
  done
done
export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/spfused.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/sf_gputest.log 2>&1; echo spfused_parity_rc=$?; tail -3 $OUT/sf_gputest.log
