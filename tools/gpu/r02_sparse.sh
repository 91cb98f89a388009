# Sparse raw bitmap (TG_K1_SPARSE=1 variant) on the split K1 / K1b launches of
# configs 3/4: GPU suite on the variant, then same-box A/B against the build.
OUT=gpurun_out
export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/sparse.so
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/sp_gputest.log 2>&1; echo sparse_gputest_rc=$?; tail -3 $OUT/sp_gputest.log
unset TANGRAM_GPU_LIB
bash tools/gpu/cfg4_lib_ms.sh default sparse 2>&1
for v in default sparse; do
  if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
  echo "[$v cfg3] $(python bench.py --config cfg3 --no-cpu --no-e2e --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])")"
done
