# Does K1 lose anything at 4 ring slots (the sparse build's 64-word parts fit
# 4 in shared memory; 60-word parts fit 5)?  Dense build, 5 vs 4 slots.
export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/dense.so
for round in 1 2; do
  for sl in 5 4; do
    export TG_K1_SLOTS=$sl
    echo "[dense slots=$sl cfg4] $(python bench.py --no-cpu --no-e2e --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['launch_ms_isolated'])")"
    echo "[dense slots=$sl cfg2] $(python bench.py --config cfg2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['launch_ms'])")"
  done
done
