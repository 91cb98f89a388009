# A/B of library variants on configs 3 and 5 (device value only)
for round in 1 2; do
  for v in "$@"; do
    if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
    for c in cfg3 cfg5; do
      echo "[$v $c] $(python bench.py --config $c --no-cpu --no-e2e --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d.get('sweep', ''))" 2>&1 | cut -c1-300)"
    done
  done
done
