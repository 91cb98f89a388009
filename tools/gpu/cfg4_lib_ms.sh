# cfg4 ms/step for library variants (paper_2404_09267_b200/lib/variants/<v>.so; "default" = the build)
for round in 1 2; do
  for v in "$@"; do
    if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
    echo "[$v] $(python bench.py --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])")"
  done
done
