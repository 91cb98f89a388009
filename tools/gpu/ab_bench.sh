# A/B of a library variant against the current build inside one gpurun call:
# bench (cfg4 headline + cfg2 secondary, no CPU / e2e legs), twice each, interleaved
summ() { python -c "
import json,sys;d=json.load(open(sys.argv[1]))
s=d['secondary']['cfg2']
print(sys.argv[2], 'cfg4', d['value'], d['ms_per_step'], 'K1', d['roofline']['launch_ms'], 'cfg2', s['value'], s['ms_per_step'], s['path']['stage_ms'], d['clocks']['reasons'])" $1 $2; }
for round in 1 2; do
  for v in "$@"; do
    if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
    python bench.py --no-cpu --no-e2e > gpurun_out/ab_$v.json 2>/dev/null && summ gpurun_out/ab_$v.json $v
  done
done
