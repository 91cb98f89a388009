# cfg4 ms/step of bench variants selected by environment assignments, e.g.
#   bash tools/gpu/cfg4_ms.sh "" "TG_SPLIT_MASK=1" "TG_SPLIT_MASK=1 TG_K5_BPS=2"
for round in 1 2; do
  for v in "$@"; do
    ms=$(env $v python bench.py --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])")
    echo "[$v] $ms"
  done
done
