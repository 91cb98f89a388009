# config-4 pass vs the event gather's grid (TG_BENCH_GATHER_GRID; 0 = SMs x occupancy)
for round in 1 2; do
  for g in 296 222 370 444 148; do
    echo "[grid $g] $(TG_BENCH_GATHER_GRID=$g python bench.py --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['launch_ms'])")"
  done
done
