# Per-rank load of config 4 at N = 1/2/4/8 (64/N cameras x 30 frames on one
# GPU, no collective): projects the strong-scaling curve the driver measures.
OUT=gpurun_out
for c in 64 32 16 8; do
  timeout 400 python bench.py --cams $c --steps 20 --warmup 5 --no-e2e --no-cpu --no-secondary > $OUT/ss_cams$c.json 2> $OUT/ss_cams$c.err; echo cams=$c rc=$?
  python -c "import json;d=json.load(open('$OUT/ss_cams$c.json'));print($c, d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d['clocks'])"
done
