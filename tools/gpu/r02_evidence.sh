# Round-2 evidence at HEAD: the GPU test suite, every bench line with all legs,
# the reference arm, then the profiling recipe (launch lists + set-full
# captures), summarized on the box (profiles/ copies come back in
# gpurun_out/evidence/; the large .ncu-rep files are dropped).
OUT=gpurun_out
mkdir -p $OUT/evidence
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/ev_smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/ev_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/ev_pytest.log
for c in cfg4 cfg2 cfg3 cfg5; do
  timeout 900 python bench.py --config $c > $OUT/ev_bench_$c.json 2> $OUT/ev_bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > $OUT/ev_ref_cfg4.json 2> $OUT/ev_ref_cfg4.err; echo "ref rc=$?"
bash tools/gpu/r02_profile.sh > $OUT/ev_profile.log 2>&1; echo "profile rc=$?"
python tools/summarize_profiles.py r02_cfg4 1984 profiles/r02_k1_cfg4_traffic.json "Config 4 (BASELINE configs[3]): 64 cameras x 30 4K frames on one GPU, one pass = K1 over 1,920 frames (64 chains + backgrounds = 1,984 frame reads), K1b, planner + device descriptors, one K5 launch for every invoke event's canvases." > $OUT/ev_sum4.log 2>&1
python tools/summarize_profiles.py r02_cfg2 301 profiles/k1_traffic.json "Config 2 (BASELINE configs[1]): one 4K camera, 300 frames per step (301 frame reads); fused mask launch (K1 + K1b tasks), planner, K5." > $OUT/ev_sum2.log 2>&1
cp profiles/r02_cfg4_summary.md profiles/r02_cfg4_launches.csv profiles/r02_cfg2_summary.md profiles/r02_cfg2_launches.csv profiles/r02_k1_cfg4_traffic.json profiles/k1_traffic.json $OUT/evidence/
rm -f $OUT/*.ncu-rep
du -sh $OUT
