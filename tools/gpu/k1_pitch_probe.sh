# raw-bitmap row pitch / L2-hint variants: fused mask stage time, 300 4K frames,
# two interleaved rounds (base = unpadded rows, no hints: the round-1 kernel)
for round in 1 2; do
for v in base keep0_p128 keep0_p160 keep1_p128 default; do
  if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
  echo "== $v $(python tools/mask_split.py 300 fused 2>&1 | tail -1)"
done
done
