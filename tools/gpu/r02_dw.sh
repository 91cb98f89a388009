# fused mask stage: K1b task warps beside the stream (dw*) x dedicated K1b CTAs (TG_K1_DCTAS)
V=paper_2404_09267_b200/lib/variants
for rep in 1 2; do
echo "== base"; timeout 120 python tools/mask_split.py 300 fused 2>&1 | tail -1
for d in 0 4; do echo "== base dctas=$d"; TG_K1_DCTAS=$d timeout 120 python tools/mask_split.py 300 fused 2>&1 | tail -1; done
for w in 1 2 4; do
  echo "== dw$w"; TANGRAM_GPU_LIB=$V/dw$w.so timeout 120 python tools/mask_split.py 300 fused 2>&1 | tail -1
  for d in 0 4; do echo "== dw$w dctas=$d"; TG_K1_DCTAS=$d TANGRAM_GPU_LIB=$V/dw$w.so timeout 120 python tools/mask_split.py 300 fused 2>&1 | tail -1; done
done
done
