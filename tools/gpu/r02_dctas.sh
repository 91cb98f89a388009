for rep in 1 2; do
for d in 13 8 10 11 12 14 16; do echo "dctas=$d $(TG_K1_DCTAS=$d timeout 120 python tools/mask_split.py 300 fused 2>&1 | tail -1)"; done
done
