# trailing K1b (publisher warp + task order) vs the round-1 kernel (base):
# fused mask stage, 300 4K frames; K1b CTA counts; publish block sizes
run() { echo "== $1 $(python tools/mask_split.py 300 fused 2>&1 | tail -1)"; }
for round in 1 2; do
  export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/base.so; run base
  unset TANGRAM_GPU_LIB; run trail8
  for d in 10 16 20; do TG_K1_DCTAS=$d run trail8_dctas$d; done
  export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/pub4.so; run pub4
  export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/pub16.so; run pub16
  export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/trail_nohint.so; run trail_nohint
  unset TANGRAM_GPU_LIB
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:mask_fg -s 3 -c 1 --csv python tools/mask_split.py 300 fused 2>/dev/null | grep -E "mask_fg" | awk -F'","' '{print $(NF-2), $NF}'
