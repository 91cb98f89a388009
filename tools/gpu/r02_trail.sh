# fused mask stage (300 4K frames): time + DRAM bytes per library variant
for v in "$@"; do
  if [ $v = default ]; then unset TANGRAM_GPU_LIB; else export TANGRAM_GPU_LIB=paper_2404_09267_b200/lib/variants/$v.so; fi
  echo "[$v] $(python tools/mask_split.py 300 fused | tail -1)"
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:mask_fg -s 3 -c 1 --csv python tools/mask_split.py 300 fused 2>/dev/null | grep -E 'dram__bytes|duration' | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
done
