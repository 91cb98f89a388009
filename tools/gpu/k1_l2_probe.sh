# K1 L2-residency probe: mask stage time (fused launch, 300 4K frames) and
# ncu DRAM bytes for: raw bitmap round trip as before (keep0), evict hints +
# discard without / with the persisting-L2 set-aside (keep1).
V=paper_2404_09267_b200/lib/variants/keep0.so
for cfg in "keep0 $V -1" "keep1_nopersist - 0" "keep1 - -1"; do
  set -- $cfg
  name=$1; lib=$2; mb=$3
  export TG_L2_PERSIST_MB=$mb
  if [ "$lib" != "-" ]; then export TANGRAM_GPU_LIB=$lib; else unset TANGRAM_GPU_LIB; fi
  echo "== $name"
  python tools/mask_split.py 300 fused 2>&1 | tail -1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:mask_fg -s 3 -c 1 --csv python tools/mask_split.py 300 fused 2>/dev/null | grep -E "mask_fg" | awk -F'","' '{print $(NF-2), $NF}'
done
