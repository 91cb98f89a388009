OUT=gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:mask_fg -s 2 -c 1 -o $OUT/$1_k1 -f python tools/mask_split.py 300 k1 > $OUT/$1_k1ncu.log 2>&1; echo ncu rc=$?
