set -x
export TG_BENCH_SHARE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --cams 8 --frames 10 --steps 3 --warmup 2 --e2e-steps 1 > gpurun_out/r2_n2.json 2> gpurun_out/r2_n2.err; echo rc=$?; tail -3 gpurun_out/r2_n2.err; head -c 1500 gpurun_out/r2_n2.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --cams 8 --frames 10 --steps 3 --warmup 2 --e2e-steps 1 --global-batching --no-secondary > gpurun_out/r2_n2g.json 2> gpurun_out/r2_n2g.err; echo rc=$?; tail -3 gpurun_out/r2_n2g.err; head -c 600 gpurun_out/r2_n2g.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --impl reference --cams 4 --frames 4 --steps 1 --warmup 1 > gpurun_out/r2_n2r.json 2> gpurun_out/r2_n2r.err; echo rc=$?; tail -3 gpurun_out/r2_n2r.err; cat gpurun_out/r2_n2r.json
unset TG_BENCH_SHARE_GPU
python bench.py --config cfg3 > gpurun_out/r2_cfg3.json 2> gpurun_out/r2_cfg3.err; echo rc=$?; tail -2 gpurun_out/r2_cfg3.err
python bench.py --config cfg5 > gpurun_out/r2_cfg5.json 2> gpurun_out/r2_cfg5.err; echo rc=$?; tail -2 gpurun_out/r2_cfg5.err
python bench.py --config cfg2 > gpurun_out/r2_cfg2.json 2> gpurun_out/r2_cfg2.err; echo rc=$?; tail -2 gpurun_out/r2_cfg2.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"mask_fg|plan_kernel|gather_kernel" -c 12 --csv --log-file gpurun_out/r2_cfg4_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary > gpurun_out/r2_ncu_cfg4.log 2>&1; echo ncu_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --cams 8 --frames 30 > gpurun_out/r2_ncu_list.log 2>&1; echo ncu_rc=$?
