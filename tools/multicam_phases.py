"""Wall-clock split of one config-3/4 step (device planes, descriptor D2H,
host batcher replay, device gather) -- tuning aid."""
import sys
import time
sys.path.insert(0, ".")
from paper_2404_09267_b200 import api as A
from paper_2404_09267_b200 import multicam as MC
import bench

W, H = 3840, 2160
ncam, frames = (5, 300) if (len(sys.argv) > 1 and sys.argv[1] == "cfg3") else (64, 30)
ctx = A.Context(0)
path = MC.MultiCameraPath(ctx, list(range(ncam)), W, H, frames, bench.SIM_PROFILE,
                          bandwidth_mbps=bench.SIM_BANDWIDTH_MBPS, gpu_memory_gb=bench.SIM_GPU_MEMORY_GB,
                          model_size_gb=4.0, trace_kw=dict(roi_proportion_mean=0.10, roi_max_dim=480))
for it in range(6):
    t0 = time.perf_counter()
    path.run_planes()
    ctx.stream_sync(path.stream)
    t1 = time.perf_counter()
    desc = path.descriptors()
    t2 = time.perf_counter()
    path.schedule(desc)
    t3 = time.perf_counter()
    n = path.gather()
    ctx.stream_sync(path.stream)
    t4 = time.perf_counter()
    print(f"planes {1e3*(t1-t0):.2f} ms  desc {1e3*(t2-t1):.2f} ms  schedule {1e3*(t3-t2):.2f} ms  "
          f"gather {1e3*(t4-t3):.2f} ms  canvases {n}  patches {len(desc)}", flush=True)
