"""Device timeline of the pipelined config-3/4 passes (MultiCameraPath.
run_pipelined with CUDA events around the planes on `stream` and the gathers
on `gstream`), to find bubbles.  Tuning aid."""
import sys
import time

sys.path.insert(0, ".")
from paper_2404_09267_b200 import api as A  # noqa: E402
from paper_2404_09267_b200 import multicam as MC  # noqa: E402
import bench  # noqa: E402

W, H = 3840, 2160
ncam, frames = (5, 300) if (len(sys.argv) > 1 and sys.argv[1] == "cfg3") else (64, 30)
ctx = A.Context(0)
path = MC.MultiCameraPath(ctx, list(range(ncam)), W, H, frames, bench.SIM_PROFILE,
                          bandwidth_mbps=bench.SIM_BANDWIDTH_MBPS,
                          gpu_memory_gb=bench.SIM_GPU_MEMORY_GB, model_size_gb=4.0,
                          trace_kw=dict(roi_proportion_mean=0.10, roi_max_dim=480))
path.run_pipelined(3)
ctx.synchronize()
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ev = {k: [ctx.event() for _ in range(steps + 1)] for k in ("p0", "p1", "g0", "g1")}
host = []
t_start = time.perf_counter()


def planes(i):
    ctx.record(ev["p0"][i], path.stream)
    path.run_planes()
    ctx.record(ev["p1"][i], path.stream)


origin = ctx.event()
ctx.record(origin, path.stream)
planes(0)
path.fetch_descriptors(0)
for i in range(steps):  # MultiCameraPath.run_pipelined, with events
    h0 = time.perf_counter()
    if i + 1 < steps:
        planes(i + 1)
        path.fetch_descriptors((i + 1) % 2)
    desc = path.compact_descriptors(i % 2)
    path.schedule(desc)
    h1 = time.perf_counter()
    ctx.record(ev["g0"][i], path.gstream)
    path.gather(join=False)
    ctx.record(ev["g1"][i], path.gstream)
    host.append((1e3 * (h0 - t_start), 1e3 * (h1 - h0)))
path.join()
ctx.synchronize()
for i in range(steps):
    p0 = ctx.elapsed_ms(origin, ev["p0"][i])
    p1 = ctx.elapsed_ms(origin, ev["p1"][i])
    g0 = ctx.elapsed_ms(origin, ev["g0"][i])
    g1 = ctx.elapsed_ms(origin, ev["g1"][i])
    print(f"pass {i}: planes {p0:8.2f} -> {p1:8.2f} ({p1 - p0:5.2f})  gather {g0:8.2f} -> {g1:8.2f} "
          f"({g1 - g0:5.2f})  host loop start {host[i][0]:8.2f} schedule {host[i][1]:5.2f}", flush=True)
