"""Device timeline of the pipelined config-3/4 passes (MultiCameraPath.
run_pipelined with CUDA events around K1, the planner and the descriptor
read-back on `stream` and around K5 on `gstream`), to find bubbles.
Tuning aid.   python tools/multicam_timeline.py [cfg3|cfg4] [passes]"""
import sys
import time

sys.path.insert(0, ".")
from paper_2404_09267_b200 import _native as N  # noqa: E402
from paper_2404_09267_b200 import api as A  # noqa: E402
from paper_2404_09267_b200 import multicam as MC  # noqa: E402
import bench  # noqa: E402

W, H = 3840, 2160
ncam, frames = (5, 300) if (len(sys.argv) > 1 and sys.argv[1] == "cfg3") else (64, 30)
ctx = A.Context(0)
path = MC.MultiCameraPath(ctx, list(range(ncam)), W, H, frames, bench.SIM_PROFILE,
                          trace_kw=dict(bench.TRACE), **bench.SIM)
path.run_pipelined(3)
ctx.synchronize()
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
names = ("k1a", "k1b", "k1c", "pl", "fe", "g0", "g1")
split = __import__("os").environ.get("TG_FUSED_MASK") != "1"  # MultiCameraPath: split
ev = {k: [ctx.event() for _ in range(steps + 1)] for k in names}
host = []
lib = N.lib()
F = ncam * frames


def planes(i):  # MultiCameraPath.run_planes, with events
    ctx.record(ev["k1a"][i], path.stream)
    if split:
        A.check(lib.tg_pipeline_stage_mask_fg(path.pipe.handle, F, path.d_cur, path.d_prev,
                                              path.stream))
        ctx.record(ev["k1b"][i], path.stream)
        A.check(lib.tg_pipeline_stage_mask_cells(path.pipe.handle, F, path.stream))
    else:
        A.check(lib.tg_pipeline_stage_mask(path.pipe.handle, F, path.d_cur, path.d_prev,
                                           path.stream))
        ctx.record(ev["k1b"][i], path.stream)
    ctx.record(ev["k1c"][i], path.stream)
    A.check(lib.tg_pipeline_stage_plan(path.pipe.handle, F, path.d_ids, path.d_gen, 0, path.stream))
    ctx.record(ev["pl"][i], path.stream)


origin = ctx.event()
ctx.record(origin, path.stream)
t_start = time.perf_counter()
planes(0)
path.fetch_descriptors(0)
ctx.record(ev["fe"][0], path.stream)
for i in range(steps):  # MultiCameraPath.run_pipelined, with events
    h0 = time.perf_counter()
    if i + 1 < steps:
        planes(i + 1)
        path.fetch_descriptors((i + 1) % 2)
        ctx.record(ev["fe"][i + 1], path.stream)
    desc = path.compact_descriptors(i % 2)
    h1 = time.perf_counter()
    path.schedule(desc)
    h2 = time.perf_counter()
    ctx.record(ev["g0"][i], path.gstream)
    path.gather(join=False)
    ctx.record(ev["g1"][i], path.gstream)
    host.append((1e3 * (h0 - t_start), 1e3 * (h1 - h0), 1e3 * (h2 - h1)))
path.join()
ctx.synchronize()
t = {k: [ctx.elapsed_ms(origin, e) for e in ev[k][:steps]] for k in names}
for i in range(steps):
    print(f"pass {i}: K1 {t['k1a'][i]:8.2f}->{t['k1b'][i]:8.2f} ({t['k1b'][i]-t['k1a'][i]:5.2f}) "
          f"K1b ->{t['k1c'][i]:8.2f} ({t['k1c'][i]-t['k1b'][i]:4.2f}) "
          f"plan ->{t['pl'][i]:8.2f} ({t['pl'][i]-t['k1c'][i]:4.2f}) fetch ->{t['fe'][i]:8.2f} "
          f"K5 {t['g0'][i]:8.2f}->{t['g1'][i]:8.2f} ({t['g1'][i]-t['g0'][i]:5.2f})  host start "
          f"{host[i][0]:8.2f} wait+flatten {host[i][1]:5.2f} schedule {host[i][2]:5.2f}", flush=True)
span = t["g1"][steps - 1] - t["k1a"][1]
print(f"passes 1..{steps - 1}: {span / (steps - 1):.3f} ms per pass")
