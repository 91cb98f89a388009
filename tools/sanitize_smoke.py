"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck /
synccheck): the per-frame pipeline (fused and staged mask paths), the
batcher gather, and the drop-in stitch.  Tuning / verification aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2404_09267_b200 import _native as N  # noqa: E402
from paper_2404_09267_b200 import api as A  # noqa: E402
from paper_2404_09267_b200 import multicam as MC  # noqa: E402
from tests._helpers import GpuRun  # noqa: E402

ctx = A.Context(0)
run = GpuRun(ctx, 640, 368, 4, seed=1000, trace_kw=dict(roi_max_dim=200), keep_mask=False)
gpu = run.run()
A.check(N.lib().tg_pipeline_stage_mask_fg(run.pipe.handle, run.n, run.d_cur, run.d_prev, None))
A.check(N.lib().tg_pipeline_stage_mask_cells(run.pipe.handle, run.n, None))
ctx.synchronize()
print("pipeline", gpu["total_canvases"], "canvases")
run.close()
# edge geometries: partial words / cell rows, uneven K1 parts, radius 0 / 8,
# odd canvases, fine zone grids, padded pitch, masks kept
for W, H, n, kw in [(208, 100, 3, dict(radius=2)), (2080, 70, 3, {}), (8192, 48, 2, {}),
                    (640, 360, 3, dict(radius=8, keep_mask=True)), (640, 360, 3, dict(radius=0)),
                    (1280, 720, 2, dict(zones=(8, 8))),
                    (1280, 720, 2, dict(zones=(3, 5), canvas=(300, 200))),
                    (640, 352, 2, dict(pitch=640 * 3 + 64))]:
    kw = dict(kw)
    kw.setdefault("keep_mask", False)
    r = GpuRun(ctx, W, H, n, seed=7, trace_kw=dict(roi_max_dim=min(480, W, H)), **kw)
    g = r.run()
    ctx.synchronize()
    print("edge", W, H, g["total_canvases"], "canvases")
    r.close()
path = MC.MultiCameraPath(ctx, [0, 1], 640, 368, 4, [(1, 60.0, 3.0), (2, 85.0, 4.0)],
                          bandwidth_mbps=40.0, trace_kw=dict(roi_max_dim=200))
_, n_ev, n_canv = path.step()
ctx.synchronize()
print("batcher", n_ev, "events", n_canv, "canvases")
path.close()
A.check(N.lib().tg_ctx_set_option(ctx.handle, N.TG_OPT_GATHER_BAND, 256))  # tall units
path = MC.MultiCameraPath(ctx, [0, 1], 640, 368, 4, [(1, 60.0, 3.0), (2, 85.0, 4.0)],
                          bandwidth_mbps=40.0, trace_kw=dict(roi_max_dim=200))
_, n_ev, n_canv = path.step()
ctx.synchronize()
print("batcher band 256", n_ev, "events", n_canv, "canvases")
path.close()
A.check(N.lib().tg_ctx_set_option(ctx.handle, N.TG_OPT_GATHER_BAND, 0))
comm = A.Comm.nccl(ctx, A.Comm.unique_id(), 0, 1)  # device descriptor all-gather
path = MC.MultiCameraPath(ctx, [0, 1], 640, 368, 4, [(1, 60.0, 3.0), (2, 85.0, 4.0)],
                          bandwidth_mbps=40.0, trace_kw=dict(roi_max_dim=200), comm=comm)
print("nccl pass", path.run_pipelined(2), "canvases")
path.close()
comm.close()
q = [A.PatchMeta(i, 0, A.Rect(0, 0, 30 + 7 * i, 20 + 5 * i), 0, 1, 1, 1) for i in range(12)]
res = A.stitch_all(q, A.CanvasSpec(128, 128), ctx=ctx)
print("stitch", res.canvas_count(), "canvases")
q = [A.PatchMeta(i, 0, A.Rect(0, 0, 20 + i % 50, 10 + i % 30), 0, 1, 1, 1) for i in range(300)]
res = A.stitch_all(q, A.CanvasSpec(100, 100), ctx=ctx)  # longer than the staged queue
print("stitch long", res.canvas_count(), "canvases")
z = A.make_zones(A.FrameSpec(0, 640, 360), A.PartitionConfig(4, 4))
print("partition", len(A.partition(A.FrameSpec(0, 640, 360), A.PartitionConfig(4, 4),
                                    [A.Rect(10, 10, 100, 50), A.Rect(300, 200, 40, 40)], 1.5,
                                    ctx=ctx)), "patches", len(z), "zones")
ctx.close()
