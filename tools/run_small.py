"""Debug helper: one small pipeline run (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09267_b200 import api as A, _native as N
from tests._helpers import GpuRun
W, H, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ctx = A.Context(0)
run = GpuRun(ctx, W, H, n, seed=1000, trace_kw=dict(roi_max_dim=min(480, W, H)))
A.check(N.lib().tg_pipeline_stage_mask(run.pipe.handle, n, run.d_cur, run.d_prev, None)); ctx.stream_sync(); print("mask ok", flush=True)
A.check(N.lib().tg_pipeline_stage_plan(run.pipe.handle, n, run.d_ids, run.d_gen, 0, None)); ctx.stream_sync(); print("plan ok", flush=True)
A.check(N.lib().tg_pipeline_stage_gather(run.pipe.handle, n, run.d_cur, run.d_canvases, None)); ctx.stream_sync(); print("gather ok", flush=True)
