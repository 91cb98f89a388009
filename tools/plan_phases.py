"""Per-phase cycle split of the planner (plan_kernel) on the cfg2 workload:
builds a diagnostics variant of the library with -DTG_PLAN_PHASES (thread 0
of every frame CTA marks clock64 after each phase) and prints the mean
cycles per frame CTA of each phase.  Tuning aid; run on the GPU box."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANT = os.path.join(ROOT, "paper_2404_09267_b200", "lib", "variants", "libtangram_gpu_phases.so")

if os.environ.get("TANGRAM_GPU_LIB") != VARIANT:
    from paper_2404_09267_b200 import build as B
    B.build(force=True, defines=["-DTG_PLAN_PHASES"], out=VARIANT)
    env = dict(os.environ, TANGRAM_GPU_LIB=VARIANT)
    sys.exit(subprocess.call([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))

import ctypes as C  # noqa: E402

from paper_2404_09267_b200 import _native as N  # noqa: E402
from paper_2404_09267_b200 import api as A  # noqa: E402

W, H, n = 3840, 2160, int(sys.argv[1]) if len(sys.argv) > 1 else 300
ctx = A.Context(0)
t_us, rects = A.generate_trace(n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                               roi_proportion_mean=0.10, roi_max_dim=480, seed=1000)
ring = A.FrameRing(ctx, W, H, n)
ring.synthesize(A.derive_seed(1000, "pixels"), rects)
pipe = A.Pipeline(ctx, W, H, max_frames=n, max_canvases=n * 16)
d_cur, d_prev = ring.tables()
d_ids, d_gen = ctx.malloc(8 * n), ctx.malloc(8 * n)
import numpy as np  # noqa: E402
ctx.upload(d_ids, np.arange(n, dtype=np.uint64))
ctx.upload(d_gen, np.array(t_us, np.int64))
lib = N.lib()
lib.tg_debug_plan_phases.argtypes = [C.POINTER(C.c_ulonglong)]
out = (C.c_ulonglong * 16)()
A.check(lib.tg_pipeline_stage_mask(pipe.handle, n, d_cur, d_prev, None))
for _ in range(3):
    A.check(lib.tg_pipeline_stage_plan(pipe.handle, n, d_ids, d_gen, 0, None))
ctx.stream_sync()
lib.tg_debug_plan_phases(out)
reps = 10
for _ in range(reps):
    A.check(lib.tg_pipeline_stage_plan(pipe.handle, n, d_ids, d_gen, 0, None))
ctx.stream_sync()
lib.tg_debug_plan_phases(out)
names = ["", "load activity words", "label run heads", "unions (row above)", "roots + compress",
         "scan + box init", "box fold pass 0 (x, bottom row)", "box fold pass 1 (y, top/bottom rows)",
         "partition accumulate", "partition emit + admission", "BSSF stitch", "publish + jobs",
         "look-back", "ids, ranges, placements"]
ctas = out[0]
tot = sum(out[i] for i in range(1, 14))
print(f"{ctas} frame CTAs; mean {tot / ctas:.0f} cycles per CTA")
for i in range(1, 14):
    print(f"  {names[i]:40s} {out[i] / ctas:9.0f}  {100.0 * out[i] / tot:5.1f} %")
