"""Debug helper: K1 alone vs oracle for several radii / grids (test infrastructure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2404_09267_b200 import api as A, _native as N
from tests._helpers import GpuRun
ctx = A.Context(0)
W, H, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
for r in (0, 1, 2, 4):
    run = GpuRun(ctx, W, H, n, seed=1000, radius=r)
    A.check(N.lib().tg_pipeline_stage_mask(run.pipe.handle, n, run.d_cur, run.d_prev, None))
    ctx.stream_sync()
    gm = run.pipe.mask(n)
    fr = run.host_frames()
    bad = []
    for i in range(n):
        d = gm[i] != O.mask(fr[i + 1], fr[i], W, H, 25, r)
        if d.any():
            bad.append((i, np.where(d.any(axis=1))[0][:4].tolist()))
    print(W, H, n, "r", r, "bad", len(bad), bad[:4], flush=True)
    run.close()
