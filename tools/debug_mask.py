"""Debug helper: where do GPU and oracle masks differ (test infrastructure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2404_09267_b200 import api as A
from tests._helpers import GpuRun

ctx = A.Context(0)
for (W, H, n, r) in [(3840, 2160, 2, 2), (3840, 256, 2, 2), (1920, 2160, 2, 2), (3840, 2160, 2, 0), (3840, 2160, 1, 2), (2560, 512, 2, 2), (3072, 512, 2, 2)]:
    run = GpuRun(ctx, W, H, n, seed=1000, radius=r)
    gpu = run.run()
    gm = run.pipe.mask(n)
    fr = run.host_frames()
    for i in range(n):
        om = O.mask(fr[i + 1], fr[i], W, H, 25, r)
        d = gm[i] != om
        if d.any():
            rows = np.where(d.any(axis=1))[0]
            cols = np.where(d.any(axis=0))[0]
            extra = int((gm[i] & ~om)[d].astype(bool).sum())
            missing = int((om & ~gm[i])[d].astype(bool).sum())
            print(W, H, r, "frame", i, "rows", len(rows), rows[:10], "cols", cols[:20], "extra", extra, "missing", missing, flush=True)
        else:
            print(W, H, r, "frame", i, "OK", flush=True)
    run.close()
