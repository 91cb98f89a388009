"""Debug helper: stage-by-stage K1 check on the 20-frame 4K case."""
import sys, os, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2404_09267_b200 import api as A, _native as N
from tests._helpers import GpuRun

ctx = A.Context(0)
for n in (20, 9, 5):
    run = GpuRun(ctx, 3840, 2160, n, seed=1000)
    lib = N.lib()
    fr0 = [hashlib.md5(f.tobytes()).hexdigest() for f in run.host_frames()]
    A.check(lib.tg_pipeline_stage_mask(run.pipe.handle, n, run.d_cur, run.d_prev, None))
    ctx.stream_sync()
    gm = run.pipe.mask(n)
    fr = run.host_frames()
    bad = []
    for i in range(n):
        om = O.mask(fr[i + 1], fr[i], 3840, 2160, 25, 2)
        d = gm[i] != om
        if d.any():
            rows = np.where(d.any(axis=1))[0]
            bad.append((i, len(rows), rows[:6].tolist(), rows[-3:].tolist()))
    print("n", n, "mask-only bad:", bad[:8], flush=True)
    run.run()
    fr1 = [hashlib.md5(f.tobytes()).hexdigest() for f in run.host_frames()]
    print("frames unchanged after full run:", fr0 == fr1, flush=True)
    run.close()
