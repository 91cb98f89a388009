"""Debug helper: characterize bad rows (test infrastructure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2404_09267_b200 import api as A, _native as N
from tests._helpers import GpuRun

def bits(m, W):
    return np.unpackbits(m.view(np.uint8), bitorder="little").reshape(m.shape[0], -1)[:, :W].astype(bool)

def dil(f0, r):
    H, W = f0.shape
    out = np.zeros_like(f0)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            ys, ye = max(0, dy), H + min(0, dy)
            xs, xe = max(0, dx), W + min(0, dx)
            out[ys - dy:ye - dy, xs - dx:xe - dx] |= f0[ys:ye, xs:xe]
    return out

ctx = A.Context(0)
W, H, n = 3840, 2160, 6
run = GpuRun(ctx, W, H, n, seed=1000)
lib = N.lib()
A.check(lib.tg_pipeline_stage_mask(run.pipe.handle, n, run.d_cur, run.d_prev, None))
ctx.stream_sync()
gm = run.pipe.mask(n)
fr = run.host_frames()
for i in range(n):
    f0 = bits(O.mask(fr[i + 1], fr[i], W, H, 25, 0), W)
    g = bits(gm[i], W)
    o = dil(f0, 2)
    bad = np.where((g != o).any(axis=1))[0]
    for y in bad[:4]:
        # hypothesis: look-ahead rows treated as zero
        f0z = f0.copy(); f0z[y + 1:] = False
        hz = dil(f0z, 2)[y]
        # hypothesis: dilation without rows below? above?
        print("frame", i, "row", y, "extra", int((g[y] & ~o[y]).sum()), "missing", int((o[y] & ~g[y]).sum()),
              "eq_zero_lookahead", bool((hz == g[y]).all()),
              "eq_fg0_row", bool((f0[y] == g[y]).all()), flush=True)
        cols = np.where(g[y] != o[y])[0]
        print("   cols", cols[:12], "gpu row bits", np.where(g[y])[0][:8], "orc", np.where(o[y])[0][:8])
run.close()
