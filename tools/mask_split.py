"""Times the mask stage of the cfg2 workload three ways on one GPU: the
fused launch (K1 + K1b tasks, tg_pipeline_stage_mask), K1 alone
(tg_pipeline_stage_mask_fg), K1b alone (tg_pipeline_stage_mask_cells) and
the two back to back ("split").
Tuning aid; CUDA events on the launching stream, mean of N launches."""
import sys

import numpy as np

sys.path.insert(0, ".")
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
lib, st = N.lib(), ctx.new_stream()
calls = {
    "fused": lambda: A.check(lib.tg_pipeline_stage_mask(pipe.handle, n, d_cur, d_prev, st)),
    "k1": lambda: A.check(lib.tg_pipeline_stage_mask_fg(pipe.handle, n, d_cur, d_prev, st)),
    "k1b": lambda: A.check(lib.tg_pipeline_stage_mask_cells(pipe.handle, n, st)),
}
calls["split"] = lambda: (calls["k1"](), calls["k1b"]())
which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fused", "k1", "k1b"]
for name, fn in [(k, calls[k]) for k in which] * 2:
    for _ in range(3):
        fn()
    e0, e1 = ctx.event(), ctx.event()
    ctx.stream_sync(st)
    ctx.record(e0, st)
    for _ in range(20):
        fn()
    ctx.record(e1, st)
    ctx.stream_sync(st)
    print(f"{name:6s} {ctx.elapsed_ms(e0, e1) / 20:.4f} ms", flush=True)
