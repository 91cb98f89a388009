import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2404_09267_b200 import api as A
W, H, n = 3840, 2160, 300
ctx = A.Context(0)
t_us, rects = A.generate_trace(n_frames=n, fps=30.0, frame_width=W, frame_height=H, roi_proportion_mean=0.10, roi_max_dim=480, seed=1000)
ring = A.FrameRing(ctx, W, H, n); ring.synthesize(A.derive_seed(1000, "pixels"), rects)
pipe = A.Pipeline(ctx, W, H, max_frames=n, max_canvases=n * 16)
d_cur, d_prev = ring.tables()
d_ids, d_gen = ctx.malloc(8 * n), ctx.malloc(8 * n)
ctx.upload(d_ids, np.arange(n, dtype=np.uint64)); ctx.upload(d_gen, np.array(t_us, np.int64))
d_canv = ctx.malloc(pipe.canvas_bytes * n * 16)
st = ctx.new_stream()
g = pipe.graph(n, d_cur, d_prev, d_ids, d_gen, 0, d_canv, st)
for name, fn in [("run", lambda: pipe.run(n, d_cur, d_prev, d_ids, d_gen, 0, d_canv, st)), ("graph", lambda: g.launch(st))] * 2:
    for _ in range(5): fn()
    e0, e1 = ctx.event(), ctx.event()
    ctx.stream_sync(st); ctx.record(e0, st)
    for _ in range(40): fn()
    ctx.record(e1, st); ctx.stream_sync(st)
    print(name, ctx.elapsed_ms(e0, e1) / 40, flush=True)

# event overhead inside the step: stage calls with 0 / 2 (around K1) / 4 events per step
from paper_2404_09267_b200 import _native as N
lib = N.lib()
def step(evs):
    if evs: ctx.record(evs[0], st)
    A.check(lib.tg_pipeline_stage_mask(pipe.handle, n, d_cur, d_prev, st))
    if evs: ctx.record(evs[1], st)
    A.check(lib.tg_pipeline_stage_plan(pipe.handle, n, d_ids, d_gen, 0, st))
    if evs and len(evs) > 2: ctx.record(evs[2], st)
    A.check(lib.tg_pipeline_stage_gather(pipe.handle, n, d_cur, d_canv, st))
    if evs and len(evs) > 2: ctx.record(evs[3], st)
for ne in (0, 2, 4, 0, 2, 4):
    evs = [[ctx.event() for _ in range(ne)] for _ in range(40)]
    for _ in range(5): step(None)
    e0, e1 = ctx.event(), ctx.event()
    ctx.stream_sync(st); ctx.record(e0, st)
    for k in range(40): step(evs[k] if ne else None)
    ctx.record(e1, st); ctx.stream_sync(st)
    print("events/step", ne, ctx.elapsed_ms(e0, e1) / 40, flush=True)
