"""cfg2 steps with the gather of step i-1 overlapping the planner of step i
(two pipelines, two streams) vs the plain sequential step.  Tuning aid:
prints ms per step of both schedules."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2404_09267_b200 import _native as N  # noqa: E402
from paper_2404_09267_b200 import api as A  # noqa: E402

W, H, n = 3840, 2160, 300
K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ctx = A.Context(0)
t_us, rects = A.generate_trace(n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                               roi_proportion_mean=0.10, roi_max_dim=480, seed=1000)
ring = A.FrameRing(ctx, W, H, n)
ring.synthesize(A.derive_seed(1000, "pixels"), rects)
d_cur, d_prev = ring.tables()
d_ids, d_gen = ctx.malloc(8 * n), ctx.malloc(8 * n)
ctx.upload(d_ids, np.arange(n, dtype=np.uint64))
ctx.upload(d_gen, np.array(t_us, np.int64))
max_canv = n * 4
pipes = [A.Pipeline(ctx, W, H, max_frames=n, max_canvases=max_canv) for _ in range(2)]
canv = [ctx.malloc(pipes[0].canvas_bytes * max_canv) for _ in range(2)]
lib = N.lib()
s1, s2 = ctx.new_stream(high_priority=True), ctx.new_stream()


def wait(stream, ev):
    A.check(lib.tg_stream_wait_event(ctx.handle, stream, ev))


def seq(k):
    p = pipes[0]
    A.check(lib.tg_pipeline_stage_mask(p.handle, n, d_cur, d_prev, s1))
    A.check(lib.tg_pipeline_stage_plan(p.handle, n, d_ids, d_gen, 0, s1))
    A.check(lib.tg_pipeline_stage_gather(p.handle, n, d_cur, canv[0], s1))


def overlapped(steps):
    ev_k1 = [ctx.event() for _ in range(steps + 1)]
    ev_k5 = [ctx.event() for _ in range(steps)]
    ev_end = ctx.event()
    for i in range(steps):
        p = pipes[i % 2]
        if i >= 2:
            wait(s1, ev_k5[i - 2])
        A.check(lib.tg_pipeline_stage_mask(p.handle, n, d_cur, d_prev, s1))
        ctx.record(ev_k1[i], s1)
        if i >= 1:
            q = pipes[(i - 1) % 2]
            wait(s2, ev_k1[i])
            A.check(lib.tg_pipeline_stage_gather(q.handle, n, d_cur, canv[(i - 1) % 2], s2))
            ctx.record(ev_k5[i - 1], s2)
        A.check(lib.tg_pipeline_stage_plan(p.handle, n, d_ids, d_gen, 0, s1))
    ctx.record(ev_k1[steps], s1)
    wait(s2, ev_k1[steps])
    q = pipes[(steps - 1) % 2]
    A.check(lib.tg_pipeline_stage_gather(q.handle, n, d_cur, canv[(steps - 1) % 2], s2))
    ctx.record(ev_end, s2)
    wait(s1, ev_end)


for name in ["seq", "overlap", "seq", "overlap"]:
    for _ in range(3):
        seq(0)
    ctx.synchronize()
    e0, e1 = ctx.event(), ctx.event()
    ctx.record(e0, s1)
    if name == "seq":
        for k in range(K):
            seq(k)
    else:
        overlapped(K)
    ctx.record(e1, s1)
    ctx.synchronize()
    print(f"{name:8s} {ctx.elapsed_ms(e0, e1) / K:.4f} ms/step", flush=True)
# the overlapped canvases equal the sequential ones
ctx.synchronize()
seq(0)
ctx.synchronize()
r0 = pipes[0].results(n)
tot = int(r0["total_canvases"])
a = ctx.download(canv[0], (tot, pipes[0].canvas_bytes), np.uint8)
overlapped(3)
ctx.synchronize()
b = ctx.download(canv[0], (tot, pipes[0].canvas_bytes), np.uint8)
c = ctx.download(canv[1], (tot, pipes[0].canvas_bytes), np.uint8)
print("canvases equal:", bool(np.array_equal(a, b) and np.array_equal(a, c)), tot)
