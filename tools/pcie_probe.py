"""Host->device bandwidth from pinned memory (one stream, and two streams in
parallel) -- the ceiling of the e2e figure.  Tuning aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09267_b200 import api as A  # noqa: E402

ctx = A.Context(0)
GB = 1 << 30
n = 2 * GB
h = ctx.malloc_host(n)
d = ctx.malloc(n)
s1, s2 = ctx.new_stream(), ctx.new_stream()
e0, e1 = ctx.event(), ctx.event()
for name, parts in (("1 stream", 1), ("2 streams", 2), ("4 streams", 4)):
    streams = [ctx.new_stream() for _ in range(parts)]
    for rep in range(3):
        ctx.synchronize()
        ctx.record(e0, streams[0])
        evs = []
        for k, st in enumerate(streams):
            if k:
                A.check(ctx._lib.tg_stream_wait_event(ctx.handle, st, e0))
            ctx.memcpy(d + k * (n // parts), h + k * (n // parts), n // parts, 0, st)
            ev = ctx.event()
            ctx.record(ev, st)
            evs.append(ev)
        for ev in evs[1:]:
            A.check(ctx._lib.tg_stream_wait_event(ctx.handle, streams[0], ev))
        ctx.record(e1, streams[0])
        ctx.stream_sync(streams[0])
    ms = ctx.elapsed_ms(e0, e1)
    print(f"H2D {name}: {n / ms / 1e6:.1f} GB/s", flush=True)
