"""Micro-benchmarks of plain memset / D2D copy on the device (roofline context)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09267_b200 import api as A
ctx = A.Context(0)
GB = 1 << 30
a = ctx.malloc(3 * GB); b = ctx.malloc(3 * GB)
e0, e1 = ctx.event(), ctx.event()
for name, fn, nbytes in [("memset 2.8GB", lambda: ctx.memset(a, 0, int(2.8e9)), 2.8e9),
                         ("d2d copy 1.5GB (r+w)", lambda: ctx.memcpy(b, a, int(1.5e9), 2), 3.0e9),
                         ("d2d copy 3GB (r+w)", lambda: ctx.memcpy(b, a, 3 * GB, 2), 6 * GB)]:
    for _ in range(3): fn()
    ctx.record(e0)
    for _ in range(10): fn()
    ctx.record(e1); ctx.stream_sync()
    ms = ctx.elapsed_ms(e0, e1) / 10
    print(f"{name}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
