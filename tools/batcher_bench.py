"""Host-side timing of the config-4 batcher (no GPU needed): 64 4K cameras x
30 frames of patches (oracle partition of generate_trace rects, enlarged like
the pixel path's dilated unions), ids renumbered, uplinks + SLO batcher
replayed through tg_batcher_replay_links, and the event plans built by
tg_batcher_plan_all -- the host work one config-4 step does.  Tuning aid."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (test infrastructure: patch source only)
from paper_2404_09267_b200 import api as A  # noqa: E402
from paper_2404_09267_b200 import multicam as MC  # noqa: E402
import bench  # noqa: E402

W, H = 3840, 2160
ncam, n = (5, 300) if (len(sys.argv) > 1 and sys.argv[1] == "cfg3") else (64, 30)
recs = []
for c in range(ncam):
    t_us, rects = O.generate_trace(O.gen_cfg(n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                                             roi_proportion_mean=0.10, roi_max_dim=480,
                                             seed=O.derive_seed(1000 + c, "trace")))
    for f in range(n):
        rois = [(max(0, x - 8), max(0, y - 8), min(W - max(0, x - 8), w + 16),
                 min(H - max(0, y - 8), h + 16)) for (x, y, w, h) in rects[f]]
        for p in O.partition(f, W, H, t_us[f], 1_000_000, 4, 4, rois, 1.5):
            r = np.zeros(1, MC.DESC_DTYPE)
            pp = r["patch"]
            pp["patch_id"], pp["source_frame_id"] = p["patch_id"], p["source_frame_id"]
            pp["x"], pp["y"], pp["w"], pp["h"] = p["rect"]
            pp["generation_time_us"], pp["slo_us"] = p["generation_time_us"], p["slo_us"]
            pp["deadline_us"], pp["size_bytes"] = p["deadline_us"], p["size_bytes"]
            r["patch"] = pp
            r["camera"], r["frame"] = c, f
            r["admitted"] = int(p["rect"][2] <= 1024 and p["rect"][3] <= 1024)
            recs.append(r)
desc = np.concatenate(recs)
prof = A.LatencyProfile(1024, 1024, bench.SIM_PROFILE)
sched = A.SloScheduler(A.CanvasSpec(1024, 1024), prof, A.max_canvases_per_batch(80.0, 4.0, 1.0))
for it in range(5):
    t0 = time.perf_counter()
    nev, arr, plan = MC.schedule_descriptors(sched, desc, range(ncam), n, bench.SIM_BANDWIDTH_MBPS)
    t1 = time.perf_counter()
    print(f"patches {len(desc)} admitted {len(plan['patches'])} events {nev}  "
          f"schedule {1e3 * (t1 - t0):.2f} ms", flush=True)
if "--split" in sys.argv:
    import ctypes as C
    from paper_2404_09267_b200 import _native as N
    d = np.array(desc, copy=True)
    d["patch"]["patch_id"] = np.arange(len(d), dtype=np.uint64)
    adm = d[d["admitted"] != 0]
    offs = np.zeros(ncam + 1, np.int32)
    offs[1:] = np.cumsum(np.bincount(adm["camera"], minlength=ncam))
    src = (adm["camera"] * (n + 1) + adm["frame"] + 1).astype(np.int32)
    patches = np.ascontiguousarray(adm["patch"])
    arrival = np.zeros(len(patches), np.int64)
    nev = C.c_int32()
    for it in range(3):
        t0 = time.perf_counter()
        A.check(N.lib().tg_batcher_replay_links(sched.handle, ncam, offs.ctypes.data,
                                                patches.ctypes.data, src.ctypes.data,
                                                float(bench.SIM_BANDWIDTH_MBPS), 1,
                                                arrival.ctypes.data, C.byref(nev)))
        t1 = time.perf_counter()
        print(f"replay_links alone {1e3 * (t1 - t0):.2f} ms", flush=True)
if "--dump" in sys.argv:
    patches.tofile("/tmp/bh/patches.bin")
    src.tofile("/tmp/bh/src.bin")
    offs.tofile("/tmp/bh/offs.bin")
    print("dumped", len(patches), ncam)
