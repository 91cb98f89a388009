"""Multi-camera frame->canvas path (BASELINE configs 3 and 4).

One GPU holds a shard of cameras.  Per step:

1. every camera's frames run through K1 (mask/cells) and K2-K4 (RoIs,
   partition, per-frame plan) on the device -- the per-frame canvases are not
   materialized, the batcher decides canvases across cameras;
2. the patch descriptors (64 B each) come back to the host -- a few hundred
   KB, never pixels;
3. patch ids are renumbered camera-major (sim.hpp:249-251), admission applied
   (sim.hpp:262), per-camera uplink arrivals computed (trace.hpp:255-267) and
   the SLO batcher replays the reference event loop (sim.hpp:334-458);
4. every invoke event's canvases are written by one K5 launch straight from
   the device-resident frames of all cameras.

Across GPUs (config 4) cameras are sharded in contiguous blocks (camera c on
rank floor(c*G/n)); canvases are shard-local, and the descriptors are
all-gathered (NCCL through torch.distributed) so every rank holds the global
patch list in reference order (`gather_descriptors`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .api import (CanvasSpec, Context, FrameRing, LatencyProfile, Pipeline, check, derive_seed,
                  generate_trace, max_canvases_per_batch)

# tg_patch_meta as a numpy record (64 bytes)
PATCH_DTYPE = np.dtype([("patch_id", "<u8"), ("source_frame_id", "<u8"), ("x", "<i4"),
                        ("y", "<i4"), ("w", "<i4"), ("h", "<i4"), ("generation_time_us", "<i8"),
                        ("slo_us", "<i8"), ("deadline_us", "<i8"), ("size_bytes", "<i8")])
assert PATCH_DTYPE.itemsize == 64

# descriptor record exchanged between ranks: patch + camera + admission
DESC_DTYPE = np.dtype([("patch", PATCH_DTYPE), ("camera", "<i4"), ("frame", "<i4"),
                       ("admitted", "<i4"), ("pad", "<i4")])


def shard_cameras(n_cams: int, world: int, rank: int) -> list[int]:
    """Camera c runs on rank floor(c * world / n_cams) (contiguous blocks)."""
    return [c for c in range(n_cams) if (c * world) // n_cams == rank]


class MultiCameraPath:
    def __init__(self, ctx: Context, cameras, width, height, n_frames, profile, bandwidth_mbps=80.0,
                 gpu_memory_gb=6.0, model_size_gb=2.0, canvas=(1024, 1024), zones=(4, 4),
                 slo_us=1_000_000, fps=30.0, per_camera_link=True, trace_kw=None,
                 canvas_capacity=None):
        self.ctx, self.cameras, self.W, self.H, self.n = ctx, list(cameras), width, height, n_frames
        self.canvas = canvas
        self.bandwidth, self.per_camera_link = bandwidth_mbps, per_camera_link
        trace_kw = dict(trace_kw or {})
        self.rings, self.pipes, self.tables, self.t_us, self.rects = [], [], [], [], []
        self.d_ids, self.d_gen = [], []
        for c in self.cameras:
            t_us, rects = generate_trace(n_frames=n_frames, fps=fps, frame_width=width,
                                         frame_height=height, seed=1000 + c, **trace_kw)
            ring = FrameRing(ctx, width, height, n_frames)
            ring.synthesize(derive_seed(1000 + c, "pixels"), rects)
            pipe = Pipeline(ctx, width, height, max_frames=n_frames, max_canvases=0, zones=zones,
                            canvas=canvas, slo_us=slo_us)
            self.rings.append(ring)
            self.pipes.append(pipe)
            self.tables.append(ring.tables())
            self.t_us.append(t_us)
            self.rects.append(rects)
            d_ids, d_gen = ctx.malloc(8 * n_frames), ctx.malloc(8 * n_frames)
            ctx.upload(d_ids, np.arange(n_frames, dtype=np.uint64))
            ctx.upload(d_gen, np.array(t_us, np.int64))
            self.d_ids.append(d_ids)
            self.d_gen.append(d_gen)
        self.zones = self.pipes[0].zones if self.pipes else zones[0] * zones[1]
        # one device table of every frame of every camera: index cam*(n+1) + slot
        ptrs = np.array([s for ring in self.rings for s in ring.slots], np.uint64)
        self.d_frames = ctx.malloc(8 * max(1, len(ptrs)))
        ctx.upload(self.d_frames, ptrs)
        self.profile = LatencyProfile(canvas[0], canvas[1], profile)
        self.max_canvases = max_canvases_per_batch(gpu_memory_gb, model_size_gb, 1.0)
        from .api import SloScheduler
        self.sched = SloScheduler(CanvasSpec(*canvas), self.profile, self.max_canvases)
        self.canvas_bytes = canvas[0] * canvas[1] * 3
        self.canvas_cap = canvas_capacity
        self.d_canvases = None
        self.stream = ctx.new_stream()
        self._pat = np.zeros(len(self.cameras) * n_frames * self.zones, PATCH_DTYPE)
        self._adm = np.zeros(len(self.cameras) * n_frames * self.zones, np.uint8)
        self._np = np.zeros(len(self.cameras) * n_frames, np.int32)

    def close(self):
        for p in self.pipes:
            p.close()
        for r in self.rings:
            r.close()
        for p in self.d_ids + self.d_gen + [self.d_frames]:
            self.ctx.free(p)
        if self.d_canvases:
            self.ctx.free(self.d_canvases)
        self.sched.close()

    # ---- 1. device: K1-K4 for every camera --------------------------------
    def run_planes(self):
        lib = N.lib()
        for k, pipe in enumerate(self.pipes):
            d_cur, d_prev = self.tables[k]
            check(lib.tg_pipeline_stage_mask(pipe.handle, self.n, d_cur, d_prev, self.stream))
            check(lib.tg_pipeline_stage_plan(pipe.handle, self.n, self.d_ids[k], self.d_gen[k], 0,
                                             self.stream))

    # ---- 2. descriptors to the host ----------------------------------------
    def descriptors(self) -> np.ndarray:
        """DESC_DTYPE records of every patch of the shard, camera-major,
        frame order, zone order (ids still camera-local)."""
        n, Z = self.n, self.zones
        for k, pipe in enumerate(self.pipes):
            v = pipe.views
            self.ctx.memcpy(self._pat[k * n * Z:].ctypes.data, v.patches, n * Z * 64, 1, self.stream)
            self.ctx.memcpy(self._adm[k * n * Z:].ctypes.data, v.admitted, n * Z, 1, self.stream)
            self.ctx.memcpy(self._np[k * n:].ctypes.data, v.n_patches, n * 4, 1, self.stream)
        self.ctx.stream_sync(self.stream)
        counts = self._np.reshape(len(self.pipes), n)
        valid = (np.arange(Z)[None, None, :] < counts[:, :, None]).reshape(-1)
        out = np.zeros(int(valid.sum()), DESC_DTYPE)
        out["patch"] = self._pat[valid]
        cams = np.repeat(np.array(self.cameras, np.int32), n * Z)[valid]
        frames = np.tile(np.repeat(np.arange(n, dtype=np.int32), Z), len(self.pipes))[valid]
        out["camera"], out["frame"], out["admitted"] = cams, frames, self._adm[valid]
        return out

    # ---- 3. host: ids, admission, links, batcher ----------------------------
    def schedule(self, desc: np.ndarray):
        """Renumbers patch ids camera-major, keeps admitted patches and
        replays the batcher; returns the number of invoke events."""
        self._nev, self.arrival, self._last = schedule_descriptors(
            self.sched, desc, self.cameras, self.n, self.bandwidth, self.per_camera_link)
        return self._nev

    # ---- 4. device: every event's canvases ----------------------------------
    def gather(self) -> int:
        if self.d_canvases is None:
            cap = self.canvas_cap or max(1, len(self._last["patches"]))
            self.canvas_cap = cap
            self.d_canvases = self.ctx.malloc(cap * self.canvas_bytes)
        n = C.c_int64()
        check(N.lib().tg_batcher_gather_all(self.ctx.handle, self.sched.handle, self.d_frames,
                                            3 * self.W, self.d_canvases, self.canvas_cap,
                                            C.byref(n), self.stream))
        return n.value

    def step(self):
        self.run_planes()
        desc = self.descriptors()
        n_events = self.schedule(desc)
        n_canvases = self.gather()
        return desc, n_events, n_canvases

    def events(self):
        """InvokeEvents of the last step (readable until the next batcher call)."""
        return self.sched._events(self._nev)

    def canvases(self, count: int) -> np.ndarray:
        return self.ctx.download(self.d_canvases, (count, self.canvas[1], self.canvas[0] * 3),
                                 np.uint8, self.stream)


def schedule_descriptors(sched, desc: np.ndarray, cameras, n_frames: int, bandwidth_mbps: float,
                         per_camera_link: bool = True):
    """Host half of configs 3/4 on DESC_DTYPE records (camera-major, frame
    and zone order): ids renumbered camera-major over all patches
    (sim.hpp:249-251), admitted ones (sim.hpp:262) sent over the uplinks and
    replayed through `sched` (an api.SloScheduler).  Returns (number of
    events, arrival times of the admitted patches, plan dict)."""
    d = np.array(desc, copy=True)
    d["patch"]["patch_id"] = np.arange(len(d), dtype=np.uint64)
    adm = d[d["admitted"] != 0]
    cams = np.asarray(list(cameras), np.int64)
    lut = np.full(int(cams.max()) + 1 if len(cams) else 1, -1, np.int32)
    lut[cams] = np.arange(len(cams), dtype=np.int32)
    cam_slot = lut[adm["camera"]]
    offs = np.zeros(len(cams) + 1, np.int32)
    offs[1:] = np.cumsum(np.bincount(cam_slot, minlength=len(cams)))
    src = (cam_slot * (n_frames + 1) + adm["frame"] + 1).astype(np.int32)
    patches = np.ascontiguousarray(adm["patch"])
    arrival = np.zeros(max(1, len(patches)), np.int64)
    n_ev = C.c_int32()
    check(N.lib().tg_batcher_replay_links(sched.handle, len(cams), offs.ctypes.data,
                                          patches.ctypes.data, src.ctypes.data,
                                          float(bandwidth_mbps), int(per_camera_link),
                                          arrival.ctypes.data, C.byref(n_ev)))
    return n_ev.value, arrival[:len(patches)], dict(patches=patches, src=src, offs=offs)


def gather_descriptors(local: np.ndarray, dist, device=None) -> np.ndarray:
    """All-gathers every rank's DESC_DTYPE records (variable counts) and
    returns them camera-major -- the global patch list in reference order.
    `dist` is torch.distributed (NCCL on GPUs, gloo on CPU)."""
    import torch
    world = dist.get_world_size()
    raw = torch.from_numpy(local.view(np.uint8).copy())
    if device is not None:
        raw = raw.to(device)
    n = torch.tensor([raw.numel()], dtype=torch.int64, device=raw.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    cap = int(max(s.item() for s in sizes))
    buf = torch.zeros(cap, dtype=torch.uint8, device=raw.device)
    buf[:raw.numel()] = raw
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    recs = [p[:int(s.item())].cpu().numpy().view(DESC_DTYPE) for p, s in zip(parts, sizes)]
    allrec = np.concatenate(recs) if recs else np.zeros(0, DESC_DTYPE)
    order = np.lexsort((np.arange(len(allrec)), allrec["camera"]))  # stable, camera-major
    return allrec[order]
