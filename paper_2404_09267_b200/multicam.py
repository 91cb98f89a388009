"""Multi-camera frame->canvas path (BASELINE configs 3 and 4).

One GPU holds a shard of cameras.  Per step:

1. every camera's frames run through K1 (mask/cells) and K2-K4 (RoIs,
   partition, per-frame plan) on the device -- the per-frame canvases are not
   materialized, the batcher decides canvases across cameras;
2. the planner writes every patch as a dense 80-byte descriptor on the
   device (its frame-order look-back prefix is the compaction scan); the
   descriptor block comes back to the host -- a few hundred KB, never
   pixels;
3. patch ids are renumbered camera-major (sim.hpp:249-251), admission applied
   (sim.hpp:262), per-camera uplink arrivals computed (trace.hpp:255-267) and
   the SLO batcher replays the reference event loop (sim.hpp:334-458);
4. every invoke event's canvases are written by one K5 launch straight from
   the device-resident frames of all cameras.

Across GPUs (config 4) cameras are sharded in contiguous blocks (camera c on
rank floor(c*G/n)); canvases are shard-local, and the device descriptor
blocks are all-gathered by the C ABI's communicator (api.Comm: NCCL on the
device blocks, or a host transport) so every rank holds the global patch
list in reference order.
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


def block_bytes(cap: int) -> int:
    """Bytes of one descriptor block (tg_descriptor_header + cap records)."""
    return int(N.lib().tg_descriptor_block_bytes(cap))


def descriptor_block(records: np.ndarray, cap: int) -> np.ndarray:
    """Host descriptor block (header + cap records) holding `records`."""
    records = np.ascontiguousarray(records, DESC_DTYPE)
    if len(records) > cap:
        raise ValueError(f"{len(records)} records exceed the block capacity {cap}")
    blk = np.zeros(block_bytes(cap), np.uint8)
    blk[:16].view(np.int64)[:] = (len(records), cap)
    blk[DESC_DTYPE.itemsize:DESC_DTYPE.itemsize * (1 + len(records))] = records.view(np.uint8)
    return blk


def flatten_blocks(ptr: int, n_blocks: int, cap: int, out: np.ndarray | None = None) -> np.ndarray:
    """Valid records of n_blocks consecutive blocks at host address `ptr`,
    rank-major (tg_descriptor_blocks_flatten)."""
    if out is None:
        out = np.zeros(max(1, n_blocks * cap), DESC_DTYPE)
    n = C.c_int64()
    check(N.lib().tg_descriptor_blocks_flatten(ptr, n_blocks, cap, out.ctypes.data, len(out),
                                               C.byref(n)))
    return out[:n.value]


def allgather_descriptors(comm, records: np.ndarray, cap: int) -> np.ndarray:
    """All-gathers every rank's host descriptor records through `comm`
    (api.Comm) as blocks of `cap` records (equal on every rank) and returns
    them rank-major -- camera-major under contiguous sharding."""
    blk = descriptor_block(records, cap)
    world = comm.world
    if comm.on_device:
        ctx, nb = comm.ctx, blk.nbytes
        d_send, d_recv = ctx.malloc(nb), ctx.malloc(nb * world)
        ctx.upload(d_send, blk)
        comm.allgather(d_send, nb, d_recv, ctx.stream)
        got = ctx.download(d_recv, (world * nb,), np.uint8)
        ctx.free(d_send)
        ctx.free(d_recv)
    else:
        got = np.zeros(blk.nbytes * world, np.uint8)
        comm.allgather(blk.ctypes.data, blk.nbytes, got.ctypes.data)
    return flatten_blocks(got.ctypes.data, world, cap).copy()


class MultiCameraPath:
    def __init__(self, ctx: Context, cameras, width, height, n_frames, profile, bandwidth_mbps=80.0,
                 gpu_memory_gb=6.0, model_size_gb=2.0, canvas=(1024, 1024), zones=(4, 4),
                 slo_us=1_000_000, fps=30.0, per_camera_link=True, trace_kw=None,
                 canvas_capacity=None, comm=None, cameras_per_rank=None, gather_grid=None):
        """`comm` (api.Comm, optional): every pass all-gathers the ranks'
        descriptor blocks through it; blocks hold `cameras_per_rank` (the
        largest shard; equal on every rank) x n_frames x zones records."""
        self.ctx, self.cameras, self.W, self.H, self.n = ctx, list(cameras), width, height, n_frames
        self.canvas = canvas
        self.bandwidth, self.per_camera_link = bandwidth_mbps, per_camera_link
        self.comm = comm
        trace_kw = dict(trace_kw or {})
        self.rings, self.t_us, self.rects = [], [], []
        for c in self.cameras:
            t_us, rects = generate_trace(n_frames=n_frames, fps=fps, frame_width=width,
                                         frame_height=height, seed=1000 + c, **trace_kw)
            ring = FrameRing(ctx, width, height, n_frames)
            ring.synthesize(derive_seed(1000 + c, "pixels"), rects)
            self.rings.append(ring)
            self.t_us.append(t_us)
            self.rects.append(rects)
        # ONE pipeline over the frames of every camera of the shard, camera-major:
        # frame k*n + i is camera k's frame i, its predecessor that camera's slot i
        # (K1 restarts the frame chain at each camera boundary), so the shard's
        # masks, cells and plans take one K1 and one K2-K4 launch per step.
        F = max(1, len(self.cameras) * n_frames)
        self.pipe = Pipeline(ctx, width, height, max_frames=F, max_canvases=0, zones=zones,
                             canvas=canvas, slo_us=slo_us)
        cur = np.array([r.slots[1 + i] for r in self.rings for i in range(n_frames)], np.uint64)
        prev = np.array([r.slots[i] for r in self.rings for i in range(n_frames)], np.uint64)
        ids = np.tile(np.arange(n_frames, dtype=np.uint64), len(self.cameras))
        gen = np.array([t for t_us in self.t_us for t in t_us], np.int64)
        self.d_cur, self.d_prev, self.d_ids, self.d_gen = (ctx.malloc(8 * F) for _ in range(4))
        if len(cur):
            for d, a in ((self.d_cur, cur), (self.d_prev, prev), (self.d_ids, ids),
                         (self.d_gen, gen)):
                ctx.upload(d, a)
        self.zones = self.pipe.zones
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
        # the event gather's persistent grid (default 2 CTAs per SM) leaves room
        # for the next pass's K1b and planner CTAs
        check(N.lib().tg_ctx_set_option(ctx.handle, N.TG_OPT_GATHER_GRID,
                                        gather_grid if gather_grid is not None
                                        else 2 * ctx.sm_count()))
        # the planner's dense descriptor block (device), gathered per pass
        self.world = comm.world if comm is not None else 1
        self.cap = max(1, (cameras_per_rank or len(self.cameras))) * n_frames * self.zones
        self.bb = block_bytes(self.cap)
        self.d_block = ctx.malloc(self.bb)
        self.d_cams = ctx.malloc(4 * max(1, len(self.cameras)))
        if self.cameras:
            ctx.upload(self.d_cams, np.array(self.cameras, np.int32))
        self.pipe.set_descriptor_output(self.d_block, self.cap, self.d_cams, n_frames)
        self.d_blocks = ctx.malloc(self.world * self.bb) if comm is not None and comm.on_device \
            else None
        # K1-K4 and the descriptor read-back; high priority, so pass i+1's
        # planner CTAs run ahead of pass i's pending K5 CTAs and the host gets
        # the descriptors without waiting for the gather
        self.stream = ctx.new_stream(high_priority=True)
        self.gstream = ctx.new_stream()  # K5 (event canvases)
        self._gdone = ctx.event()
        # pinned landing zone of the read-back, two of them: pass i+1's
        # read-back lands while pass i's is scheduled
        self._hslot = self.world * self.bb
        self._h = ctx.malloc_host(2 * self._hslot)
        self._fetched = [ctx.event(), ctx.event()]
        self._desc = np.zeros(self.world * self.cap, DESC_DTYPE)
        self._nev, self._last = 0, {"patches": np.zeros(0, PATCH_DTYPE)}

    def close(self):
        self.pipe.close()
        for r in self.rings:
            r.close()
        for p in (self.d_cur, self.d_prev, self.d_ids, self.d_gen, self.d_frames, self.d_block,
                  self.d_cams):
            self.ctx.free(p)
        if self.d_blocks:
            self.ctx.free(self.d_blocks)
        if self.d_canvases:
            self.ctx.free(self.d_canvases)
        self.ctx.free_host(self._h)
        self.sched.close()

    # ---- 1. device: K1-K4 for every camera, descriptors on the device -------
    def run_planes(self, mask_events=None):
        """`mask_events` (optional (start, stop) CUDA events) bracket K1 on
        `stream`."""
        lib, F = N.lib(), len(self.cameras) * self.n
        if mask_events:
            self.ctx.record(mask_events[0], self.stream)
        # K1 on every SM, then K1b as its own kernel: the previous pass's event
        # gather (K5, capped at 2 CTAs per SM) leaves room for K1b's and the
        # planner's CTAs, so they co-run with it instead of K1b running as the
        # fused launch's tail (cfg4: 11.86 -> 11.66 ms per pass)
        check(lib.tg_pipeline_stage_mask_fg(self.pipe.handle, F, self.d_cur, self.d_prev,
                                            self.stream))
        if mask_events:
            self.ctx.record(mask_events[1], self.stream)
        check(lib.tg_pipeline_stage_mask_cells(self.pipe.handle, F, self.stream))
        check(lib.tg_pipeline_stage_plan(self.pipe.handle, F, self.d_ids, self.d_gen, 0,
                                         self.stream))

    # ---- 2. descriptor blocks: all-gather (NCCL) and read-back ---------------
    def fetch_descriptors(self, slot: int = 0):
        """Enqueues, on `stream` after the planes: the NCCL all-gather of the
        ranks' device blocks (device communicator) and the read-back of the
        gathered blocks -- or of this rank's block -- into pinned slot `slot`."""
        h = self._h + slot * self._hslot
        if self.d_blocks is not None:
            check(N.lib().tg_descriptors_allgather(self.comm.handle, self.d_block, self.cap,
                                                   self.d_blocks, self.stream))
            self.ctx.memcpy(h, self.d_blocks, self.world * self.bb, 1, self.stream)
        else:
            self.ctx.memcpy(h, self.d_block, self.bb, 1, self.stream)
        self.ctx.record(self._fetched[slot], self.stream)

    def compact_descriptors(self, slot: int = 0) -> np.ndarray:
        """Waits for read-back `slot` and returns the gathered records
        (DESC_DTYPE, rank-major = camera-major); with a host communicator the
        ranks' blocks are exchanged here.  The view is valid until the next
        call."""
        self.ctx.event_sync(self._fetched[slot])
        h = self._h + slot * self._hslot
        if self.comm is not None and self.d_blocks is None:  # host transport
            mine = C.string_at(h, self.bb)
            C.memmove(h, b"".join(self.comm.allgather_bytes(mine)), self._hslot)
        return flatten_blocks(h, self.world, self.cap, self._desc)

    def descriptors(self) -> np.ndarray:
        """DESC_DTYPE records of every patch of every rank's shard (this
        shard's alone without a communicator), camera-major, frame order,
        zone order (ids numbered per shard; `schedule` renumbers them over
        the whole camera set).  Waits for the planes."""
        self.fetch_descriptors(0)
        return self.compact_descriptors(0)

    # ---- 3. host: ids, admission, links, batcher ----------------------------
    def schedule(self, desc: np.ndarray):
        """Renumbers patch ids camera-major, keeps this shard's admitted
        patches and replays the batcher; returns the number of invoke events."""
        self._nev, self.arrival, self._last = schedule_descriptors(
            self.sched, desc, self.cameras, self.n, self.bandwidth, self.per_camera_link)
        return self._nev

    # ---- 4. device: every event's canvases ----------------------------------
    def gather(self, join: bool = True) -> int:
        """Writes every event's canvases (one K5 launch on `gstream`); with
        `join`, `stream` waits for them (so syncing `stream` covers them)."""
        if self.d_canvases is None:
            cap = self.canvas_cap or max(1, len(self._last["patches"]))
            self.canvas_cap = cap
            self.d_canvases = self.ctx.malloc(cap * self.canvas_bytes)
        n = C.c_int64()
        check(N.lib().tg_batcher_gather_all(self.ctx.handle, self.sched.handle, self.d_frames,
                                            3 * self.W, self.d_canvases, self.canvas_cap,
                                            C.byref(n), self.gstream))
        if join:
            self.join()
        return n.value

    def join(self):
        """Orders `stream` after every gather issued so far."""
        self.ctx.record(self._gdone, self.gstream)
        check(N.lib().tg_stream_wait_event(self.ctx.handle, self.stream, self._gdone))

    def run_pipelined(self, steps: int, mask_events=None) -> int:
        """`steps` passes over the shard's frames with the host batcher of
        pass i overlapping the device planes (K1-K4) of pass i+1, which are
        queued behind pass i's descriptor all-gather and read-back
        (double-buffered pinned memory), so the device never waits for the
        host; K5 of pass i runs on `gstream`.  mask_events[i] (optional
        (start, stop) pair or None) brackets pass i's mask launch.  Returns
        the last pass's canvas count; `stream` is joined with every gather."""
        n_canv = 0
        ev = (lambda i: mask_events[i] if mask_events else None)
        self.run_planes(ev(0))
        self.fetch_descriptors(0)
        for i in range(steps):
            if i + 1 < steps:  # queued behind pass i's read-back: no host wait in between
                self.run_planes(ev(i + 1))
                self.fetch_descriptors((i + 1) % 2)
            desc = self.compact_descriptors(i % 2)
            self.schedule(desc)
            n_canv = self.gather(join=False)
        self.join()
        return n_canv

    def step(self):
        self.run_planes()
        desc = self.descriptors()
        n_events = self.schedule(desc)
        n_canvases = self.gather()
        return desc, n_events, n_canvases

    def camera_results(self, k: int) -> dict:
        """Per-frame results (RoIs, patches, ...) of the shard's k-th camera
        from the last step (blocking download)."""
        n = self.n
        res = self.pipe.results(len(self.cameras) * n, self.stream)
        return {key: (val[k * n:(k + 1) * n] if isinstance(val, np.ndarray) else val)
                for key, val in res.items() if key in ("n_rois", "rois", "n_patches", "admitted")}

    def events(self):
        """InvokeEvents of the last step (readable until the next batcher call)."""
        return self.sched._events(self._nev)

    def canvases(self, count: int) -> np.ndarray:
        return self.ctx.download(self.d_canvases, (count, self.canvas[1], self.canvas[0] * 3),
                                 np.uint8, self.stream)


class GlobalCameraPath(MultiCameraPath):
    """Global cross-camera mode: ONE batcher over every camera
    of the job -- the reference's single SloScheduler over all scenes
    (sim.hpp:392) -- replicated on every rank from the all-gathered
    descriptors, so all ranks take the same decisions without a broadcast.
    Rank r writes the canvases of invoke events r, r+G, r+2G, ...; patches
    of other ranks' cameras are read straight from their frame rings through
    CUDA IPC (peer reads over NVLink; on one GPU, the same memory).  Each
    rank still runs K1-K4 only on its own cameras.

    `comm` (api.Comm) exchanges the rings' IPC handles once, here, and the
    descriptor blocks every pass."""

    def __init__(self, ctx: Context, n_cameras: int, comm, width, height, n_frames, profile, **kw):
        rank, world = comm.rank, comm.world
        per_rank = max(len(shard_cameras(n_cameras, world, r)) for r in range(world))
        super().__init__(ctx, shard_cameras(n_cameras, world, rank), width, height, n_frames,
                         profile, comm=comm, cameras_per_rank=per_rank, **kw)
        self.all_cameras = list(range(n_cameras))
        self.rank = rank
        # (camera id, IPC handle of its ring) per owned camera, padded to the
        # largest shard so every rank sends the same number of bytes
        rec = np.zeros(per_rank, [("camera", "<i4"), ("handle", "u1", 64)])
        rec["camera"] = -1
        for k, (c, r) in enumerate(zip(self.cameras, self.rings)):
            rec[k] = (c, np.frombuffer(ctx.ipc_export(r.base), np.uint8))
        base, self._imported = {}, []
        for r, raw in enumerate(comm.allgather_bytes(rec.tobytes())):
            for c, h in np.frombuffer(raw, rec.dtype):
                c = int(c)
                if c < 0:
                    continue
                if r == rank:
                    base[c] = self.rings[self.cameras.index(c)].base
                else:
                    base[c] = ctx.ipc_import(h.tobytes())
                    self._imported.append(base[c])
        fb = self.rings[0].frame_bytes if self.rings else 3 * width * height
        ptrs = np.array([base[c] + s * fb for c in self.all_cameras for s in range(n_frames + 1)],
                        np.uint64)
        self.d_frames_global = ctx.malloc(8 * max(1, len(ptrs)))
        ctx.upload(self.d_frames_global, ptrs)
        self.frame_base = base

    def close(self):
        for p in self._imported:
            self.ctx.ipc_close(p)
        self._imported = []
        self.ctx.free(self.d_frames_global)
        super().close()

    def schedule(self, desc: np.ndarray):
        """`desc`: the all-gathered list of every camera."""
        self._nev, self.arrival, self._last = schedule_descriptors(
            self.sched, desc, self.all_cameras, self.n, self.bandwidth, self.per_camera_link)
        return self._nev

    def gather(self, join: bool = True) -> int:
        if self.d_canvases is None:
            cap = self.canvas_cap or max(1, len(self._last["patches"]))
            self.canvas_cap = cap
            self.d_canvases = self.ctx.malloc(cap * self.canvas_bytes)
        n = C.c_int64()
        check(N.lib().tg_batcher_gather_events(self.ctx.handle, self.sched.handle, self.rank,
                                               self.world, self.d_frames_global, 3 * self.W,
                                               self.d_canvases, self.canvas_cap, C.byref(n),
                                               self.gstream))
        if join:
            self.join()
        return n.value


def schedule_descriptors(sched, desc: np.ndarray, cameras, n_frames: int, bandwidth_mbps: float,
                         per_camera_link: bool = True):
    """Host half of configs 3/4 on DESC_DTYPE records (camera-major in the
    order of `cameras`, frame and zone order), tg_batcher_schedule: ids
    renumbered over all patches (sim.hpp:249-251), admitted ones
    (sim.hpp:262) sent over the uplinks and replayed through `sched` (an
    api.SloScheduler).  Returns (number of events, arrival times of the
    admitted patches, dict(patches=their renumbered metas, src=their frame
    table indices, infeasible=infeasible-at-arrival flags, sim.hpp:296-300))."""
    desc = np.ascontiguousarray(desc, DESC_DTYPE)
    cams = np.ascontiguousarray(list(cameras), np.int32)
    n = len(desc)
    patches = np.zeros(max(1, n), PATCH_DTYPE)
    src = np.zeros(max(1, n), np.int32)
    arrival = np.zeros(max(1, n), np.int64)
    n_adm, n_ev = C.c_int64(), C.c_int32()
    check(N.lib().tg_batcher_schedule(sched.handle, desc.ctypes.data, n, cams.ctypes.data,
                                      len(cams), n_frames, float(bandwidth_mbps),
                                      int(per_camera_link), patches.ctypes.data, src.ctypes.data,
                                      arrival.ctypes.data, C.byref(n_adm), C.byref(n_ev)))
    k = n_adm.value
    # sim.hpp:296-300: a patch whose deadline minus the single-canvas slack
    # is already behind its arrival (a metrics flag; scheduling is unchanged)
    infeasible = patches[:k]["deadline_us"] - sched.profile.slack_us(1) < arrival[:k]
    return n_ev.value, arrival[:k], dict(patches=patches[:k], src=src[:k], infeasible=infeasible)
