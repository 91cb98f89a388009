"""Python mirror of the reference's hot-path API, executed on the B200.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/tangram/{geometry,partition,stitch}.hpp:

* ``partition(frame, cfg, rois, bytes_per_pixel, first_patch_id=0)``
  (partition.hpp:119-143) and ``stitch_all(queue, spec)`` (stitch.hpp:108-146)
  run as CUDA kernels through the C ABI;
* ``std::invalid_argument`` surfaces as :class:`InvalidArgument` (a
  ``ValueError``) and ``std::out_of_range`` as :class:`OutOfRange` (an
  ``IndexError``), with the reference's message texts;
* value helpers (``area``, ``overlap_area``, ``canvas_efficiency``,
  ``extract_canvas``, ``concat_stitches``, ``dump_layout``) are plain data
  manipulation, as in the reference headers.

The frame->canvas hot path itself is :class:`Pipeline` (device-resident
frames in, device-resident canvases out).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native as N


# ---------------------------------------------------------------- errors
class TangramError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """Reference: std::invalid_argument."""


class OutOfRange(IndexError):
    """Reference: std::out_of_range."""


class CapacityError(TangramError):
    pass


class CudaError(TangramError):
    pass


class NoDevice(TangramError):
    pass


class CommError(TangramError):
    pass


_ERRS = {N.TG_ERR_INVALID_ARGUMENT: InvalidArgument, N.TG_ERR_OUT_OF_RANGE: OutOfRange,
         N.TG_ERR_CAPACITY: CapacityError, N.TG_ERR_CUDA: CudaError, N.TG_ERR_NO_DEVICE: NoDevice,
         N.TG_ERR_COMM: CommError}


def check(status: int) -> None:
    if status != N.TG_OK:
        msg = N.lib().tg_last_error().decode()
        raise _ERRS.get(status, TangramError)(msg)


# ------------------------------------------------------------ value types
@dataclass(frozen=True)
class Rect:
    """geometry.hpp:28-38 -- bottom-left origin; memory row r is y = r."""
    x: int = 0
    y: int = 0
    w: int = 0
    h: int = 0

    def right(self) -> int:
        return self.x + self.w

    def top(self) -> int:
        return self.y + self.h


def area(r: Rect) -> int:
    return r.w * r.h


def overlap_area(a: Rect, b: Rect) -> int:
    ow = min(a.right(), b.right()) - max(a.x, b.x)
    oh = min(a.top(), b.top()) - max(a.y, b.y)
    return ow * oh if ow > 0 and oh > 0 else 0


def contains(outer: Rect, inner: Rect) -> bool:
    return (inner.x >= outer.x and inner.y >= outer.y and inner.right() <= outer.right()
            and inner.top() <= outer.top())


def enclosing_rect(rects: Sequence[Rect]) -> Rect:
    if not rects:
        raise InvalidArgument("empty rect set")
    x0 = min(r.x for r in rects)
    y0 = min(r.y for r in rects)
    x1 = max(r.right() for r in rects)
    y1 = max(r.top() for r in rects)
    return Rect(x0, y0, x1 - x0, y1 - y0)


@dataclass
class FrameSpec:
    frame_id: int = 0
    width: int = 0
    height: int = 0
    generation_time_us: int = 0
    slo_us: int = 0


@dataclass
class PartitionConfig:
    zones_x: int = 4
    zones_y: int = 4


@dataclass
class PatchMeta:
    patch_id: int = 0
    source_frame_id: int = 0
    rect: Rect = field(default_factory=Rect)
    generation_time_us: int = 0
    slo_us: int = 0
    deadline_us: int = 0
    size_bytes: int = 0


@dataclass
class CanvasSpec:
    width: int = 1024
    height: int = 1024
    vram_per_canvas_gb: float = 1.0

    def surface_area(self) -> int:
        return self.width * self.height


@dataclass
class Placement:
    patch_id: int = 0
    canvas_index: int = 0
    position: Rect = field(default_factory=Rect)


@dataclass
class CanvasState:
    placements: list = field(default_factory=list)
    free_rects: list = field(default_factory=list)
    used_area: int = 0


@dataclass
class StitchResult:
    spec: CanvasSpec = field(default_factory=CanvasSpec)
    canvases: list = field(default_factory=list)
    placement_index: dict = field(default_factory=dict)

    def canvas_count(self) -> int:
        return len(self.canvases)

    def empty(self) -> bool:
        return not self.canvases


def _rect(r) -> Rect:
    return r if isinstance(r, Rect) else Rect(*r)


def _c_rect(r: Rect) -> N.tg_rect:
    return N.tg_rect(r.x, r.y, r.w, r.h)


def _py_rect(r: N.tg_rect) -> Rect:
    return Rect(r.x, r.y, r.w, r.h)


def _c_patch(p: PatchMeta) -> N.tg_patch_meta:
    return N.tg_patch_meta(p.patch_id, p.source_frame_id, _c_rect(p.rect), p.generation_time_us,
                           p.slo_us, p.deadline_us, p.size_bytes)


def _py_patch(p: N.tg_patch_meta) -> PatchMeta:
    return PatchMeta(p.patch_id, p.source_frame_id, _py_rect(p.rect), p.generation_time_us,
                     p.slo_us, p.deadline_us, p.size_bytes)


# ---------------------------------------------------------------- context
class Context:
    """One CUDA device + stream (tg_ctx)."""

    def __init__(self, device: int = 0):
        self._lib = N.lib()
        h = C.c_void_p()
        check(self._lib.tg_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            self._lib.tg_ctx_destroy(self.handle)
            self.handle = None

    @property
    def stream(self) -> int:
        return self._lib.tg_ctx_stream(self.handle)

    def synchronize(self) -> None:
        check(self._lib.tg_ctx_synchronize(self.handle))

    def sm_count(self) -> int:
        n = C.c_int32()
        check(self._lib.tg_device_sm_count(self.handle, C.byref(n)))
        return n.value

    # plumbing
    def malloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        check(self._lib.tg_malloc_device(self.handle, max(1, nbytes), C.byref(p)))
        return p.value

    def free(self, ptr: int) -> None:
        check(self._lib.tg_free_device(self.handle, ptr))

    def malloc_host(self, nbytes: int) -> int:
        p = C.c_void_p()
        check(self._lib.tg_malloc_host(self.handle, max(1, nbytes), C.byref(p)))
        return p.value

    def free_host(self, ptr: int) -> None:
        check(self._lib.tg_free_host(self.handle, ptr))

    def ipc_export(self, dptr: int) -> bytes:
        """64-byte handle of a device allocation for other processes."""
        h = N.tg_ipc_handle()
        check(self._lib.tg_ipc_export(self.handle, dptr, C.byref(h)))
        return bytes(h.bytes)

    def ipc_import(self, handle: bytes) -> int:
        h = N.tg_ipc_handle()
        C.memmove(h.bytes, handle, 64)
        p = C.c_void_p()
        check(self._lib.tg_ipc_import(self.handle, C.byref(h), C.byref(p)))
        return p.value

    def ipc_close(self, dptr: int) -> None:
        check(self._lib.tg_ipc_close(self.handle, dptr))

    def memcpy(self, dst: int, src: int, nbytes: int, kind: int, stream=None) -> None:
        check(self._lib.tg_memcpy_async(self.handle, dst, src, nbytes, kind, stream))

    def upload(self, dptr: int, arr: np.ndarray, stream=None) -> None:
        arr = np.ascontiguousarray(arr)
        self.memcpy(dptr, arr.ctypes.data, arr.nbytes, 0, stream)
        self.stream_sync(stream)

    def download(self, dptr: int, shape, dtype, stream=None) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        self.memcpy(out.ctypes.data, dptr, out.nbytes, 1, stream)
        self.stream_sync(stream)
        return out

    def memset(self, dptr: int, value: int, nbytes: int, stream=None) -> None:
        check(self._lib.tg_memset_async(self.handle, dptr, value, nbytes, stream))

    def stream_sync(self, stream=None) -> None:
        check(self._lib.tg_stream_synchronize(self.handle, stream))

    def new_stream(self, high_priority: bool = False) -> int:
        s = C.c_void_p()
        if high_priority:
            check(self._lib.tg_stream_create_priority(self.handle, 1, C.byref(s)))
        else:
            check(self._lib.tg_stream_create(self.handle, C.byref(s)))
        return s.value

    def event(self) -> int:
        e = C.c_void_p()
        check(self._lib.tg_event_create(self.handle, C.byref(e)))
        return e.value

    def record(self, ev: int, stream=None) -> None:
        check(self._lib.tg_event_record(self.handle, ev, stream))

    def event_sync(self, ev: int) -> None:
        check(self._lib.tg_event_synchronize(self.handle, ev))

    def elapsed_ms(self, start: int, stop: int) -> float:
        ms = C.c_float()
        check(self._lib.tg_event_elapsed_ms(self.handle, start, stop, C.byref(ms)))
        return ms.value


class Comm:
    """The descriptor all-gather's communicator (tg_comm): NCCL over device
    buffers (stream-ordered), or a host transport -- any callable
    ``allgather(data: bytes) -> list[bytes]`` (rank-major) -- over host
    buffers.  Ranks of a device communicator meet through a 128-byte id that
    rank 0 creates (:meth:`unique_id`) and sends out of band."""

    def __init__(self, handle, ctx: Context | None, rank: int, world: int, on_device: bool,
                 keep=None):
        self.handle, self.ctx, self.rank, self.world = handle, ctx, rank, world
        self.on_device, self._keep = on_device, keep

    @staticmethod
    def unique_id() -> bytes:
        Comm._prefer_bundled_nccl()
        uid = N.tg_comm_id()
        check(N.lib().tg_comm_get_unique_id(C.byref(uid)))
        return bytes(uid.bytes)

    @staticmethod
    def _prefer_bundled_nccl() -> None:
        """NCCL is opened at run time; prefer the copy a Python environment
        ships (nvidia-nccl wheel), so a framework imported later binds to
        the same libnccl.so.2."""
        import importlib.util
        import os
        if os.environ.get("TG_NCCL_LIB"):
            return
        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["TG_NCCL_LIB"] = cand
                return

    @classmethod
    def nccl(cls, ctx: Context, uid: bytes, rank: int, world: int) -> "Comm":
        cls._prefer_bundled_nccl()
        u = N.tg_comm_id()
        C.memmove(u.bytes, uid, 128)
        h = C.c_void_p()
        check(N.lib().tg_comm_create(ctx.handle, C.byref(u), rank, world, C.byref(h)))
        return cls(h, ctx, rank, world, True)

    @classmethod
    def host(cls, rank: int, world: int, allgather) -> "Comm":
        def fn(send, nbytes, recv, _user):
            try:
                parts = allgather(C.string_at(send, nbytes) if nbytes else b"")
                if len(parts) != world or any(len(x) != nbytes for x in parts):
                    return 1
                if nbytes:
                    C.memmove(recv, b"".join(parts), nbytes * world)
                return 0
            except Exception:
                return 1
        cb = N.HOST_ALLGATHER_FN(fn)
        h = C.c_void_p()
        check(N.lib().tg_comm_create_host(rank, world, cb, None, C.byref(h)))
        return cls(h, None, rank, world, False, keep=cb)

    def allgather(self, send: int, nbytes: int, recv: int, stream=None) -> None:
        """Raw all-gather (device pointers for NCCL, host pointers otherwise)."""
        check(N.lib().tg_comm_allgather(self.handle, send, nbytes, recv, stream))

    def allgather_bytes(self, data: bytes) -> list[bytes]:
        """Blocking all-gather of equal-sized host byte strings (e.g. IPC
        handles), staged through device memory on an NCCL communicator."""
        n = len(data)
        out = C.create_string_buffer(max(1, n * self.world))
        src = C.create_string_buffer(data, max(1, n))
        if self.on_device:
            d_send, d_recv = self.ctx.malloc(n), self.ctx.malloc(n * self.world)
            self.ctx.memcpy(d_send, C.addressof(src), n, 0)
            self.allgather(d_send, n, d_recv, self.ctx.stream)
            self.ctx.memcpy(C.addressof(out), d_recv, n * self.world, 1)
            self.ctx.stream_sync()
            self.ctx.free(d_send)
            self.ctx.free(d_recv)
        else:
            self.allgather(C.addressof(src), n, C.addressof(out))
        raw = out.raw
        return [raw[r * n:(r + 1) * n] for r in range(self.world)]

    def close(self):
        if self.handle:
            N.lib().tg_comm_destroy(self.handle)
            self.handle = None


_DEFAULT: Context | None = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context(0)
    return _DEFAULT


# ------------------------------------------------------ rect-level drop-in
def make_zones(frame: FrameSpec, cfg: PartitionConfig) -> list[Rect]:
    """partition.hpp:69-88."""
    n = max(1, cfg.zones_x * cfg.zones_y)
    out = (N.tg_rect * n)()
    fs = N.tg_frame_spec(frame.frame_id, frame.width, frame.height, frame.generation_time_us,
                         frame.slo_us)
    check(N.lib().tg_make_zones(C.byref(fs), N.tg_partition_config(cfg.zones_x, cfg.zones_y),
                                out, n))
    return [_py_rect(r) for r in out]


def assign_rois(rois: Sequence[Rect], zones: Sequence[Rect], ctx: Context | None = None):
    """partition.hpp:93-112: per-zone lists of RoI indices."""
    ctx = ctx or default_context()
    rois = [_rect(r) for r in rois]
    n, nz = len(rois), len(zones)
    rarr = (N.tg_rect * max(1, n))(*[_c_rect(r) for r in rois])
    zarr = (N.tg_rect * max(1, nz))(*[_c_rect(_rect(z)) for z in zones])
    zone_of = (C.c_int32 * max(1, n))()
    check(N.lib().tg_assign_rois(ctx.handle, rarr, n, zarr, nz, zone_of))
    lists = [[] for _ in range(nz)]
    for i in range(n):
        lists[zone_of[i]].append(i)
    return lists


def partition(frame: FrameSpec, cfg: PartitionConfig, rois: Iterable, bytes_per_pixel: float,
              first_patch_id: int = 0, ctx: Context | None = None) -> list[PatchMeta]:
    """partition.hpp:119-143, on the device."""
    ctx = ctx or default_context()
    rois = [_rect(r) for r in rois]
    n = len(rois)
    rarr = (N.tg_rect * max(1, n))(*[_c_rect(r) for r in rois])
    cap = max(1, cfg.zones_x * cfg.zones_y)
    out = (N.tg_patch_meta * cap)()
    got = C.c_int32()
    fs = N.tg_frame_spec(frame.frame_id, frame.width, frame.height, frame.generation_time_us,
                         frame.slo_us)
    check(N.lib().tg_partition(ctx.handle, C.byref(fs),
                               N.tg_partition_config(cfg.zones_x, cfg.zones_y), rarr, n,
                               float(bytes_per_pixel), first_patch_id, out, cap, C.byref(got)))
    return [_py_patch(out[i]) for i in range(got.value)]


def stitch_all(queue: Sequence[PatchMeta], spec: CanvasSpec,
               ctx: Context | None = None) -> StitchResult:
    """stitch.hpp:108-146, on the device, placements bit-identical."""
    ctx = ctx or default_context()
    n = len(queue)
    q = (N.tg_patch_meta * max(1, n))(*[_c_patch(p) for p in queue])
    pl = (N.tg_placement * max(1, n))()
    cap = 2 * n + 1
    fr = (N.tg_free_rect * cap)()
    nc, nf = C.c_int32(), C.c_int32()
    check(N.lib().tg_stitch_all(ctx.handle, q, n,
                                N.tg_canvas_spec(spec.width, spec.height, spec.vram_per_canvas_gb),
                                pl, C.byref(nc), fr, cap, C.byref(nf)))
    res = StitchResult(spec=spec, canvases=[CanvasState() for _ in range(nc.value)])
    for i in range(n):
        p = Placement(pl[i].patch_id, pl[i].canvas_index, _py_rect(pl[i].position))
        cs = res.canvases[p.canvas_index]
        cs.placements.append(p)
        cs.used_area += area(p.position)
        res.placement_index[p.patch_id] = p
    for i in range(nf.value):
        res.canvases[fr[i].canvas_index].free_rects.append(_py_rect(fr[i].rect))
    return res


def canvas_efficiency(result: StitchResult) -> list[float]:
    """stitch.hpp:149-157."""
    s = float(result.spec.surface_area())
    return [c.used_area / s for c in result.canvases]


def dump_layout(result: StitchResult) -> str:
    """stitch.hpp:160-176."""
    out = []
    eff = canvas_efficiency(result)
    for ci, c in enumerate(result.canvases):
        out.append(f"canvas {ci} ({result.spec.width}x{result.spec.height}) "
                   f"efficiency={eff[ci]:.4f}\n")
        for p in c.placements:
            out.append(f"  patch {p.patch_id} at ({p.position.x},{p.position.y}) "
                       f"{p.position.w}x{p.position.h}\n")
    return "".join(out)


def extract_canvas(result: StitchResult, canvas_index: int) -> StitchResult:
    """stitch.hpp:179-190."""
    if canvas_index < 0 or canvas_index >= result.canvas_count():
        raise OutOfRange("canvas index out of range")
    src = result.canvases[canvas_index]
    c = CanvasState([Placement(p.patch_id, 0, p.position) for p in src.placements],
                    list(src.free_rects), src.used_area)
    return StitchResult(result.spec, [c], {p.patch_id: p for p in c.placements})


def concat_stitches(parts: Sequence[StitchResult]) -> StitchResult:
    """stitch.hpp:193-208."""
    out = StitchResult()
    if parts:
        out.spec = parts[0].spec
    for part in parts:
        base = out.canvas_count()
        for c in part.canvases:
            cc = CanvasState([Placement(p.patch_id, p.canvas_index + base, p.position)
                              for p in c.placements], list(c.free_rects), c.used_area)
            for p in cc.placements:
                out.placement_index[p.patch_id] = p
            out.canvases.append(cc)
    return out


# --------------------------------------------------------- synthetic input
def derive_seed(master: int, component: str) -> int:
    return N.lib().tg_derive_seed(master, component.encode())


def generate_trace(n_frames=150, fps=15.0, frame_width=1920, frame_height=1080,
                   roi_proportion_mean=0.10, roi_proportion_jitter=0.5, burst_probability=0.05,
                   burst_multiplier=3.0, roi_count_min=2, roi_count_max=12, roi_aspect_min=0.5,
                   roi_aspect_max=2.0, roi_max_dim=480, seed=1):
    """trace.hpp:184-231.  Returns (t_us list, per-frame lists of Rect)."""
    cfg = N.tg_workload_config(n_frames, fps, frame_width, frame_height, roi_proportion_mean,
                               roi_proportion_jitter, burst_probability, burst_multiplier,
                               roi_count_min, roi_count_max, roi_aspect_min, roi_aspect_max,
                               roi_max_dim, seed)
    n = max(1, n_frames)
    cap = max(1, n_frames * max(1, roi_count_max))
    t = (C.c_int64 * n)()
    cnt = (C.c_int32 * n)()
    rois = (N.tg_rect * cap)()
    tot = C.c_int64()
    check(N.lib().tg_generate_trace(C.byref(cfg), t, cnt, rois, cap, C.byref(tot)))
    frames, k = [], 0
    for i in range(n_frames):
        frames.append([_py_rect(rois[k + j]) for j in range(cnt[i])])
        k += cnt[i]
    return [t[i] for i in range(n_frames)], frames


class FrameRing:
    """Device-resident frames of one camera: slot 0 is the background-only
    frame (t = -1), slot i+1 is frame i.  Frame i's predecessor is slot i."""

    def __init__(self, ctx: Context, width: int, height: int, n_frames: int, pitch=None):
        self.ctx, self.W, self.H, self.n = ctx, width, height, n_frames
        self.pitch = pitch or 3 * width
        self.frame_bytes = self.pitch * height
        self.base = ctx.malloc(self.frame_bytes * (n_frames + 1))
        self.slots = [self.base + i * self.frame_bytes for i in range(n_frames + 1)]
        self._tables = []

    def close(self):
        for t in self._tables:
            self.ctx.free(t)
        self._tables = []
        if self.base:
            self.ctx.free(self.base)
            self.base = None

    def synthesize(self, pixel_seed: int, rects_per_frame: Sequence[Sequence[Rect]]):
        """Writes the background frame and frames 0..n-1 on the device."""
        lib, ctx = N.lib(), self.ctx
        flat = [r for fr in rects_per_frame for r in fr]
        offs = np.zeros(self.n + 2, np.int32)
        offs[2:] = np.cumsum([len(fr) for fr in rects_per_frame])
        d_rects = ctx.malloc(16 * max(1, len(flat)))
        d_offs = ctx.malloc(4 * len(offs))
        d_ptrs = ctx.malloc(8 * (self.n + 1))
        if flat:
            ctx.upload(d_rects, np.array([(r.x, r.y, r.w, r.h) for r in flat], np.int32))
        ctx.upload(d_offs, offs)
        ctx.upload(d_ptrs, np.array(self.slots, np.uint64))
        # background (t=-1) uses offsets[0..1] = empty
        check(lib.tg_synth_frames(ctx.handle, self.W, self.H, self.pitch, pixel_seed, 1, -1,
                                  d_rects, d_offs, d_ptrs, None))
        check(lib.tg_synth_frames(ctx.handle, self.W, self.H, self.pitch, pixel_seed, self.n, 0,
                                  d_rects, d_offs + 4, d_ptrs + 8, None))
        ctx.stream_sync()
        for p in (d_rects, d_offs, d_ptrs):
            ctx.free(p)

    def upload_frame(self, slot: int, arr: np.ndarray):
        assert arr.nbytes == self.frame_bytes
        self.ctx.upload(self.slots[slot], arr)

    def download_frame(self, slot: int) -> np.ndarray:
        return self.ctx.download(self.slots[slot], (self.H, self.pitch), np.uint8)

    def tables(self, first: int = 0, count: int | None = None):
        """Device pointer tables (cur, prev) for frames first..first+count-1."""
        count = self.n - first if count is None else count
        cur = np.array(self.slots[first + 1:first + 1 + count], np.uint64)
        prev = np.array(self.slots[first:first + count], np.uint64)
        d_cur, d_prev = self.ctx.malloc(8 * count), self.ctx.malloc(8 * count)
        self.ctx.upload(d_cur, cur)
        self.ctx.upload(d_prev, prev)
        self._tables += [d_cur, d_prev]
        return d_cur, d_prev


class Pipeline:
    """frames -> masks -> cells -> RoIs -> patches -> placements -> canvases."""

    def __init__(self, ctx: Context, width: int, height: int, **overrides):
        self.ctx = ctx
        lib = N.lib()
        p = N.tg_pipeline_params()
        check(lib.tg_pipeline_params_default(width, height, C.byref(p)))
        for k, v in overrides.items():
            if k == "zones":
                p.partition = N.tg_partition_config(*v)
            elif k == "canvas":
                p.canvas = N.tg_canvas_spec(v[0], v[1], 1.0)
            else:
                setattr(p, k, v)
        self.params = p
        h = C.c_void_p()
        check(lib.tg_pipeline_create(ctx.handle, C.byref(p), C.byref(h)))
        self.handle = h
        v = N.tg_pipeline_views()
        check(lib.tg_pipeline_device_views(h, C.byref(v)))
        self.views = v
        self.zones = v.zones

    def close(self):
        if self.handle:
            N.lib().tg_pipeline_destroy(self.handle)
            self.handle = None

    @property
    def canvas_bytes(self) -> int:
        return self.params.canvas.width * self.params.canvas.height * 3

    def run(self, n_frames, d_cur, d_prev, d_frame_ids, d_gen_us, first_patch_id, d_canvases,
            stream=None):
        check(N.lib().tg_pipeline_run(self.handle, n_frames, d_cur, d_prev, d_frame_ids, d_gen_us,
                                      first_patch_id, d_canvases, stream))

    def graph(self, n_frames, d_cur, d_prev, d_frame_ids, d_gen_us, first_patch_id, d_canvases,
              stream=None) -> "Graph":
        g = C.c_void_p()
        check(N.lib().tg_pipeline_graph_create(self.handle, n_frames, d_cur, d_prev, d_frame_ids,
                                               d_gen_us, first_patch_id, d_canvases, stream,
                                               C.byref(g)))
        return Graph(g)

    def results(self, n_frames: int, stream=None) -> dict:
        """Blocking download of the last run's per-frame results."""
        F, Z, R = n_frames, self.zones, self.params.max_rois_per_frame
        out = dict(
            n_rois=np.zeros(F, np.int32), rois=np.zeros((F, R, 4), np.int32),
            n_patches=np.zeros(F, np.int32), patches=(N.tg_patch_meta * max(1, F * Z))(),
            admitted=np.zeros((F, Z), np.uint8), n_placements=np.zeros(F, np.int32),
            placements=(N.tg_placement * max(1, F * Z))(), n_canvases=np.zeros(F, np.int32))
        total = C.c_int64()
        check(N.lib().tg_pipeline_download(
            self.handle, F, stream, out["n_rois"].ctypes.data, out["rois"].ctypes.data,
            out["n_patches"].ctypes.data, C.cast(out["patches"], C.c_void_p),
            out["admitted"].ctypes.data, out["n_placements"].ctypes.data,
            C.cast(out["placements"], C.c_void_p), out["n_canvases"].ctypes.data, C.byref(total)))
        out["total_canvases"] = total.value
        out["patch_list"] = [[_py_patch(out["patches"][f * Z + j]) for j in range(out["n_patches"][f])]
                             for f in range(F)]
        out["placement_list"] = [
            [(pl.patch_id, pl.canvas_index, pl.position.x, pl.position.y, pl.position.w,
              pl.position.h) for pl in (out["placements"][f * Z + k]
                                        for k in range(out["n_placements"][f]))]
            for f in range(F)]
        return out

    def set_descriptor_output(self, d_block: int | None, cap: int = 0, d_cameras: int | None = None,
                              frames_per_camera: int = 1) -> None:
        """Plan stages write the run's patches as dense device descriptors
        (tg_pipeline_set_descriptor_output); None detaches."""
        check(N.lib().tg_pipeline_set_descriptor_output(self.handle, d_block, cap, d_cameras,
                                                        frames_per_camera))

    def stats(self) -> dict:
        s = N.tg_pipeline_stats()
        check(N.lib().tg_pipeline_get_stats(self.handle, C.byref(s)))
        return {"mask_fused_launches": s.mask_fused_launches,
                "mask_split_launches": s.mask_split_launches}

    def free_rects(self, frame: int):
        cap = 3 * self.zones + 4
        arr = (N.tg_free_rect * cap)()
        n = C.c_int32()
        check(N.lib().tg_pipeline_free_rects(self.handle, frame, arr, cap, C.byref(n)))
        return [(arr[i].canvas_index, arr[i].rect.x, arr[i].rect.y, arr[i].rect.w, arr[i].rect.h)
                for i in range(n.value)]

    def cells(self, n_frames: int) -> np.ndarray:
        v = self.views
        return self.ctx.download(v.cells, (n_frames, v.cells_y, v.cells_x), np.uint32)

    def mask(self, n_frames: int) -> np.ndarray:
        v = self.views
        if not v.mask:
            raise TangramError("pipeline was created without keep_mask")
        return self.ctx.download(v.mask, (n_frames, self.params.height, v.mask_words), np.uint32)


class Graph:
    def __init__(self, handle):
        self.handle = handle

    def launch(self, stream=None):
        check(N.lib().tg_graph_launch(self.handle, stream))

    def close(self):
        if self.handle:
            N.lib().tg_graph_destroy(self.handle)
            self.handle = None


# ------------------------------------------------------------- SLO batcher
_TRIGGERS = {0: "deadline_timer", 1: "infeasible_arrival", 2: "memory_cap"}


@dataclass
class InvokeEvent:
    """scheduler.hpp:46-53."""
    fire_time_us: int = 0
    stitch: StitchResult = field(default_factory=StitchResult)
    patch_ids: list = field(default_factory=list)
    batch_size: int = 0
    estimated_slack_us: int = 0
    trigger: str = "deadline_timer"


@dataclass
class TimerHandle:
    fire_at_us: int = 0
    epoch: int = 0


class LatencyProfile:
    """latency.hpp:44-118 (slack = mu + 3 sigma, interpolated)."""

    def __init__(self, canvas_w: int, canvas_h: int, entries):
        self.canvas_w, self.canvas_h = canvas_w, canvas_h
        self.entries = [tuple(e) for e in entries]
        self._arr = (N.tg_profile_entry * max(1, len(self.entries)))(
            *[N.tg_profile_entry(int(k), float(mu), float(sd)) for k, mu, sd in self.entries])
        self.slack_us(1)  # validates like LatencyProfile::from_entries

    @classmethod
    def from_entries(cls, canvas_w, canvas_h, entries):
        return cls(canvas_w, canvas_h, entries)

    def slack_us(self, k: int) -> int:
        out = C.c_int64()
        check(N.lib().tg_profile_slack_us(self._arr, len(self.entries), k, C.byref(out)))
        return out.value


def max_canvases_per_batch(gpu_memory_gb: float, model_size_gb: float,
                           vram_per_canvas_gb: float) -> int:
    """cost.hpp:107-115."""
    k = C.c_int32()
    check(N.lib().tg_max_canvases_per_batch(gpu_memory_gb, model_size_gb, vram_per_canvas_gb,
                                            C.byref(k)))
    return k.value


def transmission_schedule(patches: Sequence[PatchMeta], bandwidth_mbps: float) -> list[int]:
    """trace.hpp:255-267 (per-link FIFO)."""
    n = len(patches)
    arr = (N.tg_patch_meta * max(1, n))(*[_c_patch(p) for p in patches])
    out = (C.c_int64 * max(1, n))()
    check(N.lib().tg_transmission_schedule(arr, n, float(bandwidth_mbps), out))
    return [out[i] for i in range(n)]


class SloScheduler:
    """The Alg. 2 invoker (scheduler.hpp:79-215) with an incremental repack;
    decisions, epochs and stitch results equal the reference's."""

    def __init__(self, spec: CanvasSpec, profile: LatencyProfile, max_canvases: int):
        if profile is None:
            raise InvalidArgument("scheduler needs a latency profile")
        self.spec = spec
        self.profile = profile
        h = C.c_void_p()
        check(N.lib().tg_batcher_create(
            N.tg_canvas_spec(spec.width, spec.height, spec.vram_per_canvas_gb), profile._arr,
            len(profile.entries), max_canvases, C.byref(h)))
        self.handle = h

    def enable_log(self, policy: str = "tangram") -> None:
        """Record the reference scheduler's event-log lines (scheduler.hpp:
        93-188) from now on."""
        check(N.lib().tg_batcher_set_log(self.handle, policy.encode()))

    def take_log(self) -> str:
        """The JSON lines recorded since the last call."""
        n = C.c_int64()
        check(N.lib().tg_batcher_take_log(self.handle, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(1, n.value))
        check(N.lib().tg_batcher_take_log(self.handle, buf, n.value, C.byref(n)))
        return buf.raw[:n.value].decode()

    def close(self):
        if self.handle:
            N.lib().tg_batcher_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _events(self, n: int) -> list[InvokeEvent]:
        out = []
        for i in range(n):
            info = N.tg_invoke_info()
            check(N.lib().tg_batcher_event(self.handle, i, C.byref(info), None, None, None))
            ids = (C.c_uint64 * max(1, info.n_patches))()
            pl = (N.tg_placement * max(1, info.n_patches))()
            fr = (N.tg_free_rect * max(1, info.n_free))()
            check(N.lib().tg_batcher_event(self.handle, i, None, ids, pl, fr))
            res = StitchResult(spec=self.spec, canvases=[CanvasState() for _ in range(info.batch_size)])
            for k in range(info.n_patches):
                p = Placement(pl[k].patch_id, pl[k].canvas_index, _py_rect(pl[k].position))
                cs = res.canvases[p.canvas_index]
                cs.placements.append(p)
                cs.used_area += area(p.position)
                res.placement_index[p.patch_id] = p
            for k in range(info.n_free):
                res.canvases[fr[k].canvas_index].free_rects.append(_py_rect(fr[k].rect))
            out.append(InvokeEvent(info.fire_time_us, res, [ids[k] for k in range(info.n_patches)],
                                   info.batch_size, info.estimated_slack_us,
                                   _TRIGGERS[info.trigger]))
        return out

    def on_patch_arrival(self, patch: PatchMeta, now: int, src_frame: int = -1):
        n = C.c_int32()
        check(N.lib().tg_batcher_on_patch_arrival(self.handle, C.byref(_c_patch(patch)), src_frame,
                                                  now, C.byref(n)))
        return self._events(n.value)

    def on_timer(self, now: int, epoch: int):
        n = C.c_int32()
        check(N.lib().tg_batcher_on_timer(self.handle, now, epoch, C.byref(n)))
        ev = self._events(n.value)
        return ev[0] if ev else None

    def pending_timer(self):
        has, at, ep = C.c_int32(), C.c_int64(), C.c_uint64()
        check(N.lib().tg_batcher_pending_timer(self.handle, C.byref(has), C.byref(at), C.byref(ep)))
        return TimerHandle(at.value, ep.value) if has.value else None

    def _status(self):
        q, c, d, r = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
        check(N.lib().tg_batcher_status(self.handle, C.byref(q), C.byref(c), C.byref(d), C.byref(r)))
        return q.value, c.value, d.value, r.value

    def idle(self) -> bool:
        return self._status()[0] == 0

    def _current(self):
        lib, info = N.lib(), N.tg_invoke_info()
        check(lib.tg_batcher_current(self.handle, C.byref(info), None, None, None))
        q = (N.tg_patch_meta * max(1, info.n_patches))()
        pl = (N.tg_placement * max(1, info.n_patches))()
        fr = (N.tg_free_rect * max(1, info.n_free))()
        check(lib.tg_batcher_current(self.handle, C.byref(info), q, pl, fr))
        return info, q, pl, fr

    def queue(self) -> list[PatchMeta]:
        """The queued patches in arrival order (scheduler.hpp:137)."""
        info, q, _, _ = self._current()
        return [_py_patch(q[i]) for i in range(info.n_patches)]

    def current_stitch(self) -> StitchResult:
        """The live batch's packing (scheduler.hpp:138)."""
        info, _, pl, fr = self._current()
        res = StitchResult(spec=self.spec, canvases=[CanvasState() for _ in range(info.batch_size)])
        for k in range(info.n_patches):
            p = Placement(pl[k].patch_id, pl[k].canvas_index, _py_rect(pl[k].position))
            cs = res.canvases[p.canvas_index]
            cs.placements.append(p)
            cs.used_area += area(p.position)
            res.placement_index[p.patch_id] = p
        for k in range(info.n_free):
            res.canvases[fr[k].canvas_index].free_rects.append(_py_rect(fr[k].rect))
        return res

    def queue_size(self) -> int:
        return self._status()[0]

    def current_canvas_count(self) -> int:
        return self._status()[1]

    def earliest_deadline_us(self) -> int:
        return self._status()[2]

    def remaining_time_us(self) -> int:
        return self._status()[3]

    def replay(self, patches: Sequence[PatchMeta], arrival_us: Sequence[int],
               src_frames: Sequence[int] | None = None) -> list[InvokeEvent]:
        """The reference event loop for the tangram policy (sim.hpp:334-458)."""
        n = len(patches)
        arr = (N.tg_patch_meta * max(1, n))(*[_c_patch(p) for p in patches])
        arv = (C.c_int64 * max(1, n))(*arrival_us)
        src = (C.c_int32 * max(1, n))(*(src_frames if src_frames is not None else [-1] * n))
        cnt = C.c_int32()
        check(N.lib().tg_batcher_replay(self.handle, arr, src, arv, n, C.byref(cnt)))
        return self._events(cnt.value)

    def replay_links(self, camera_patches: Sequence[Sequence[PatchMeta]], bandwidth_mbps: float,
                     per_camera_link: bool = True) -> tuple[list[InvokeEvent], list[int]]:
        """Multi-camera front end (sim.hpp:274-290) + the event loop: each
        camera's admitted patches, in generation order, delivered over one
        FIFO uplink per camera (or one shared link).  Returns the events and
        each patch's arrival time (camera-major order)."""
        flat = [p for cam in camera_patches for p in cam]
        n = len(flat)
        offs = [0]
        for cam in camera_patches:
            offs.append(offs[-1] + len(cam))
        c_offs = (C.c_int32 * len(offs))(*offs)
        arr = (N.tg_patch_meta * max(1, n))(*[_c_patch(p) for p in flat])
        src = (C.c_int32 * max(1, n))(*([-1] * n))
        arv = (C.c_int64 * max(1, n))()
        cnt = C.c_int32()
        check(N.lib().tg_batcher_replay_links(self.handle, len(camera_patches), c_offs, arr, src,
                                              float(bandwidth_mbps), int(bool(per_camera_link)),
                                              arv, C.byref(cnt)))
        return self._events(cnt.value), list(arv[:n])

    def gather(self, ctx: Context, event_index: int, d_frames: int, pitch: int, d_canvases: int,
               stream=None) -> None:
        """Writes event `event_index` (of the last call) into d_canvases."""
        check(N.lib().tg_batcher_gather(ctx.handle, self.handle, event_index, d_frames, pitch,
                                        d_canvases, stream))
