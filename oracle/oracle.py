"""ctypes front-end for the oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  It wraps

* ``oracle/_build/liboracle.so``    -- the C restatement (tangram_oracle.c), and
* ``oracle/_ref/libtangram_ref.so`` -- the reference's own headers compiled
  as-is (ref_shim.cpp), present wherever the reference could be built.

Both expose the same POD interface, so every helper below takes ``lib=``
("port" or "ref").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtangram_ref.so")
CELL = 16


class Rect(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("w", C.c_int32), ("h", C.c_int32)]


class Patch(C.Structure):
    _fields_ = [("patch_id", C.c_uint64), ("source_frame_id", C.c_uint64), ("rect", Rect),
                ("generation_time_us", C.c_int64), ("slo_us", C.c_int64),
                ("deadline_us", C.c_int64), ("size_bytes", C.c_int64)]


class Placement(C.Structure):
    _fields_ = [("patch_id", C.c_uint64), ("canvas_index", C.c_int32), ("position", Rect),
                ("pad_", C.c_int32)]


class FreeRect(C.Structure):
    _fields_ = [("r", Rect), ("canvas", C.c_int32)]


class FillJob(C.Structure):
    _fields_ = [("frame", C.c_int32), ("sx", C.c_int32), ("sy", C.c_int32), ("dx", C.c_int32),
                ("dy", C.c_int32), ("w", C.c_int32), ("h", C.c_int32)]


class GenCfg(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("fps", C.c_double), ("frame_width", C.c_int32),
                ("frame_height", C.c_int32), ("roi_proportion_mean", C.c_double),
                ("roi_proportion_jitter", C.c_double), ("burst_probability", C.c_double),
                ("burst_multiplier", C.c_double), ("roi_count_min", C.c_int32),
                ("roi_count_max", C.c_int32), ("roi_aspect_min", C.c_double),
                ("roi_aspect_max", C.c_double), ("roi_max_dim", C.c_int32), ("seed", C.c_uint64)]


class PathParams(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("pitch", C.c_int32),
                ("threshold", C.c_int32), ("radius", C.c_int32), ("zones_x", C.c_int32),
                ("zones_y", C.c_int32), ("canvas_w", C.c_int32), ("canvas_h", C.c_int32),
                ("bytes_per_pixel", C.c_double), ("slo_us", C.c_int64), ("max_rois", C.c_int32),
                ("threads", C.c_int32)]


class PathOut(C.Structure):
    _fields_ = [("n_rois", C.c_void_p), ("rois", C.c_void_p), ("n_patches", C.c_void_p),
                ("patches", C.c_void_p), ("admitted", C.c_void_p), ("n_canvases", C.c_void_p),
                ("placements", C.c_void_p), ("n_placements", C.c_void_p),
                ("canvases", C.c_void_p), ("canvas_cap", C.c_int64), ("cells", C.c_void_p),
                ("total_canvases", C.c_int64)]


class OracleError(Exception):
    """Raised with the oracle's (reference-identical) error message."""


def build() -> None:
    """Builds liboracle.so, and libtangram_ref.so when /root/reference exists."""
    subprocess.check_call(["make", "-s", "-C", HERE, "_build/liboracle.so"])
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


_LIBS: dict[str, C.CDLL] = {}


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def load(lib: str = "port") -> C.CDLL:
    if lib in _LIBS:
        return _LIBS[lib]
    path = PORT_SO if lib == "port" else REF_SO
    if not os.path.exists(path):
        build()
    dll = C.CDLL(path)
    pre = "orc_" if lib == "port" else "ref_"
    P = C.POINTER
    sig = {
        "derive_seed": (C.c_uint64, [C.c_uint64, C.c_char_p]),
        "generate_trace": (C.c_int64, [P(GenCfg), P(C.c_int64), P(C.c_int32), P(Rect), C.c_int64]),
        "make_zones": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, P(Rect)]),
        "partition": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                P(Rect), C.c_int, C.c_double, C.c_uint64, P(Patch)]),
        "stitch_all": (C.c_int, [P(Patch), C.c_int, C.c_int, C.c_int, P(Placement), P(C.c_int),
                                 P(FreeRect), C.c_int, P(C.c_int)]),
        "process_frames": (C.c_int, [P(PathParams), C.c_int, P(C.c_void_p), P(C.c_void_p),
                                     P(C.c_uint64), P(C.c_int64), C.c_uint64, P(PathOut)]),
        "last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(dll, pre + name)
        fn.restype, fn.argtypes = res, args
    if lib == "port":
        dll.orc_synth_frame.restype = None
        dll.orc_synth_frame.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int32, P(Rect),
                                        C.c_int, C.c_void_p]
        dll.orc_synth_rect.restype = None
        dll.orc_synth_rect.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int32, P(Rect), C.c_int,
                                       Rect, C.c_void_p, C.c_int]
        dll.orc_mask.restype = None
        dll.orc_mask.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.c_int, C.c_void_p]
        dll.orc_cells.restype = None
        dll.orc_cells.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        dll.orc_extract_rois.restype = C.c_int
        dll.orc_extract_rois.argtypes = [C.c_void_p, C.c_int, C.c_int, P(Rect), C.c_int]
        dll.orc_hash32.restype = C.c_uint32
        dll.orc_hash32.argtypes = [C.c_uint32]
        dll.orc_fill_jobs.restype = None
        dll.orc_fill_jobs.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                      C.c_int, C.c_void_p, C.c_int]
        dll.orc_rng_seed.restype = None
        dll.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        for n, r in (("orc_rng_next", C.c_uint64), ("orc_rng_uniform01", C.c_double)):
            getattr(dll, n).restype = r
            getattr(dll, n).argtypes = [C.c_void_p]
        dll.orc_rng_uniform_int.restype = C.c_int64
        dll.orc_rng_uniform_int.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        dll.orc_rng_normal.restype = C.c_double
        dll.orc_rng_normal.argtypes = [C.c_void_p, C.c_double, C.c_double]
        dll.orc_gen_cfg_default.restype = None
        dll.orc_gen_cfg_default.argtypes = [P(GenCfg)]
    else:
        dll.ref_rng_draws.restype = None
        dll.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_int,
                                      P(C.c_double), P(C.c_uint64)]
    _LIBS[lib] = dll
    return dll


def _err(dll, lib):
    return (dll.orc_last_error() if lib == "port" else dll.ref_last_error()).decode()


def _fn(dll, lib, name):
    return getattr(dll, ("orc_" if lib == "port" else "ref_") + name)


# ---------------------------------------------------------------- rng / trace
def derive_seed(master: int, component: str, lib: str = "port") -> int:
    dll = load(lib)
    return _fn(dll, lib, "derive_seed")(master, component.encode())


class Rng:
    """The port's mt19937_64-backed Rng (rng.hpp:42-70)."""

    def __init__(self, seed: int):
        self._dll = load("port")
        self._state = C.create_string_buffer(312 * 8 + 16)
        self._dll.orc_rng_seed(self._state, seed)

    def next(self) -> int:
        return self._dll.orc_rng_next(self._state)

    def uniform01(self) -> float:
        return self._dll.orc_rng_uniform01(self._state)

    def uniform_int(self, lo: int, hi: int) -> int:
        return self._dll.orc_rng_uniform_int(self._state, lo, hi)

    def normal(self, mu: float, sigma: float) -> float:
        return self._dll.orc_rng_normal(self._state, mu, sigma)


def gen_cfg(**kw) -> GenCfg:
    cfg = GenCfg()
    load("port").orc_gen_cfg_default(C.byref(cfg))
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def generate_trace(cfg: GenCfg, lib: str = "port"):
    """Returns (t_us[n], list of per-frame lists of (x, y, w, h))."""
    dll = load(lib)
    n = cfg.n_frames
    cap = max(1, n * max(1, cfg.roi_count_max))
    t_us = (C.c_int64 * max(1, n))()
    counts = (C.c_int32 * max(1, n))()
    rois = (Rect * cap)()
    got = _fn(dll, lib, "generate_trace")(C.byref(cfg), t_us, counts, rois, cap)
    if got < 0:
        raise OracleError(_err(dll, lib))
    frames, k = [], 0
    for i in range(n):
        frames.append([(rois[k + j].x, rois[k + j].y, rois[k + j].w, rois[k + j].h)
                       for j in range(counts[i])])
        k += counts[i]
    return [t_us[i] for i in range(n)], frames


# ------------------------------------------------------------ partition/stitch
def make_zones(width, height, zx, zy, lib="port"):
    dll = load(lib)
    out = (Rect * (zx * zy if zx > 0 and zy > 0 else 1))()
    if _fn(dll, lib, "make_zones")(width, height, zx, zy, out):
        raise OracleError(_err(dll, lib))
    return [(r.x, r.y, r.w, r.h) for r in out]


def partition(frame_id, width, height, gen_us, slo_us, zx, zy, rois, bpp, first_patch_id=0,
              lib="port"):
    """Returns a list of dicts mirroring PatchMeta (partition.hpp:56-64)."""
    dll = load(lib)
    n = len(rois)
    arr = (Rect * max(1, n))(*[Rect(*r) for r in rois])
    out = (Patch * max(1, zx * zy))()
    got = _fn(dll, lib, "partition")(frame_id, width, height, gen_us, slo_us, zx, zy, arr, n, bpp,
                                     first_patch_id, out)
    if got < 0:
        raise OracleError(_err(dll, lib))
    return [patch_dict(out[i]) for i in range(got)]


def patch_dict(p: Patch) -> dict:
    return dict(patch_id=p.patch_id, source_frame_id=p.source_frame_id,
                rect=(p.rect.x, p.rect.y, p.rect.w, p.rect.h),
                generation_time_us=p.generation_time_us, slo_us=p.slo_us,
                deadline_us=p.deadline_us, size_bytes=p.size_bytes)


def stitch_all(queue, canvas_w, canvas_h, lib="port"):
    """queue: list of (patch_id, w, h).  Returns (placements, n_canvases,
    free_rects) with placements in queue order as (patch_id, canvas, x, y, w,
    h) and free_rects as (canvas, x, y, w, h) in reference list order."""
    dll = load(lib)
    n = len(queue)
    q = (Patch * max(1, n))()
    for i, (pid, w, h) in enumerate(queue):
        q[i].patch_id = pid
        q[i].rect = Rect(0, 0, w, h)
    pl = (Placement * max(1, n))()
    cap = 2 * n + 4
    fr = (FreeRect * cap)()
    nc, nf = C.c_int(0), C.c_int(0)
    rc = _fn(dll, lib, "stitch_all")(q, n, canvas_w, canvas_h, pl, C.byref(nc), fr, cap, C.byref(nf))
    if rc:
        raise OracleError(_err(dll, lib))
    placements = [(pl[i].patch_id, pl[i].canvas_index, pl[i].position.x, pl[i].position.y,
                   pl[i].position.w, pl[i].position.h) for i in range(n)]
    free = [(fr[i].canvas, fr[i].r.x, fr[i].r.y, fr[i].r.w, fr[i].r.h) for i in range(nf.value)]
    return placements, nc.value, free


# ------------------------------------------------------------------- pixels
def synth_frame(width, height, pixel_seed, t, rects, pitch=None):
    dll = load("port")
    pitch = pitch or width * 3
    out = np.zeros((height, pitch), dtype=np.uint8)
    arr = (Rect * max(1, len(rects)))(*[Rect(*r) for r in rects])
    dll.orc_synth_frame(width, height, pitch, pixel_seed, t, arr, len(rects), out.ctypes.data)
    return out


def synth_rect(width, height, pixel_seed, t, rects, region, out=None):
    """Pixels (h, 3w) of `region` = (x, y, w, h) of synthetic frame t: the
    bytes synth_frame would write there."""
    dll = load("port")
    x, y, w, h = region
    if out is None:
        out = np.empty((h, 3 * w), np.uint8)
    arr = (Rect * max(1, len(rects)))(*[Rect(*r) for r in rects])
    dll.orc_synth_rect(width, height, pixel_seed, t, arr, len(rects), Rect(x, y, w, h),
                       out.ctypes.data, out.strides[0])
    return out


def synth_frames(width, height, pixel_seed, rects_per_frame, threads=None):
    """Background frame (t = -1) then frames 0..n-1, synthesized in parallel."""
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or os.cpu_count() or 1
    n = len(rects_per_frame)
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(lambda i: synth_frame(width, height, pixel_seed, i,
                                                 rects_per_frame[i] if i >= 0 else []),
                           range(-1, n)))


def mask(cur, prev, width, height, threshold=25, radius=2):
    dll = load("port")
    nw = (width + 31) // 32
    out = np.zeros((height, nw), dtype=np.uint32)
    cur = np.ascontiguousarray(cur)
    prev = np.ascontiguousarray(prev)
    dll.orc_mask(cur.ctypes.data, prev.ctypes.data, width, height, cur.shape[1], threshold, radius,
                 out.ctypes.data)
    return out


def cells(mask_words, width, height):
    dll = load("port")
    cx, cy = (width + CELL - 1) // CELL, (height + CELL - 1) // CELL
    out = np.zeros((cy, cx), dtype=np.uint32)
    m = np.ascontiguousarray(mask_words)
    dll.orc_cells(m.ctypes.data, width, height, out.ctypes.data)
    return out


def extract_rois(cell_grid, cap=4096):
    dll = load("port")
    g = np.ascontiguousarray(cell_grid, dtype=np.uint32)
    out = (Rect * cap)()
    n = dll.orc_extract_rois(g.ctypes.data, g.shape[1], g.shape[0], out, cap)
    if n < 0:
        raise OracleError("roi capacity exceeded")
    return [(out[i].x, out[i].y, out[i].w, out[i].h) for i in range(n)]


def process_frames(params: dict, cur_frames, prev_frames, frame_ids, gen_us, first_patch_id=0,
                   want_canvases=True, want_cells=False, canvas_cap=None, lib="port",
                   canvas_out=None):
    """Runs the whole per-frame CPU path.  cur_frames/prev_frames are lists
    of (H, pitch) uint8 arrays.  Returns a dict of per-frame results.
    canvas_out: a preallocated (cap, N, 3M) uint8 buffer for the canvases."""
    dll = load(lib)
    p = PathParams(**params)
    n = len(cur_frames)
    nz = p.zones_x * p.zones_y
    cx, cy = (p.width + CELL - 1) // CELL, (p.height + CELL - 1) // CELL
    res = dict(
        n_rois=np.zeros(n, np.int32), rois=np.zeros((n, p.max_rois, 4), np.int32),
        n_patches=np.zeros(n, np.int32), patches=(Patch * max(1, n * nz))(),
        admitted=np.zeros((n, nz), np.uint8), n_canvases=np.zeros(n, np.int32),
        placements=(Placement * max(1, n * nz))(), n_placements=np.zeros(n, np.int32))
    if canvas_cap is None:
        canvas_cap = n * nz if want_canvases else 0
    if want_canvases and canvas_out is not None:
        canv, canvas_cap = canvas_out, len(canvas_out)
    else:
        canv = np.zeros((canvas_cap, p.canvas_h, p.canvas_w * 3), np.uint8) if want_canvases else None
    cells_arr = np.zeros((n, cy, cx), np.uint32) if want_cells else None
    out = PathOut(res["n_rois"].ctypes.data, res["rois"].ctypes.data, res["n_patches"].ctypes.data,
                  C.cast(res["patches"], C.c_void_p), res["admitted"].ctypes.data,
                  res["n_canvases"].ctypes.data, C.cast(res["placements"], C.c_void_p),
                  res["n_placements"].ctypes.data,
                  canv.ctypes.data if canv is not None else None, canvas_cap,
                  cells_arr.ctypes.data if cells_arr is not None else None, 0)
    curp = (C.c_void_p * max(1, n))(*[f.ctypes.data for f in cur_frames])
    prevp = (C.c_void_p * max(1, n))(*[f.ctypes.data for f in prev_frames])
    fids = (C.c_uint64 * max(1, n))(*frame_ids)
    gens = (C.c_int64 * max(1, n))(*gen_us)
    rc = _fn(dll, lib, "process_frames")(C.byref(p), n, curp, prevp, fids, gens, first_patch_id,
                                         C.byref(out))
    if rc:
        raise OracleError(_err(dll, lib))
    res["total_canvases"] = out.total_canvases
    res["canvases"] = canv
    res["cells"] = cells_arr
    res["patch_list"] = [[patch_dict(res["patches"][f * nz + j]) for j in range(res["n_patches"][f])]
                         for f in range(n)]
    res["placement_list"] = [
        [(pl.patch_id, pl.canvas_index, pl.position.x, pl.position.y, pl.position.w, pl.position.h)
         for pl in (res["placements"][f * nz + k] for k in range(res["n_placements"][f]))]
        for f in range(n)]
    return res


# ------------------------------------------------------ reference scheduler
class SimCfg(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("zones_x", C.c_int32),
                ("zones_y", C.c_int32), ("canvas_w", C.c_int32), ("canvas_h", C.c_int32),
                ("per_scene_link", C.c_int32), ("vram_per_canvas_gb", C.c_double),
                ("gpu_memory_gb", C.c_double), ("model_size_gb", C.c_double),
                ("bandwidth_mbps", C.c_double), ("bytes_per_pixel", C.c_double),
                ("slo_us", C.c_int64)]


def _profile_arr(entries):
    flat = [float(v) for e in entries for v in e]
    return (C.c_double * max(1, len(flat)))(*flat), len(entries)


def run_tangram(scenes, width, height, profile, zones=(4, 4), canvas=(1024, 1024),
                vram_per_canvas_gb=1.0, gpu_memory_gb=6.0, model_size_gb=2.0, bandwidth_mbps=80.0,
                per_scene_link=True, bytes_per_pixel=1.5, slo_us=1_000_000):
    """The reference's tangram::run() (sim.hpp:206-552, tangram policy) on
    scenes = [(t_us list, per-frame rect lists)].  Returns per-patch
    (admitted, infeasible-at-arrival, arrival_us), the scheduler's invoke
    events and its raw event log (JSON lines)."""
    dll = load("ref")
    dll.ref_run_tangram.restype = C.c_int
    cfg = SimCfg(width, height, zones[0], zones[1], canvas[0], canvas[1], int(per_scene_link),
                 vram_per_canvas_gb, gpu_memory_gb, model_size_gb, bandwidth_mbps, bytes_per_pixel,
                 slo_us)
    fps = (C.c_int32 * len(scenes))(*[len(t) for t, _ in scenes])
    t_flat = [t for ts, _ in scenes for t in ts]
    cnt = [len(f) for _, fr in scenes for f in fr]
    rects = [r for _, fr in scenes for f in fr for r in f]
    t_arr = (C.c_int64 * max(1, len(t_flat)))(*t_flat)
    c_arr = (C.c_int32 * max(1, len(cnt)))(*cnt)
    r_arr = (Rect * max(1, len(rects)))(*[Rect(*r) for r in rects])
    prof, n_prof = _profile_arr(profile)
    pcap = max(1, len(t_flat) * zones[0] * zones[1])
    arrival = (C.c_int64 * pcap)()
    adm = (C.c_uint8 * pcap)()
    npatch = C.c_int32()
    ecap, icap = pcap, pcap
    ev_fire = (C.c_int64 * ecap)()
    ev_trig = (C.c_int32 * ecap)()
    ev_k = (C.c_int32 * ecap)()
    ev_slack = (C.c_int64 * ecap)()
    ev_np = (C.c_int32 * ecap)()
    ev_ids = (C.c_uint64 * icap)()
    nev = C.c_int32()
    eff_mean, eff_median = C.c_double(), C.c_double()
    rc = dll.ref_run_tangram(C.byref(cfg), len(scenes), fps, t_arr, c_arr, r_arr, prof, n_prof,
                             arrival, adm, C.byref(npatch), C.c_int64(pcap), C.byref(nev), ev_fire,
                             ev_trig, ev_k, ev_slack, ev_np, ev_ids, C.c_int64(ecap),
                             C.c_int64(icap), C.byref(eff_mean), C.byref(eff_median))
    if rc:
        raise OracleError(_err(dll, "ref"))
    events, k = [], 0
    for i in range(nev.value):
        ids = [ev_ids[k + j] for j in range(ev_np[i])]
        k += ev_np[i]
        events.append(dict(fire_time_us=ev_fire[i], trigger=ev_trig[i], batch_size=ev_k[i],
                           estimated_slack_us=ev_slack[i], patch_ids=ids))
    dll.ref_last_log.restype = C.c_int64
    nlog = dll.ref_last_log(None, C.c_int64(0))
    logbuf = C.create_string_buffer(max(1, nlog))
    dll.ref_last_log(logbuf, C.c_int64(nlog))
    return dict(log=logbuf.raw[:nlog].decode(),
                admitted=[adm[i] & 1 for i in range(npatch.value)],
                infeasible=[adm[i] >> 1 & 1 for i in range(npatch.value)],
                arrival_us=[arrival[i] for i in range(npatch.value)], events=events,
                mean_canvas_efficiency=eff_mean.value, median_canvas_efficiency=eff_median.value)


def save_trace_ref(scenes, width, height) -> str:
    """The reference's save_trace (trace.hpp:79-90) text for scenes =
    [(t_us list, per-frame rect lists)], scene ids cam0, cam1, ..."""
    dll = load("ref")
    dll.ref_save_trace.restype = C.c_int64
    fps = (C.c_int32 * len(scenes))(*[len(t) for t, _ in scenes])
    t_flat = [t for ts, _ in scenes for t in ts]
    cnt = [len(f) for _, fr in scenes for f in fr]
    rects = [r for _, fr in scenes for f in fr for r in f]
    t_arr = (C.c_int64 * max(1, len(t_flat)))(*t_flat)
    c_arr = (C.c_int32 * max(1, len(cnt)))(*cnt)
    r_arr = (Rect * max(1, len(rects)))(*[Rect(*r) for r in rects])
    cap = 64 * 1024 * 1024
    buf = C.create_string_buffer(cap)
    n = dll.ref_save_trace(len(scenes), fps, t_arr, c_arr, r_arr, width, height, buf, C.c_int64(cap))
    if n < 0:
        raise OracleError(_err(dll, "ref"))
    return buf.raw[:n].decode()


class RefScheduler:
    """The reference SloScheduler (scheduler.hpp:79-215), call by call."""

    def __init__(self, canvas_w, canvas_h, profile, max_canvases):
        self.dll = dll = load("ref")
        dll.ref_sched_create.restype = C.c_void_p
        dll.ref_sched_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int]
        for n in ("ref_sched_arrival", "ref_sched_timer", "ref_sched_pending", "ref_sched_event"):
            getattr(dll, n).restype = C.c_int
        dll.ref_sched_arrival.argtypes = [C.c_void_p, C.POINTER(Patch), C.c_int64]
        dll.ref_sched_timer.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        dll.ref_sched_pending.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        dll.ref_sched_destroy.argtypes = [C.c_void_p]
        prof, n = _profile_arr(profile)
        self.h = dll.ref_sched_create(canvas_w, canvas_h, prof, n, max_canvases)
        if not self.h:
            raise OracleError(_err(dll, "ref"))

    def __del__(self):
        if getattr(self, "h", None):
            self.dll.ref_sched_destroy(self.h)

    def _events(self, n):
        out = []
        for i in range(n):
            fire, slack = C.c_int64(), C.c_int64()
            trig, k, nid, nf = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            ids = (C.c_uint64 * 4096)()
            pl = (Placement * 4096)()
            fr = (FreeRect * 8192)()
            self.dll.ref_sched_event(C.c_void_p(self.h), i, C.byref(fire), C.byref(trig), C.byref(k),
                                     C.byref(slack), C.byref(nid), ids, pl, C.byref(nf), fr)
            out.append(dict(
                fire_time_us=fire.value, trigger=trig.value, batch_size=k.value,
                estimated_slack_us=slack.value, patch_ids=[ids[j] for j in range(nid.value)],
                placements=[(pl[j].patch_id, pl[j].canvas_index, pl[j].position.x, pl[j].position.y,
                             pl[j].position.w, pl[j].position.h) for j in range(nid.value)],
                free=[(fr[j].canvas, fr[j].r.x, fr[j].r.y, fr[j].r.w, fr[j].r.h)
                      for j in range(nf.value)]))
        return out

    def on_patch_arrival(self, patch: dict, now: int):
        p = Patch(patch["patch_id"], patch.get("source_frame_id", 0), Rect(*patch["rect"]),
                  patch["generation_time_us"], patch["slo_us"], patch["deadline_us"],
                  patch.get("size_bytes", 0))
        n = self.dll.ref_sched_arrival(C.c_void_p(self.h), C.byref(p), now)
        if n < 0:
            raise OracleError(_err(self.dll, "ref"))
        return self._events(n)

    def on_timer(self, now: int, epoch: int):
        n = self.dll.ref_sched_timer(C.c_void_p(self.h), now, epoch)
        ev = self._events(n)
        return ev[0] if ev else None

    def pending_timer(self):
        at, ep = C.c_int64(), C.c_uint64()
        if self.dll.ref_sched_pending(C.c_void_p(self.h), C.byref(at), C.byref(ep)):
            return at.value, ep.value
        return None


# ------------------------------------------------- configs 3/4 on the CPU
def multicam_cpu(cam_frames, cam_t_us, width, height, profile, threads, canvases=None,
                 zones=(4, 4), canvas=(1024, 1024), **sim):
    """The CPU path of configs 3/4 (bench cpu legs): the restated pixel
    stages on every frame of every camera (`threads` workers; the reference's
    own partition / stitch_all inside), the reference simulator tangram::run
    (sim.hpp:206-552, tangram policy) over the extracted RoIs, and every
    invoke event's canvas pixels -- the reference stitch_all of the event's
    patches (= the scheduler's repack, scheduler.hpp:146-160), copied from
    the frames into `canvases` ((K, N, 3M) uint8, preallocated by the caller;
    None skips the pixels).  cam_frames[c] = [background, frame 0, ...].
    Returns dict(events, n_canvases, rois)."""
    lib = "ref"
    n_cams, n = len(cam_frames), len(cam_t_us[0])
    cur = [fr[i + 1] for fr in cam_frames for i in range(n)]
    prev = [fr[i] for fr in cam_frames for i in range(n)]
    params = dict(width=width, height=height, pitch=cam_frames[0][0].shape[1], threshold=25,
                  radius=2, zones_x=zones[0], zones_y=zones[1], canvas_w=canvas[0],
                  canvas_h=canvas[1], bytes_per_pixel=1.5, slo_us=1_000_000, max_rois=1024,
                  threads=threads)
    res = process_frames(params, cur, prev, [i for _ in range(n_cams) for i in range(n)],
                         [t for ts in cam_t_us for t in ts], 0, want_canvases=False, lib=lib)
    rois = [[[tuple(r) for r in res["rois"][c * n + f, :res["n_rois"][c * n + f]].tolist()]
             for f in range(n)] for c in range(n_cams)]
    ref = run_tangram([(cam_t_us[c], rois[c]) for c in range(n_cams)], width, height, profile,
                      zones=zones, canvas=canvas, **sim)
    # the path's patches carry run()'s ids: scene-major, frame order (sim.hpp:249-251)
    where = {}
    for f, plist in enumerate(res["patch_list"]):
        for p in plist:
            where[p["patch_id"]] = (f, p["rect"])
    jobs, offsets = [], [0]
    for e in ref["events"]:
        q = [(i, where[i][1][2], where[i][1][3]) for i in e["patch_ids"]]
        pl, nc, _ = stitch_all(q, canvas[0], canvas[1], lib=lib)
        per = [[] for _ in range(nc)]
        for (i, ci, x, y, w, h) in pl:
            f, r = where[i]
            per[ci].append((f, r[0], r[1], x, y, w, h))
        for lst in per:
            jobs += lst
            offsets.append(len(jobs))
    k = len(offsets) - 1
    if canvases is not None:
        if len(canvases) < k:
            raise OracleError(f"canvas buffer holds {len(canvases)} < {k} canvases")
        jarr = (FillJob * max(1, len(jobs)))(*[FillJob(*j) for j in jobs])
        oarr = (C.c_int64 * len(offsets))(*offsets)
        fptr = (C.c_void_p * max(1, len(cur)))(*[f.ctypes.data for f in cur])
        load("port").orc_fill_jobs(fptr, params["pitch"], jarr, oarr, k, canvas[0], canvas[1],
                                   canvases.ctypes.data, threads)
    return dict(events=ref["events"], n_canvases=k, rois=rois)
